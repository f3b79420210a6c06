# round-2 call 67: deferred bounds check (VC_DEFER_CHECK / vc_check_deferred) — GPU suite, bench x6 with
# per-step end times on the first
python -m pytest tests -m gpu -q > gpurun_out/g67_gputest.log 2>&1; tail -2 gpurun_out/g67_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g67_parity_errors.json
BENCH_STEP_EVENTS=1 python bench.py --no-cpu-baseline > gpurun_out/g67_b0.json 2> gpurun_out/g67_b0.err; grep "step end" gpurun_out/g67_b0.err | cut -c1-420
for i in 1 2 3 4 5 6; do
  python bench.py > gpurun_out/g67_bench_$i.json 2> gpurun_out/g67_bench_$i.err
  python -c "import json; d=json.load(open('gpurun_out/g67_bench_$i.json')); print('full $i', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1))"
done
