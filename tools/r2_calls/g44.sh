# round-2 call 44: final measurement set at HEAD — smoke, GPU suite, bench (b200 + reference arm), launch
# list, ncu full capture of one wave (summary, traffic, instruction counts, hot lines)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g44_smoke.log 2>&1; tail -1 gpurun_out/g44_smoke.log
python -m pytest tests -m gpu -q > gpurun_out/g44_gputest.log 2>&1; tail -2 gpurun_out/g44_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g44_parity_errors.json
python bench.py > gpurun_out/g44_bench.json 2> gpurun_out/g44_bench.err
python -c "import json; d=json.load(open('gpurun_out/g44_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g44_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g44_ncu_launch.log 2>&1
rm -f /tmp/prof.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g44_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/g44_ncu_full.md gpurun_out/g44_traffic.json > /dev/null 2> gpurun_out/g44_summary.err
for k in k_delaunay_hull k_gather_emit k_gather_eval k_gather_occl_pt k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof.ncu-rep "$k" 25 > gpurun_out/g44_lines_$k.txt 2>&1
done
timeout 900 python bench.py --impl reference > gpurun_out/g44_bench_ref.json 2> gpurun_out/g44_bench_ref.err
cat gpurun_out/g44_bench_ref.json | cut -c1-400
timeout 600 python bench.py --config cfg4-standin --steps 3 --records-per-step 512 --no-cpu-baseline > gpurun_out/g44_bench_cfg4standin.json 2> gpurun_out/g44_bench_cfg4standin.err
python -c "import json; d=json.load(open('gpurun_out/g44_bench_cfg4standin.json')); print('cfg4-standin', d['value'], d['ms_per_step'])"
