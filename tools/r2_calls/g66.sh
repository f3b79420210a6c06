# round-2 call 66: the default bench line (CPU-baseline leg included) 6 times with per-step end times
for i in 1 2 3 4 5 6; do
  BENCH_STEP_EVENTS=1 python bench.py > gpurun_out/g66_full_$i.json 2> gpurun_out/g66_full_$i.err
  python -c "import json; d=json.load(open('gpurun_out/g66_full_$i.json')); print('full $i', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1))"; grep "step end" gpurun_out/g66_full_$i.err | cut -c1-420
done
