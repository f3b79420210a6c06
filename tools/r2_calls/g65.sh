# round-2 call 65: where the occasional ~50-70 ms of idle time in the timed region comes from — full and
# --no-cpu-baseline runs alternated, with per-step end times
for i in 1 2 3 4 5 6; do
  BENCH_STEP_EVENTS=1 python bench.py --cpu-records 1 > gpurun_out/g65_full_$i.json 2> gpurun_out/g65_full_$i.err
  python -c "import json; d=json.load(open('gpurun_out/g65_full_$i.json')); print('full $i', round(d['value'],1), round(d['ms_per_step'],3))"; grep "step end" gpurun_out/g65_full_$i.err | cut -c1-400
  BENCH_STEP_EVENTS=1 python bench.py --no-cpu-baseline > gpurun_out/g65_nocpu_$i.json 2> gpurun_out/g65_nocpu_$i.err
  python -c "import json; d=json.load(open('gpurun_out/g65_nocpu_$i.json')); print('nocpu $i', round(d['value'],1), round(d['ms_per_step'],3))"; grep "step end" gpurun_out/g65_nocpu_$i.err | cut -c1-400
done
