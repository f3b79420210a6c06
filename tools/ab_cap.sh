python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/del_check.py 1024 4096 16384 > gpurun_out/del_check.log 2>&1; tail -9 gpurun_out/del_check.log
for e in 0 1; do
  echo "== CAP_GRID=$e"
  VOLCACHE_CAP_GRID=$e VOLCACHE_DEL_STATS=1 python tools/ncu_target.py 512 nowarm 2>&1 | grep fallback | tail -1
  VOLCACHE_CAP_GRID=$e ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"k_delaunay|k_cap" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -E "k_delaunay|k_cap" | awk -F'","' '{print $NF, substr($5,1,40)}'
done
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'])"
