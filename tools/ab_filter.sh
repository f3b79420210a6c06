#!/bin/bash
# gather pre-filter A/B: parity tests, kernel times with the filter off/on, bench line
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
for e in 0 1; do
  echo "== EMIT_FILTER=$e"
  VOLCACHE_EMIT_FILTER=$e ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"k_gather" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -E "k_gather" | awk -F'","' '{print $NF, substr($5,1,40)}'
done
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_share'])"
