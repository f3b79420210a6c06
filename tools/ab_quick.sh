#!/bin/bash
# GPU suite + per-kernel ncu durations of one 512-record cfg3 wave (regex $1) + bench line
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"${1:-k_}" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -E "${1:-k_}" | awk -F'","' '{print $NF, substr($5,1,40)}'
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_share'])"
