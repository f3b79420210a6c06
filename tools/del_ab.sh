#!/bin/bash
# A/B of the triangulation kernels: fallback counts and ncu durations of the delaunay
# kernels under a few VOLCACHE_* settings (one 512-record cfg3 wave); raw CSV in gpurun_out/.
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
k=0
for cfg in "$@"; do
  k=$((k+1))
  echo "== $cfg"
  env $cfg VOLCACHE_DEL_STATS=1 python tools/ncu_target.py 512 nowarm 2>&1 | grep "fallback" | tail -1
  env $cfg ncu --clock-control none --metrics $M -k regex:k_delaunay --csv python tools/ncu_target.py 512 nowarm > gpurun_out/del_ab_$k.csv 2>/dev/null
  grep "k_delaunay" gpurun_out/del_ab_$k.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(BuildParams.*)//' | cut -c1-120
done
