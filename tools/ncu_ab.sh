#!/bin/bash
# Instruction counts of one kernel for the default library and a variant (A/B under ncu).
K=${1:-k_delaunay_smem}; V=${2:-ww}
M=gpu__time_duration.sum,sm__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for v in default $V; do
  if [ $v = default ]; then unset VOLCACHE_B200_LIB; else export VOLCACHE_B200_LIB=$PWD/paper_1805_09258_b200/build/$v/libvolcache_b200.so; fi
  echo "== $v"; ncu --metrics $M -k regex:$K -c 1 --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -v "^==" | cut -d, -f12-
done
