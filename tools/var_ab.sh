#!/bin/bash
# ncu durations of kernels matching $1 for the default library and each variant directory
# under paper_1805_09258_b200/lib/variants/ (one 512-record cfg3 wave each).
K=${1:-k_}
for v in default paper_1805_09258_b200/lib/variants/*/libvolcache_b200.so; do
  if [ $v = default ]; then unset VOLCACHE_B200_LIB; else export VOLCACHE_B200_LIB=$PWD/$v; fi
  echo "== $v"
  ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"$K" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null \
    | grep -E "$K" | awk -F'","' '{print $NF, substr($5,1,40)}'
done
