#!/bin/bash
# summed ncu durations of kernels matching $1 for the default library and each variant
K=${1:-k_}
for v in default paper_1805_09258_b200/lib/variants/*/libvolcache_b200.so; do
  if [ $v = default ]; then unset VOLCACHE_B200_LIB; else export VOLCACHE_B200_LIB=$PWD/$v; fi
  t=$(ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"$K" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -E "$K" | awk -F'","' '{gsub(/[",]/,"",$NF); s+=$NF} END {print s}')
  echo "$v: $t ns"
done
