#!/bin/bash
# triangulation time (sum of the Delaunay kernels, one 512-record cfg3 wave) per hull window cap
for km in default 24 30 40 48; do
  if [ $km = default ]; then unset VOLCACHE_HULL_KMAX; else export VOLCACHE_HULL_KMAX=$km; fi
  t=$(ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"k_delaunay|k_cap" --csv python tools/ncu_target.py 512 nowarm 2>/dev/null | grep -E "k_delaunay|k_cap" | awk -F'","' '{gsub(/[",]/,"",$NF); s+=$NF} END {print s}')
  echo "kmax $km: $t ns"
done
