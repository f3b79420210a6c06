#!/bin/bash
# BVH leaf-size sweep on the cfg3 probe (env knobs read at scene upload)
for ge in "1 2" "2 1" "2 2" "3 2" "4 2" "2 4"; do set -- $ge
  echo -n "geo=$1 emit=$2 "; VOLCACHE_LEAF_GEO=$1 VOLCACHE_LEAF_EMIT=$2 python tools/probe3.py 2048 2>&1 | tail -1 | cut -c1-200
done
