#!/bin/bash
# time the default library and each experiment variant on the cfg3 probe
python tools/probe3.py 2048 2>&1 | tail -1 | sed 's/^/default /'
for v in paper_1805_09258_b200/lib/variants/*.so; do
  VOLCACHE_B200_LIB=$v python tools/probe3.py 2048 2>&1 | tail -1 | sed "s|^|$(basename $v) |"
done
