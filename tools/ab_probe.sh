for r in 1 2; do
 for v in default em10 em6; do
  if [ $v = default ]; then unset VOLCACHE_B200_LIB; else export VOLCACHE_B200_LIB=$PWD/paper_1805_09258_b200/build/$v/libvolcache_b200.so; fi
  echo -n "$v "; python tools/probe3.py 2048 2>&1 | tail -1
 done
done
unset VOLCACHE_B200_LIB
