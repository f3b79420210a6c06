# round-2 call 40: k_march tile shape (8x4 default vs 4x8 / 16x2) and occupancy bound at the tiled mapping
for v in default tw4 tw16 tw8_m10 tw8_m6; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  VOLCACHE_B200_LIB=$L timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g40_cfg5_$v.json 2> gpurun_out/g40_cfg5_$v.err
  python -c "import json; d=json.load(open('gpurun_out/g40_cfg5_$v.json')); print('$v', d['roofline']['march_ms_per_frame'], d['value'], d['config']['populate']['seconds'])"
done
