# round-2 call 39: k_march pixel mapping (8x4 tiles per warp vs 32x1 strips) and CTA size, cfg5 frame;
# render parity tests on the tiled variant
for v in default mtile mtile64 mbs64 mbs32; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  VOLCACHE_B200_LIB=$L timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g39_cfg5_$v.json 2> gpurun_out/g39_cfg5_$v.err
  python -c "import json; d=json.load(open('gpurun_out/g39_cfg5_$v.json')); print('$v', d['roofline']['march_ms_per_frame'], d['value'], d['config']['populate']['seconds'])"
done
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/mtile.so python -m pytest tests -m gpu -q -x -k "render or march or crop or populate or grow or dist" 2>&1 | tail -3
