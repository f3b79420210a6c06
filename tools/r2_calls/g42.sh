# round-2 call 42: blend with precomputed M and FMAs (VC_BLEND_FAST) vs the reference-order blend —
# cache / render / populate parity tests, cfg5 frame A/B
python -m pytest tests -m gpu -q -x -k "render or march or crop or populate or grow or dist or interpolate or cache or lookup or baseline or dropin or io" 2>&1 | tail -3
for v in default blend_ref blend_nofb; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  VOLCACHE_B200_LIB=$L timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g42_cfg5_$v.json 2> gpurun_out/g42_cfg5_$v.err
  python -c "import json; d=json.load(open('gpurun_out/g42_cfg5_$v.json')); print('$v', d['roofline']['march_ms_per_frame'], d['value'], d['config']['populate']['seconds'], d['config']['records'])"
done
