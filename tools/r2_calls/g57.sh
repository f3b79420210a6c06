# round-2 call 57: assembly CTAs per record by record size (VOLCACHE_ASM_SPLIT) on cfg1 (2D, n = 1024),
# cfg2 (3D, n = 4096) and cfg3 (n = 16384)
for c in cfg1 cfg2; do for s in 1 2 4 8 16 32; do
  VOLCACHE_ASM_SPLIT=$s python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/g57.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/g57.json')); print('$c split $s', round(d['value']), round(d['ms_per_step'],3))"
done; done
python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/g57.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g57.json')); print('cfg1 rule', round(d['value']), round(d['ms_per_step'],3))"
python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/g57.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g57.json')); print('cfg2 rule', round(d['value']), round(d['ms_per_step'],3))"
python bench.py --no-cpu-baseline > gpurun_out/g57.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g57.json')); print('cfg3 rule', round(d['value']), round(d['ms_per_step'],3))"
