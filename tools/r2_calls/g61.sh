# round-2 call 61: polar-row (cap) triangulation kernels on a side stream beside the hull classes —
# triangulation tests, per-class probe and bench A/B
python -m pytest tests -m gpu -q -x -k "delaunay or triangulation or hull or qhull or full_size or records_vs" 2>&1 | tail -2
bash tools/variants.sh
for v in default capfork_off capfork_hi default capfork_off; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  VOLCACHE_B200_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/g61.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/g61.json')); print('$v bench', round(d['value'],1), round(d['ms_per_step'],3))"
done
