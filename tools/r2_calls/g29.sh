# round-2 call 29: forked triangulation, profiler with one open interval per stream
# (A/B without per-class events via probe3 noprof, then bench for each variant)
for v in default nofork fork_hi; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  for r in 1 2; do VOLCACHE_B200_LIB=$L python tools/probe3.py 2048 noprof 2>&1 | tail -1 | sed "s/^/$v /"; done
  VOLCACHE_B200_LIB=$L python tools/probe3.py 2048 2>&1 | tail -1 | sed "s/^/$v prof /"
  VOLCACHE_B200_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/g29_bench_$v.json 2> gpurun_out/g29_bench_$v.err
  python -c "import json; d=json.load(open('gpurun_out/g29_bench_$v.json')); print('$v bench', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
