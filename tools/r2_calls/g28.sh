# round-2 call 28: triangulation on a forked side stream beside the rings + gather chain
# (GPU suite on the forked default; bench A/B: default, no fork, high-priority side stream)
python -m pytest tests -m gpu -x -q > gpurun_out/g28_gputest.log 2>&1; tail -2 gpurun_out/g28_gputest.log
for v in default nofork fork_hi default; do
  if [ $v = default ]; then L=paper_1805_09258_b200/lib/libvolcache_b200.so; else L=paper_1805_09258_b200/lib/variants/$v.so; fi
  VOLCACHE_B200_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/g28_bench_$v.json 2> gpurun_out/g28_bench_$v.err
  python -c "import json; d=json.load(open('gpurun_out/g28_bench_$v.json')); print('$v', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
