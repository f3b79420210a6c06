# round-2 call 7: hull-kernel culling (GPU suite; triangulation timing per cull radius and
# hand-back counts), the reference's own tests rebound again
python -m pytest tests -m gpu -x -q > gpurun_out/g7_gputest.log 2>&1; tail -3 gpurun_out/g7_gputest.log
for c in 0 2.0 2.5 3.0 3.5; do VOLCACHE_HULL_CULL=$c python tools/probe3.py 2048 2>&1 | tail -1 | sed "s/^/cull$c /" >> gpurun_out/g7_cull.txt; done
for c in 0 2.5 3.0; do VOLCACHE_HULL_CULL=$c VOLCACHE_DEL_STATS=1 python tools/probe3.py 512 2>&1 | grep -i -E "handed|fallback|cells|del" | head -5 | sed "s/^/cull$c /" >> gpurun_out/g7_cull.txt; done
cat gpurun_out/g7_cull.txt
bash tools/run_reference_tests.sh
