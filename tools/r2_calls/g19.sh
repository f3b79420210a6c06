# round-2 call 19: incremental record index (appended records in a second index part);
# GPU suite, populate phases, cfg5, speculation waste target with the cheaper windows
python -m pytest tests -m gpu -x -q > gpurun_out/g19_gputest.log 2>&1; tail -3 gpurun_out/g19_gputest.log
VOLCACHE_POP_TIMING=1 timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g19_pop.json 2> gpurun_out/g19_pop.err
grep "populate phases" gpurun_out/g19_pop.err | tail -1
for w in 1.0 0.5 0.3; do VOLCACHE_POP_WASTE=$w timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g19_pop_w$w.json 2>&1; tail -1 gpurun_out/g19_pop_w$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['wall_s'], d['windows'], d['builds'])"; done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g19_cfg5.json 2> gpurun_out/g19_cfg5.err
