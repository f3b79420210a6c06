# round-2 call 8: emitter-plane direction-sign pre-test in the gather (GPU suite, A/B), bench,
# populate phase timing with the hash index
python -m pytest tests -m gpu -x -q > gpurun_out/g8_gputest.log 2>&1; tail -3 gpurun_out/g8_gputest.log
bash tools/variants.sh > gpurun_out/g8_variants.txt 2>&1; cat gpurun_out/g8_variants.txt
python bench.py > gpurun_out/g8_bench.json 2> gpurun_out/g8_bench.err
VOLCACHE_POP_TIMING=1 timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g8_pop.json 2> gpurun_out/g8_pop.err
