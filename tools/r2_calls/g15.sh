# round-2 call 15: non-reflective specialisations of k_primary / k_march (no direct-lighting code),
# survivor-evaluation grid; GPU suite, bench, cfg5, populate
python -m pytest tests -m gpu -x -q > gpurun_out/g15_gputest.log 2>&1; tail -3 gpurun_out/g15_gputest.log
python tools/probe3.py 2048 > gpurun_out/g15_probe.txt 2>&1; tail -1 gpurun_out/g15_probe.txt
python bench.py > gpurun_out/g15_bench.json 2> gpurun_out/g15_bench.err
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g15_cfg5.json 2> gpurun_out/g15_cfg5.err
timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g15_pop.json 2>&1
