# round-2 call 12: populate phase timing at cfg5 size (engine cell span) + per-kernel class times
VOLCACHE_POP_TIMING=1 timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g12_pop.json 2> gpurun_out/g12_pop.err
timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g12_pop_notiming.json 2>&1
