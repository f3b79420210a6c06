# round-2 call 22: emitter filter from raw draw mantissas + MUFU sincos (filter kernel only)
python -m pytest tests -m gpu -x -q > gpurun_out/g22_gputest.log 2>&1; tail -2 gpurun_out/g22_gputest.log
python tools/probe3.py 2048 > gpurun_out/g22_probe.txt 2>&1; tail -1 gpurun_out/g22_probe.txt
ncu --clock-control none --metrics gpu__time_duration.sum,sm__inst_executed.sum -k regex:"k_gather_emit" --csv python tools/ncu_target.py 2048 nowarm 2>/dev/null | grep -E "k_gather_emit<3, 1>" | head -4
python bench.py --no-cpu-baseline > gpurun_out/g22_bench.json 2> gpurun_out/g22_bench.err
timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g22_pop.json 2>&1; tail -1 gpurun_out/g22_pop.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['wall_s'], d['kernel_ms'])"
