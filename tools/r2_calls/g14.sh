# round-2 call 14: gather emitter pass split into filter / survivor evaluation / redo (GPU suite, A/B, bench)
python -m pytest tests -m gpu -x -q > gpurun_out/g14_gputest.log 2>&1; tail -3 gpurun_out/g14_gputest.log
bash tools/variants.sh > gpurun_out/g14_variants.txt 2>&1; cat gpurun_out/g14_variants.txt
ncu --clock-control none --metrics gpu__time_duration.sum,sm__inst_executed.sum,smsp__sass_inst_executed_op_local_ld.sum -k regex:"k_gather" --csv python tools/ncu_target.py 2048 nowarm > gpurun_out/g14_ncu_gather.csv 2>/dev/null
python bench.py > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err
timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g14_pop.json 2>&1
