# round-2 call 3: GPU suite with the shared-stack / float32-pretest traversal; A/B of variants + leaf sizes
python -m pytest tests -m gpu -x -q > gpurun_out/g3_gputest.log 2>&1; tail -3 gpurun_out/g3_gputest.log
bash tools/variants.sh > gpurun_out/g3_variants.txt 2>&1
for lf in 2 4 6; do VOLCACHE_LEAF_GEO=$lf python tools/probe3.py 2048 2>&1 | tail -1 | sed "s/^/leaf$lf /" >> gpurun_out/g3_variants.txt; done
cat gpurun_out/g3_variants.txt
ncu --clock-control none --metrics gpu__time_duration.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.sum -k regex:"k_primary|k_gather" --csv python tools/ncu_target.py 2048 nowarm > gpurun_out/g3_ncu_ray.csv 2>/dev/null
python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
VOLCACHE_POP_TIMING=1 timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g3_pop.json 2> gpurun_out/g3_pop.err
