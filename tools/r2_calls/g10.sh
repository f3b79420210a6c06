# round-2 call 10: record-index cell span (cfg5 march + populate), emitter-pass occupancy, populate
# speculation waste target, per-kernel instruction counts of one wave (issue-rate model)
python -m pytest tests -m gpu -x -q -k "interp or render or populate or cache" > gpurun_out/g10_gputest.log 2>&1; tail -2 gpurun_out/g10_gputest.log
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/span1.so python -m pytest tests -m gpu -x -q -k "interp or render or populate or cache" > gpurun_out/g10_gputest_span1.log 2>&1; tail -2 gpurun_out/g10_gputest_span1.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g10_cfg5.json 2> gpurun_out/g10_cfg5.err
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/span1.so timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g10_cfg5_span1.json 2> gpurun_out/g10_cfg5_span1.err
for w in 0.5 0.25; do VOLCACHE_POP_WASTE=$w timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g10_pop_w$w.json 2>&1; done
bash tools/variants.sh > gpurun_out/g10_variants.txt 2>&1; cat gpurun_out/g10_variants.txt
ncu --clock-control none --metrics gpu__time_duration.sum,sm__inst_executed.sum --csv python tools/ncu_target.py 2048 nowarm > gpurun_out/g10_inst.csv 2>/dev/null
