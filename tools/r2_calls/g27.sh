# round-2 call 27: persistent-lane primary pass (GPU suite, A/B vs the grid-stride kernel, bench)
python -m pytest tests -m gpu -x -q > gpurun_out/g27_gputest.log 2>&1; tail -2 gpurun_out/g27_gputest.log
bash tools/variants.sh > gpurun_out/g27_variants.txt 2>&1; cat gpurun_out/g27_variants.txt
ncu --clock-control none --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.sum -k regex:"k_primary" --csv python tools/ncu_target.py 2048 nowarm 2>/dev/null | grep "k_primary" | awk -F'","' '{print $5, $(NF-2), $NF}' | head -6
python bench.py --no-cpu-baseline > gpurun_out/g27_bench.json 2> gpurun_out/g27_bench.err; python -c "import json; d=json.load(open('gpurun_out/g27_bench.json')); print(d['value'], d['ms_per_step'])"
