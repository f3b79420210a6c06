nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_gputest.log
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
timeout 1500 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g1_cfg5.json 2> gpurun_out/g1_cfg5.err; echo "cfg5 rc=$?" >> gpurun_out/g1_cfg5.err
