# round-2 call 6: GPU suite (cfg3 bench-workload reference fixture, multi-GPU populate hook),
# bench (CPU baseline over 4 spread records), the reference's own tests rebound to the device
python -m pytest tests -m gpu -x -q > gpurun_out/g6_gputest.log 2>&1; tail -3 gpurun_out/g6_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g6_parity_errors.json
python bench.py > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
bash tools/run_reference_tests.sh
