# round-2 call 11: GPU suite (multi-bounce media extension, lookup cell span 1 after populate),
# bench (issue-rate fractions), cfg5 bench, the 4-bounce cfg3 variant
python -m pytest tests -m gpu -x -q > gpurun_out/g11_gputest.log 2>&1; tail -3 gpurun_out/g11_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g11_parity_errors.json
python bench.py > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g11_cfg5.json 2> gpurun_out/g11_cfg5.err
python bench.py --media-bounces 4 --no-cpu-baseline > gpurun_out/g11_bench_4bounce.json 2> gpurun_out/g11_bench_4bounce.err
