# round-2 call 30: HEAD after the container restore — GPU suite, bench, launch list
python -m pytest tests -m gpu -q > gpurun_out/g30_gputest.log 2>&1; tail -2 gpurun_out/g30_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g30_parity_errors.json
python bench.py > gpurun_out/g30_bench.json 2> gpurun_out/g30_bench.err; cat gpurun_out/g30_bench.json
