# round-2 call 5: float32 element math in the assembly (GPU suite + parity errors), variants, bench
python -m pytest tests -m gpu -x -q > gpurun_out/g5_gputest.log 2>&1; tail -3 gpurun_out/g5_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g5_parity_errors.json
bash tools/variants.sh > gpurun_out/g5_variants.txt 2>&1
cat gpurun_out/g5_variants.txt
python bench.py > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err
