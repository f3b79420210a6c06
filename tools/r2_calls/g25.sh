# round-2 call 25: Henyey-Greenstein media extension (GPU suite), the full-spec cfg3 variant bench
python -m pytest tests -m gpu -x -q > gpurun_out/g25_gputest.log 2>&1; tail -2 gpurun_out/g25_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g25_parity_errors.json
python bench.py --media-bounces 4 --hg-g 0.5 --no-cpu-baseline --steps 3 > gpurun_out/g25_bench_hg4.json 2> gpurun_out/g25_bench_hg4.err
python -c "import json; d=json.load(open('gpurun_out/g25_bench_hg4.json')); print(d['value'], d['ms_per_step'], d['config']['workload'])"
