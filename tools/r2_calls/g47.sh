# round-2 call 47: HEAD after the hull scan change — GPU suite, bench
python -m pytest tests -m gpu -q > gpurun_out/g47_gputest.log 2>&1; tail -2 gpurun_out/g47_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g47_parity_errors.json
python bench.py > gpurun_out/g47_bench.json 2> gpurun_out/g47_bench.err
python -c "import json; d=json.load(open('gpurun_out/g47_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['largest_by_time'])"
