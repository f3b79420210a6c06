# round-2 call 49: HEAD with 128-thread emitter filter / evaluation CTAs — GPU suite, bench
python -m pytest tests -m gpu -q > gpurun_out/g49_gputest.log 2>&1; tail -2 gpurun_out/g49_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g49_parity_errors.json
python bench.py > gpurun_out/g49_bench.json 2> gpurun_out/g49_bench.err
python -c "import json; d=json.load(open('gpurun_out/g49_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
