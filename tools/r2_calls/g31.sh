# round-2 call 31: delta-light extension — GPU suite, default bench (regression check), lit variants
python -m pytest tests -m gpu -q -x > gpurun_out/g31_gputest.log 2>&1; tail -5 gpurun_out/g31_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g31_parity_errors.json
python bench.py --no-cpu-baseline > gpurun_out/g31_bench.json 2> gpurun_out/g31_bench.err; python -c "import json; d=json.load(open('gpurun_out/g31_bench.json')); print('default', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 600 python bench.py --no-cpu-baseline --lights lamp --steps 3 > gpurun_out/g31_bench_lamp.json 2> gpurun_out/g31_bench_lamp.err; python -c "import json; d=json.load(open('gpurun_out/g31_bench_lamp.json')); print('lamp', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --no-cpu-baseline --lights sun --hg-g 0.5 --media-bounces 4 --steps 3 --records-per-step 512 > gpurun_out/g31_bench_spec.json 2> gpurun_out/g31_bench_spec.err; python -c "import json; d=json.load(open('gpurun_out/g31_bench_spec.json')); print('spec', d['value'], d['ms_per_step'])"
