# round-2 call 56: assembly on 32 CTAs per record — GPU suite, cfg3 / cfg1 / cfg2 bench, cfg5 bench
python -m pytest tests -m gpu -q > gpurun_out/g56_gputest.log 2>&1; tail -2 gpurun_out/g56_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g56_parity_errors.json
python bench.py > gpurun_out/g56_bench.json 2> gpurun_out/g56_bench.err
python -c "import json; d=json.load(open('gpurun_out/g56_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'])"
for c in cfg1 cfg2; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/g56_bench_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/g56_bench_$c.json')); print('$c', d['value'], d['ms_per_step'])"
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g56_cfg5.json 2> gpurun_out/g56_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/g56_cfg5.json')); print('cfg5', d['value'], d['roofline']['march_ms_per_frame'], d['config']['populate']['seconds'], d['config']['records'])"
