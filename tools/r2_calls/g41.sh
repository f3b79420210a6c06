# round-2 call 41: HEAD with the tiled march and 128-thread primary CTAs — GPU suite, bench, cfg5 bench,
# k_march capture, launch list
python -m pytest tests -m gpu -q > gpurun_out/g41_gputest.log 2>&1; tail -2 gpurun_out/g41_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g41_parity_errors.json
python bench.py > gpurun_out/g41_bench.json 2> gpurun_out/g41_bench.err
python -c "import json; d=json.load(open('gpurun_out/g41_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g41_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g41_ncu_launch.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g41_cfg5.json 2> gpurun_out/g41_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/g41_cfg5.json')); print('cfg5', d['value'], d['roofline'], d['config']['populate']['seconds'])"
rm -f /tmp/march.ncu-rep
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_march -c 1 -f -o /tmp/march \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g41_cfg5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/march.ncu-rep gpurun_out/g41_march.md gpurun_out/g41_march_traffic.json > /dev/null 2>&1
python tools/ncu_lines.py /tmp/march.ncu-rep k_march 30 > gpurun_out/g41_lines_k_march.txt 2>&1
cat gpurun_out/g41_march.md | head -40
