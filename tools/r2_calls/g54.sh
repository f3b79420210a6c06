# round-2 call 54: lookup span 0.35 as the default — GPU suite, cfg5 bench, k_march capture, cfg3 bench
python -m pytest tests -m gpu -q > gpurun_out/g54_gputest.log 2>&1; tail -2 gpurun_out/g54_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g54_parity_errors.json
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g54_cfg5.json 2> gpurun_out/g54_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/g54_cfg5.json')); print('cfg5', d['value'], d['roofline'], d['config']['populate']['seconds'], d['e2e'])"
rm -f /tmp/march.ncu-rep
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_march -c 1 -f -o /tmp/march \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g54_cfg5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/march.ncu-rep gpurun_out/g54_march.md gpurun_out/g54_march_traffic.json > /dev/null 2>&1
python tools/ncu_lines.py /tmp/march.ncu-rep k_march 30 > gpurun_out/g54_lines_k_march.txt 2>&1
head -24 gpurun_out/g54_march.md | tail -18
python bench.py --no-cpu-baseline > gpurun_out/g54_bench.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g54_bench.json')); print('bench', d['value'], d['ms_per_step'])"
