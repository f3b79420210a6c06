# round-2 call 64: bench with NVML warmed before the timed region — 12 runs with the CPU-baseline leg skipped,
# then the full default line twice (fresh processes each time)
for i in 1 2 3 4 5 6 7 8 9 10 11 12; do
  python bench.py --no-cpu-baseline > gpurun_out/g64_bench_$i.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/g64_bench_$i.json')); print($i, round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), d['clocks']['samples'])"
done
python bench.py > gpurun_out/g64_bench.json 2> gpurun_out/g64_bench.err
python -c "import json; d=json.load(open('gpurun_out/g64_bench.json')); print('full', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/g64_cfg1.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g64_cfg1.json')); print('cfg1', d['value'], d['clocks'])"
