# round-2 call 50: run-to-run spread of the bench line at HEAD (8 runs, no CPU baseline leg)
for i in 1 2 3 4 5 6 7 8; do
  python bench.py --no-cpu-baseline > gpurun_out/g50_bench_$i.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/g50_bench_$i.json')); print($i, round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1))"
done
