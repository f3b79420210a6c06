# round-2 call 53: lookup index — smaller cell spans
for cfg in "0.5 3" "0.35 0" "0.35 2" "0.25 0" "0.25 2" "0.18 2"; do
  set -- $cfg
  VOLCACHE_IDX_SPAN=$1 VOLCACHE_IDX_LONG_CAP=$2 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g53_cfg5.json 2> gpurun_out/g53_cfg5.err
  python -c "import json; d=json.load(open('gpurun_out/g53_cfg5.json')); print('span $1 cap $2', round(d['roofline']['march_ms_per_frame'],2), round(d['value']/1e9,3), d['config']['records'], round(d['config']['populate']['seconds'],2))" || tail -3 gpurun_out/g53_cfg5.err
done
