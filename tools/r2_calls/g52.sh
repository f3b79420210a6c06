# round-2 call 52: lookup index — cell span x long-axis cap
for cfg in "1 0" "0.75 0" "0.5 0" "1 2" "1 1.5" "0.75 2" "0.75 1.5" "0.5 2"; do
  set -- $cfg
  VOLCACHE_IDX_SPAN=$1 VOLCACHE_IDX_LONG_CAP=$2 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g52_cfg5.json 2> gpurun_out/g52_cfg5.err
  python -c "import json; d=json.load(open('gpurun_out/g52_cfg5.json')); print('span $1 cap $2', round(d['roofline']['march_ms_per_frame'],2), round(d['value']/1e9,3), d['config']['records'])"
done
