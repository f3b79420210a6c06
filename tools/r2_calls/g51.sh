# round-2 call 51: index level from the middle AABB extent (long records span more, smaller cells) —
# cfg5 frame per cap, lookup parity tests at one cap
for c in 0 2 3 4 6; do
  VOLCACHE_IDX_LONG_CAP=$c timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g51_cfg5_$c.json 2> gpurun_out/g51_cfg5_$c.err
  python -c "import json; d=json.load(open('gpurun_out/g51_cfg5_$c.json')); print('cap $c', d['roofline']['march_ms_per_frame'], d['value'], d['config']['populate']['seconds'], d['config']['records'])"
done
VOLCACHE_IDX_LONG_CAP=3 python -m pytest tests -m gpu -q -x -k "render or march or crop or populate or grow or interpolate or cache or lookup" 2>&1 | tail -2
