# round-2 call 18: paired BVH node layout with packed FFMA2 slab tests; k_march at 8 CTAs/SM
python -m pytest tests -m gpu -x -q > gpurun_out/g18_gputest.log 2>&1; tail -3 gpurun_out/g18_gputest.log
python tools/probe3.py 2048 > gpurun_out/g18_probe.txt 2>&1; tail -1 gpurun_out/g18_probe.txt
python bench.py > gpurun_out/g18_bench.json 2> gpurun_out/g18_bench.err
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g18_cfg5.json 2> gpurun_out/g18_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/g18_bench.json')); print(d['value'], d['ms_per_step']); c=json.load(open('gpurun_out/g18_cfg5.json')); print(c['ms_per_step'], c['config']['populate']['seconds'])"
