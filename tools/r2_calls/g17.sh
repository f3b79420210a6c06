# round-2 call 17: k_march occupancy (min CTAs per SM 4 / 5 / 6 / 8) on the cfg5 frame
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g17_cfg5_m5.json 2> gpurun_out/g17_cfg5_m5.err
for m in 4 6 8; do VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/march$m.so timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g17_cfg5_m$m.json 2> gpurun_out/g17_cfg5_m$m.err; done
for m in 4 5 6 8; do python -c "import json; d=json.load(open('gpurun_out/g17_cfg5_m$m.json')); print($m, d['ms_per_step'], d['config']['populate']['seconds'])"; done
