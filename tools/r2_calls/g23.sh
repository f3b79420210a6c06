# round-2 call 23: bench repeat (host-gap check)
for i in 1 2 3; do python bench.py --no-cpu-baseline > gpurun_out/g23_bench$i.json 2> gpurun_out/g23_bench$i.err; python -c "import json; d=json.load(open('gpurun_out/g23_bench$i.json')); s=sum(v['ms'] for v in d['roofline']['per_kernel'].values())/d['steps']; print(d['value'], d['ms_per_step'], round(s,2), d['e2e']['value'])"; done
nproc; uptime
