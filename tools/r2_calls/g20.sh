# round-2 call 20: populate speculation waste target (default now 0.3) — 0.2 / 0.15 / 0.1
for w in 0.3 0.2 0.15 0.1; do VOLCACHE_POP_WASTE=$w timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g20_pop_w$w.json 2>&1; tail -1 gpurun_out/g20_pop_w$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['wall_s'], d['windows'], d['builds'], d['records'])"; done
python -m pytest tests -m gpu -x -q -k populate > gpurun_out/g20_gputest.log 2>&1; tail -2 gpurun_out/g20_gputest.log
