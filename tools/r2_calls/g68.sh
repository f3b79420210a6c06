# round-2 call 68: the driver's round-end sequence at HEAD — GPU suite (-x), smoke, reference arm, bench,
# torchrun launch at world size 1
python -m pytest tests/ -x -q -m gpu > gpurun_out/g68_gputest.log 2>&1; tail -2 gpurun_out/g68_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g68_smoke.log 2>&1; tail -1 gpurun_out/g68_smoke.log
python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 > gpurun_out/g68_bench_ref.json 2> gpurun_out/g68_bench_ref.err; cut -c1-200 gpurun_out/g68_bench_ref.json
python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/g68_bench.json 2> gpurun_out/g68_bench.err
python -c "import json; d=json.load(open('gpurun_out/g68_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e'], d['roofline']['kernel'], d['roofline']['frac'], d['gpu_launches'], d['clocks'])"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/g68_torchrun.json 2> gpurun_out/g68_torchrun.err
python -c "import json; d=json.load(open('gpurun_out/g68_torchrun.json')); print('torchrun', d['value'], d['ms_per_step'], d['e2e']['value'])"
