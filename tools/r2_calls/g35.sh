# round-2 call 35: measurement set at HEAD — GPU suite, bench (b200 + reference arm), launch list,
# ncu full capture of one wave (summary, traffic, instructions, hot lines), cfg5 bench + k_march capture,
# cfg1 / cfg2 parity variants and the as-specified variants (delta lights, HG)
python -m pytest tests -m gpu -q > gpurun_out/g35_gputest.log 2>&1; tail -2 gpurun_out/g35_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g35_parity_errors.json
python bench.py > gpurun_out/g35_bench.json 2> gpurun_out/g35_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g35_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g35_ncu_launch.log 2>&1
rm -f /tmp/prof.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g35_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/g35_ncu_full.md gpurun_out/g35_traffic.json > /dev/null 2> gpurun_out/g35_summary.err
for k in k_delaunay_hull k_gather_emit k_gather_eval k_gather_occl k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof.ncu-rep "$k" 25 > gpurun_out/g35_lines_$k.txt 2>&1
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g35_cfg5.json 2> gpurun_out/g35_cfg5.err
rm -f /tmp/march.ncu-rep
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_march -c 1 -f -o /tmp/march \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g35_cfg5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/march.ncu-rep gpurun_out/g35_march.md gpurun_out/g35_march_traffic.json > /dev/null 2>&1
python tools/ncu_lines.py /tmp/march.ncu-rep k_march 25 > gpurun_out/g35_lines_k_march.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/g35_bench_ref.json 2> gpurun_out/g35_bench_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g35_torchrun.json 2> gpurun_out/g35_torchrun.err
for c in cfg1 cfg2 cfg1-spec cfg2-spec; do
  timeout 600 python bench.py --config $c --cpu-records 8 > gpurun_out/g35_bench_$c.json 2> gpurun_out/g35_bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/g35_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('cpu_baseline',{}).get('value'))"
done
