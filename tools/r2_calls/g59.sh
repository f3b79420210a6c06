# round-2 call 59: final measurement set at HEAD — smoke, GPU suite, bench (b200 + reference arm), launch
# list, ncu full capture of one wave, cfg5 bench + k_march capture, cfg1 / cfg2 and the extension variants
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g59_smoke.log 2>&1; tail -1 gpurun_out/g59_smoke.log
python -m pytest tests -m gpu -q > gpurun_out/g59_gputest.log 2>&1; tail -2 gpurun_out/g59_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g59_parity_errors.json
python bench.py > gpurun_out/g59_bench.json 2> gpurun_out/g59_bench.err
python -c "import json; d=json.load(open('gpurun_out/g59_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g59_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g59_ncu_launch.log 2>&1
rm -f /tmp/prof.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g59_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/g59_ncu_full.md gpurun_out/g59_traffic.json > /dev/null 2> gpurun_out/g59_summary.err
for k in k_delaunay_hull k_gather_emit k_gather_eval k_gather_occl_pt k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof.ncu-rep "$k" 25 > gpurun_out/g59_lines_$k.txt 2>&1
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g59_cfg5.json 2> gpurun_out/g59_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/g59_cfg5.json')); print('cfg5', d['value'], d['roofline']['march_ms_per_frame'], d['config']['populate']['seconds'])"
timeout 900 python bench.py --impl reference > gpurun_out/g59_bench_ref.json 2> gpurun_out/g59_bench_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g59_torchrun.json 2> gpurun_out/g59_torchrun.err
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/g59_bench_$tag.json 2> gpurun_out/g59_bench_$tag.err; python -c "import json; d=json.load(open('gpurun_out/g59_bench_$tag.json')); print('$tag', round(d['value'],1), round(d['ms_per_step'],3), (d.get('cpu_baseline') or {}).get('value'))"; }
run cfg1 --config cfg1 --cpu-records 8
run cfg2 --config cfg2 --cpu-records 8
run cfg1spec --config cfg1-spec --cpu-records 8
run cfg2spec --config cfg2-spec --cpu-records 8
run hg1 --hg-g 0.5 --steps 5 --no-cpu-baseline
run lamp --lights lamp --steps 3 --no-cpu-baseline
run sun --lights sun --steps 3 --no-cpu-baseline
run spec --lights sun --hg-g 0.5 --media-bounces 4 --steps 3 --records-per-step 512 --no-cpu-baseline
run cfg4standin --config cfg4-standin --steps 3 --records-per-step 512 --no-cpu-baseline
