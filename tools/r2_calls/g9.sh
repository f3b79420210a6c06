# round-2 call 9: GPU suite, bench lines (b200 + reference arm), launch list, ncu full capture
# of one 2048-record wave (summary, traffic, hot lines), cfg5 bench + k_march capture, populate phases
python -m pytest tests -m gpu -x -q > gpurun_out/g9_gputest.log 2>&1; tail -3 gpurun_out/g9_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g9_parity_errors.json
python bench.py > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g9_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g9_ncu_launch.log 2>&1
rm -f /tmp/prof_round.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof_round \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g9_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_round.ncu-rep gpurun_out/g9_ncu_full.md gpurun_out/g9_traffic.json > /dev/null 2> gpurun_out/g9_summary.err
for k in k_delaunay_hull k_delaunay_capg k_delaunay_warp k_gather_emit k_gather_occl k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof_round.ncu-rep "$k" 25 > gpurun_out/g9_lines_$k.txt 2>&1
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g9_cfg5.json 2> gpurun_out/g9_cfg5.err
rm -f /tmp/march.ncu-rep
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_march -c 1 -f -o /tmp/march \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g9_cfg5_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/march.ncu-rep gpurun_out/g9_march.md gpurun_out/g9_march_traffic.json > /dev/null 2>&1
python tools/ncu_lines.py /tmp/march.ncu-rep k_march 30 > gpurun_out/g9_lines_k_march.txt 2>&1
VOLCACHE_POP_TIMING=1 timeout 600 python tools/populate_probe.py 1920 1080 0.01 3e-5 16384 > gpurun_out/g9_pop.json 2> gpurun_out/g9_pop.err
timeout 600 python bench.py --impl reference > gpurun_out/g9_bench_ref.json 2> gpurun_out/g9_bench_ref.err
