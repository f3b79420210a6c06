# round-2 call 63: ncu full capture of one wave at HEAD (after the emission-table change) + bench
python bench.py > gpurun_out/g63_bench.json 2> gpurun_out/g63_bench.err
python -c "import json; d=json.load(open('gpurun_out/g63_bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g63_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g63_ncu_launch.log 2>&1
rm -f /tmp/prof.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g63_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/g63_ncu_full.md gpurun_out/g63_traffic.json > /dev/null 2> gpurun_out/g63_summary.err
for k in k_delaunay_hull k_gather_emit k_gather_eval k_gather_occl_pt k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof.ncu-rep "$k" 25 > gpurun_out/g63_lines_$k.txt 2>&1
done
python -c "import json; print(json.load(open('gpurun_out/g63_traffic.json'))['per_class'])"
