# round-2 call 37: ncu full capture of one wave again, summarised with every gather kernel in its class
# (k_gather_eval and k_gather_occl_pt were missing from the class map: the gather's traffic and
# instruction totals read by bench.py were low)
rm -f /tmp/prof.ncu-rep
timeout 2400 ncu --set full --import-source on --clock-control none -f -o /tmp/prof \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g37_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/g37_ncu_full.md gpurun_out/g37_traffic.json > /dev/null 2> gpurun_out/g37_summary.err
for k in k_delaunay_hull k_gather_emit k_gather_eval k_gather_occl_pt k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof.ncu-rep "$k" 25 > gpurun_out/g37_lines_$k.txt 2>&1
done
cat gpurun_out/g37_traffic.json | head -60
