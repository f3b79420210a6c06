#!/bin/bash
# Round-end measurement set (GPU box): bench line, reference arm, ncu launch list, ncu full
# capture of one 2048-record wave summarised on the box (the report itself stays in /tmp:
# gpurun_out/ must stay under 64 MiB).
set -x
if [ "$1" != "ncu-only" ]; then
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
fi
python tools/ncu_target.py 2048 nowarm > gpurun_out/nt.log 2>&1 && \
rm -f /tmp/prof_round.ncu-rep && timeout 2400 ncu --set full --import-source on --clock-control none -f \
  -o /tmp/prof_round python tools/ncu_target.py 2048 nowarm > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_round.ncu-rep gpurun_out/ncu_full_summary.md gpurun_out/ncu_traffic.json \
  > /dev/null 2> gpurun_out/ncu_summary.err
for k in k_delaunay_hull k_delaunay_capg k_delaunay_warp k_gather_emit k_gather_occl k_primary k_assemble_t k_asm_eval; do
  python tools/ncu_lines.py /tmp/prof_round.ncu-rep "$k" 25 > gpurun_out/lines_$k.txt 2>&1
done
tail -3 gpurun_out/ncu_full.log
