# round-2 call 16: SASS-level hot spots of the triangulation hull kernel and the assembly;
# k_march after the non-reflective specialisation
rm -f /tmp/k.ncu-rep
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_delaunay_hull|k_asm_eval|k_assemble_t" -c 4 -f -o /tmp/k \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g16_ncu.log 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_delaunay_hull --launch-skip 0 --launch-count 1 > gpurun_out/g16_hull_sass.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_asm_eval > gpurun_out/g16_asmeval_sass.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_assemble_t > gpurun_out/g16_asmscan_sass.csv 2>/dev/null
ncu --clock-control none --metrics gpu__time_duration.sum,smsp__sass_inst_executed_op_local_ld.sum,sm__inst_executed.sum -k regex:"k_march|k_primary" --csv \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g16_march.csv 2>/dev/null
