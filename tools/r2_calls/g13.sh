# round-2 call 13: SASS-level hot spots of the gather kernels and k_primary; cfg5 bench repeat
rm -f /tmp/k.ncu-rep
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_gather_emit|k_gather_occl|k_primary" -c 3 -f -o /tmp/k \
  python tools/ncu_target.py 2048 nowarm > gpurun_out/g13_ncu.log 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_gather_emit > gpurun_out/g13_emit_sass.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_gather_occl > gpurun_out/g13_occl_sass.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_primary > gpurun_out/g13_primary_sass.csv 2>/dev/null
ls -la gpurun_out/g13_*
VOLCACHE_POP_TIMING=1 timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g13_cfg5.json 2> gpurun_out/g13_cfg5.err
