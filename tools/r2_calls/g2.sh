# round-2 call 2: bench after the async bounds check; cfg5 march ncu (launch list + full capture of k_march)
python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_march|k_interp" --csv \
  --log-file gpurun_out/g2_cfg5_launches.csv python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 \
  > gpurun_out/g2_cfg5_ncu_launch.log 2>&1
rm -f /tmp/march.ncu-rep
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_march -c 1 -f -o /tmp/march \
  python bench.py --config cfg5 --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/g2_cfg5_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/march.ncu-rep gpurun_out/g2_march_summary.md gpurun_out/g2_march_traffic.json \
  > /dev/null 2> gpurun_out/g2_summary.err
python tools/ncu_lines.py /tmp/march.ncu-rep k_march 40 > gpurun_out/g2_lines_k_march.txt 2>&1
ncu -i /tmp/march.ncu-rep --page raw --csv > gpurun_out/g2_march_raw.csv 2>/dev/null
