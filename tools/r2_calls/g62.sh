# round-2 call 62: non-reflective scenes read the surface radiance as emission[idx] (no lo array written or
# read) — GPU suite, bench, DRAM bytes of primary / rings / assembly
python -m pytest tests -m gpu -q > gpurun_out/g62_gputest.log 2>&1; tail -2 gpurun_out/g62_gputest.log
for i in 1 2; do python bench.py --no-cpu-baseline > gpurun_out/g62_bench.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/g62_bench.json')); print('bench', round(d['value'],1), round(d['ms_per_step'],3), {k:round(v['ms'],1) for k,v in d['roofline']['per_kernel'].items()})"; done
ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_primary|k_rings|k_assemble_t|k_asm_eval" --csv python tools/ncu_target.py 2048 nowarm 2>/dev/null | grep -E "k_primary|k_rings|k_assemble_t|k_asm_eval" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -16
