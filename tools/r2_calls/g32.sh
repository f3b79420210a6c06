# round-2 call 32: compute-sanitizer memcheck over the small parity cases (new delta-light kernels,
# 2D/3D goldens, populate, lookups)
export PYTHONDONTWRITEBYTECODE=1
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_elements.py -m gpu -q -x \
  -k "delta or pen2d or cfg1 or refl2d or box3d or make_record or formfactor or interpolate or media_hg or media_bounces" \
  > gpurun_out/g32_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -15 gpurun_out/g32_memcheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g32_memcheck_smoke.log 2>&1
echo "smoke memcheck rc=$?"; tail -5 gpurun_out/g32_memcheck_smoke.log
