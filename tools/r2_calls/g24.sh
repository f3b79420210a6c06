# round-2 call 24: per-hit surface radiance entry point (vc_surface_radiance) + reflective room records vs the reference
python -m pytest tests -m gpu -q > gpurun_out/g24_gputest.log 2>&1; tail -3 gpurun_out/g24_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g24_parity_errors.json
