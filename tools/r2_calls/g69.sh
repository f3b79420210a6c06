# round-2 call 69: the reference's own test files with the record path rebound to the device, at the
# final HEAD (baseline/_ref staged by tools/stage_reference.sh; not committed)
bash tools/run_reference_tests.sh
cp gpurun_out/ref_tests_rebound.log gpurun_out/g69_ref_tests_rebound.log
