# round-2 call 4: hash-grid record index (GPU suite, cfg5), traversal stack variants, cfg5 crop fixture
python -m pytest tests -m gpu -x -q > gpurun_out/g4_gputest.log 2>&1; tail -3 gpurun_out/g4_gputest.log
bash tools/variants.sh > gpurun_out/g4_variants.txt 2>&1
VOLCACHE_LEAF_GEO=4 VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/local.so python tools/probe3.py 2048 2>&1 | tail -1 | sed "s/^/local_leaf4 /" >> gpurun_out/g4_variants.txt
cat gpurun_out/g4_variants.txt
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/g4_cfg5.json 2> gpurun_out/g4_cfg5.err
timeout 900 python tools/cfg5_crop_fixture.py > gpurun_out/g4_crop.log 2>&1
