# round-2 call 36: HG in the two-pass gather, dark-scene gather skip, persistent-lane delta-light
# shadow rays — GPU suite, default bench (regression check), lit / HG variants, A/B vs the grid kernel
python -m pytest tests -m gpu -q -x > gpurun_out/g36_gputest.log 2>&1; tail -3 gpurun_out/g36_gputest.log
cp gpurun_out/parity_errors.json gpurun_out/g36_parity_errors.json
run() { tag=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/g36_bench_$tag.json 2> gpurun_out/g36_bench_$tag.err; python -c "import json; d=json.load(open('gpurun_out/g36_bench_$tag.json')); print('$tag', round(d['value'],1), round(d['ms_per_step'],2))"; }
run default
run lamp --lights lamp --steps 3
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/delta_grid.so run lamp_grid --lights lamp --steps 3
run hg1 --hg-g 0.5 --steps 5
run spec --lights sun --hg-g 0.5 --media-bounces 4 --steps 3 --records-per-step 512
run sun --lights sun --steps 3
run cfg1spec --config cfg1-spec
run cfg2spec --config cfg2-spec
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/delta_grid.so run cfg2spec_grid --config cfg2-spec
