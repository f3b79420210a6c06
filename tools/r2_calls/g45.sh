# round-2 call 45: gift wrap with two independent running bests (VC_WRAP_CHAINS=2) vs the single chain —
# triangulation tests, then the per-class probe for both
python -m pytest tests -m gpu -q -x -k "delaunay or triangulation or hull or qhull or full_size" 2>&1 | tail -3
bash tools/variants.sh
VOLCACHE_DEL_STATS=1 python tools/probe3.py 512 2>&1 | grep fallback | head -2
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/chains1.so VOLCACHE_DEL_STATS=1 python tools/probe3.py 512 2>&1 | grep fallback | head -2
