# round-2 call 46: hull scan with a packed add (u - a as add.f32x2) and unroll factors
bash tools/variants.sh
VOLCACHE_B200_LIB=paper_1805_09258_b200/lib/variants/add2.so python -m pytest tests -m gpu -q -x -k "delaunay or triangulation or hull or qhull or full_size" 2>&1 | tail -2
