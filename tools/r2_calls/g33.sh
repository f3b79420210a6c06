# round-2 call 33: hull window margin (VOLCACHE_HULL_ALPHA, mean spacings; default 2) — Delaunay class time
# and hand-back counts per margin
for a in 2.0 1.75 1.5 1.25 2.5; do
  echo "alpha $a"
  VOLCACHE_HULL_ALPHA=$a VOLCACHE_DEL_STATS=1 python tools/probe3.py 2048 2>&1 | grep -E "fallback|rec_per_s" | tail -3
  VOLCACHE_HULL_ALPHA=$a python tools/probe3.py 2048 2>&1 | tail -1
done
