# round-2 call 43: hull hand-backs per stratum row (VOLCACHE_DEL_STATS=3) and the per-row window table
VOLCACHE_DEL_STATS=3 python tools/probe3.py 512 2>&1 | grep -v "^{" | head -8
