"""Triangulation check on the GPU: hull/cap kernels vs the clipping kernel (and qhull) on a few
records of several direction counts; prints the first mismatch.  Usage: del_check.py [n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1805_09258_b200 import configs, inspect_record

def tset(t):
    return {tuple(sorted(map(int, r))) for r in np.asarray(t)}

sc = configs.cfg3_scene(n_spheres=2, level=1)
x = np.array([2.0, 1.5, 2.0])
for n in [int(a) for a in sys.argv[1:]] or [1024, 4096, 16384]:
    for k in range(3):
        seed = np.random.SeedSequence([7, 401, k])
        os.environ.pop("VOLCACHE_DEL_HULL", None)
        try:
            fast = inspect_record(sc, x, rng_seed=seed, n_angular=n, march_step=2.0)
        except Exception as e:
            print("n", n, "rec", k, "hull path error:", e); continue
        os.environ["VOLCACHE_DEL_HULL"] = "0"
        clip = inspect_record(sc, x, rng_seed=seed, n_angular=n, march_step=2.0)
        os.environ.pop("VOLCACHE_DEL_HULL", None)
        a, b = tset(fast["tris"]), tset(clip["tris"])
        print("n", n, "rec", k, "status", fast["stats"][5], "equal", a == b, "only_hull", sorted(a - b)[:4], "only_clip", sorted(b - a)[:4], flush=True)
