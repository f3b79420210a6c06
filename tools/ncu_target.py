"""Small cfg3 record build for ncu: one warm-up batch, then one profiled batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_09258_b200 import configs, estimate_moments_batch, seed_words

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
warm = not (len(sys.argv) > 2 and sys.argv[2] == "nowarm")
w = configs.cfg3()
for b in ((32, B) if warm else (B,)):
    idx = np.arange(b)
    X = torch.tensor(w.points[idx], device="cuda")
    S = torch.tensor(seed_words(w.seed, 401, idx).astype(np.int32), device="cuda")
    r = estimate_moments_batch(w.scene, X, seeds=S, n_angular=w.n_angular, march_step=w.march_step, epsilon=0.05)
    torch.cuda.synchronize()
print("ok", float(r.L.sum()))
