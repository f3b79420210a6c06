"""cfg3 per-kernel timing probe (bench-sized batch)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_09258_b200 import configs, estimate_moments_batch, seed_words, _lib

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = configs.cfg3()
idx = np.arange(B) % len(w.points)
X = torch.tensor(w.points[idx], device="cuda")
S = torch.tensor(seed_words(w.seed, 401, idx).astype(np.int32), device="cuda")
kw = dict(n_angular=w.n_angular, march_step=w.march_step, epsilon=0.05)
r = estimate_moments_batch(w.scene, X, seeds=S, **kw); torch.cuda.synchronize()
L = _lib.lib()
if "noprof" in sys.argv:  # device time of 5 batches without the per-class events
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        r = estimate_moments_batch(w.scene, X, seeds=S, **kw)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"B": B, "noprof_ms": round(e0.elapsed_time(e1) / 5, 3), "rec_per_s": round(5000 * B / e0.elapsed_time(e1), 1)}))
    sys.exit(0)
L.vc_profile(1)
t = time.perf_counter()
r = estimate_moments_batch(w.scene, X, seeds=S, **kw); torch.cuda.synchronize()
dt = time.perf_counter() - t
ms = np.zeros(12); cnt = np.zeros(12, np.int64)
L.vc_profile_read(_lib.ptr(ms), _lib.ptr(cnt), 12)
print(json.dumps({"B": B, "rec_per_s": round(B / dt, 1), "ms": {k: round(float(m), 2) for k, m in zip(_lib.KERNEL_CLASSES, ms) if m > 0},
                  "L_sum": float(r.L.sum()), "tri_fail": int((r.stats[:, 5] != 0).sum())}))
