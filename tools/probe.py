"""Quick GPU timing probe: per-kernel profile of record builds for each config."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_09258_b200 import configs, estimate_moments_batch, seed_words, device_scene, _lib

def run(w, B, reps=2, **kw):
    idx = np.arange(B) % len(w.points)
    X = torch.tensor(w.points[idx], device="cuda")
    S = torch.tensor(seed_words(w.seed, 401, idx).astype(np.int32), device="cuda")
    kw = dict(n_angular=w.n_angular, march_step=w.march_step, n_inner=w.n_inner, epsilon=w.epsilon, **kw)
    r = estimate_moments_batch(w.scene, X, seeds=S, **kw); torch.cuda.synchronize()
    L = _lib.lib(); L.vc_profile(1)
    t = time.perf_counter()
    for _ in range(reps):
        r = estimate_moments_batch(w.scene, X, seeds=S, **kw)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / reps
    ms = np.zeros(12); cnt = np.zeros(12, np.int64)
    L.vc_profile_read(_lib.ptr(ms), _lib.ptr(cnt), 12); L.vc_profile(0)
    st = r.stats.cpu().numpy()
    prof = {k: round(float(m) / reps, 3) for k, m in zip(_lib.KERNEL_CLASSES, ms) if m > 0}
    print(json.dumps({"cfg": w.name, "B": B, "s_per_batch": round(dt, 4), "rec_per_s": round(B / dt, 1),
                      "ms": prof, "mean_P": float(st[:, 3].mean()), "mean_eval": float(st[:, 0].mean()),
                      "tri_fail": int((st[:, 5] != 0).sum())}), flush=True)

print("nproc", os.cpu_count(), len(os.sched_getaffinity(0)), torch.cuda.get_device_name())
run(configs.cfg1(), 256)
run(configs.cfg1(march_step=0.1), 256)
run(configs.cfg2(), 4096, reps=1)
run(configs.cfg2(march_step=0.1), 1024, reps=1)
w3 = configs.cfg3()
device_scene(w3.scene)
run(w3, 64, reps=1)
run(w3, 512, reps=1)
