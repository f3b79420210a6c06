"""Probe the device populate engine on the cfg3 room with a cfg5-style camera.

Usage: python tools/populate_probe.py WIDTH HEIGHT STEP EPS N_ANGULAR [WINDOW]
Prints one JSON line: engine stats + wall seconds.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1805_09258_b200 import configs  # noqa: E402
from paper_1805_09258_b200.renderer import Camera, RenderSettings, populate_cache  # noqa: E402


def main():
    w, h = int(sys.argv[1]), int(sys.argv[2])
    step, eps, n = float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
    window = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    sc = configs.cfg3_scene()
    c = configs.cfg5_camera(w, h)
    cam = Camera(position=c["position"], look_at=c["look_at"], up=c["up"], fov_degrees=c["fov"], width=w, height=h)
    st = RenderSettings(mode="ours-aniso", epsilon=eps, spp=1, march_step=step, n_angular=n, seed=5)
    # warm (scene upload, BVH, emitter quadrature)
    populate_cache(sc, Camera(position=c["position"], look_at=c["look_at"], up=c["up"], fov_degrees=c["fov"],
                              width=4, height=3), st)
    import numpy as np

    from paper_1805_09258_b200 import _lib

    L = _lib.lib()
    L.vc_profile(1)
    t0 = time.perf_counter()
    cs, stats = populate_cache(sc, cam, st, window=window)
    dt = time.perf_counter() - t0
    ms = np.zeros(12)
    cnt = np.zeros(12, np.int64)
    L.vc_profile_read(_lib.ptr(ms), _lib.ptr(cnt), 12)
    L.vc_profile(0)
    stats["kernel_ms"] = {k: round(float(m), 1) for k, m in zip(_lib.KERNEL_CLASSES, ms) if m > 0}
    stats["wall_s"] = dt
    stats["records_per_s"] = stats["builds"] / dt
    stats["config"] = dict(w=w, h=h, step=step, eps=eps, n=n, window=window)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
