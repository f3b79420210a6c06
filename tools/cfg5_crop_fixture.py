"""GPU half of the cfg5 crop fixture (run on the B200 box).

Populates the cfg5 workload (cfg3 room, 1920×1080 camera, march step 0.01, ε from
bench.py) with the device engine, then keeps the records that can touch a 64×36 pixel
crop: every record whose bounding sphere (position, max radius) comes within its radius
of a crop pixel-centre ray segment inside the medium.  That is a superset of the records
covering any crop march point, so lookups over the crop are unchanged.  Writes
gpurun_out/cfg5_crop_records.npz (rows in insertion order, tags, the crop, our crop
image and stats); tests/golden/make_goldens.py gen_cfg5_crop renders the same crop with
the reference from these records.

Usage: python tools/cfg5_crop_fixture.py [ROW0 COL0]
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_1805_09258_b200 import _lib, device_scene  # noqa: E402
from paper_1805_09258_b200.renderer import render_rows, populate_cache  # noqa: E402

CROP_ROWS, CROP_COLS = 36, 64


def crop_rays(cam, r0, c0):
    py, px = np.meshgrid(np.arange(r0, r0 + CROP_ROWS), np.arange(c0, c0 + CROP_COLS), indexing="ij")
    pos = np.asarray(cam.position, float)
    fwd = np.asarray(cam.look_at, float) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, cam.up)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    th = np.tan(np.radians(cam.fov_degrees) / 2)
    u = (px.ravel() + 0.5) / cam.width
    v = (py.ravel() + 0.5) / cam.height
    d = fwd[None] + ((2 * u - 1) * th * cam.width / cam.height)[:, None] * right + ((1 - 2 * v) * th)[:, None] * up
    return pos, d / np.linalg.norm(d, axis=1, keepdims=True)


def near_rays(rows, d, pos, t_max):
    """Records whose sphere (centre, max radius) meets some segment pos + t·d, t ∈ [0, t_max]."""
    dim = 3
    P = rows[:, :dim]
    R = rows[:, -dim:].max(axis=1)
    keep = np.zeros(len(rows), bool)
    for k in range(0, len(d), 64):
        dd = d[k:k + 64]
        w = P - pos[None]
        t = np.clip(w @ dd.T, 0.0, t_max)  # (n, 64)
        foot = pos[None, None] + t[..., None] * dd[None]
        dist = np.linalg.norm(P[:, None] - foot, axis=2)
        keep |= (dist <= R[:, None] * (1 + 1e-9) + 1e-12).any(axis=1)
    return keep


def main():
    r0 = int(sys.argv[1]) if len(sys.argv) > 1 else 522
    c0 = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    sc, cam, st = bench.cfg5_setup()
    cs, pst = populate_cache(sc, cam, st)
    out = {"crop": np.array([r0, CROP_ROWS, c0, CROP_COLS]), "eps": np.array(st.epsilon),
           "step": np.array(st.march_step), "seed": np.array(st.seed),
           "pop_stats": np.array([pst["points_marched"], pst["records_single"], pst["records_multiple"]])}
    pos, d = crop_rays(cam, r0, c0)
    diag = float(np.linalg.norm(np.asarray(sc.bounds_max) - np.asarray(sc.bounds_min)))
    for name, c in (("single", cs.single), ("multiple", cs.multiple)):
        L = _lib.lib()
        n = int(L.vc_cache_size(c._handle))
        rows = np.zeros((n, 27))
        tags = np.zeros(n, np.int64)
        _lib.check(L.vc_cache_records(c._handle, _lib.ptr(rows), _lib.ptr(tags), _lib.VC_MEM_HOST, None))
        keep = near_rays(rows, d, pos, diag)
        out[f"{name}_rows"] = rows[keep]
        out[f"{name}_index"] = np.nonzero(keep)[0]
        print(name, n, "records,", int(keep.sum()), "near the crop", flush=True)
    img, rst = render_rows(sc, cam, st, cs, r0, CROP_ROWS)
    out["gpu_full_cache_crop"] = img[:, c0:c0 + CROP_COLS]
    out["gpu_stats"] = np.array([rst["cache_hits"], rst["direct_evaluations"]])
    dst = ROOT / "gpurun_out" / "cfg5_crop_records.npz"
    dst.parent.mkdir(exist_ok=True)
    np.savez_compressed(dst, **out)
    print("wrote", dst, "hits", rst, flush=True)


if __name__ == "__main__":
    main()
