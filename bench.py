"""Benchmark: cache records/sec (radiance + grad + Hessian, 16k dirs/record) on B200.

Workload (BASELINE.json configs[2], parity variant — SURVEY.md §8d): the 4×3×4 window
room with 40 seeded level-3 icospheres (51,300 triangles), σs = 0.27, σa = 0.03,
19,000 cache points (seed 2), n = 16384 stratified directions per record,
march_step 0.1, one gather direction per media sample, records finalised with ε = 0.05.
A step builds `records_per_step` records per rank (points cycle through the config in
order, per-record PCG64 streams SeedSequence([2, 401, i])).

One process per GPU (torchrun for N > 1): ranks take disjoint record shards with no
data-path collective ("weak" scaling); timing is CUDA events on each rank's stream,
max over ranks.  `--impl reference` times the CPU oracle (numpy restatement of the
reference, brute-force trace in C over all host threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cache records/sec (radiance+grad+Hessian, 16k dirs/record); % of FP32 roofline"
UNIT = "records/s"
MEASURED = ROOT / "MEASURED_PEAKS.json"

# Algorithmic flop model: divides/sqrt/exp/atan2 count 1.
F_DIR3, F_REC, F_X3, F_LVL3, F_BOX3, F_ELEM3 = 20, 150, 45, 24, 12, 640
ISSUE_PEAK = 4.0  # warp instructions per cycle per SM (4 SMSPs × 1 issue/cycle)


def f_ray(K: int) -> int:
    lg = int(np.ceil(np.log2(max(K, 2))))
    return min(F_X3 * K, F_X3 + F_LVL3 * lg) + F_BOX3


def peaks():
    pk = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}
    if MEASURED.exists():
        d = json.loads(MEASURED.read_text())
        pk.update(hbm_gbs=float(d.get("hbm_gbs", 6650.0)), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                  source="measured")
    # FP32 vector peak: SMs × 128 lanes × 2 flop × f_max
    pk["fp32_tflops"] = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    return pk


class ClockSampler:
    """NVML SM clock + throttle reasons, sampled during the timed region."""

    def __init__(self, index: int, period: float = 0.1):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # first calls outside the timed region: NVML's lazy set-up inside it stalled the launching
            # thread for ~70 ms in 2 of 10 runs (GPU idle between steps, per-kernel sums unchanged)
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None
        self.period = period

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.wait(self.period):  # samples at period, 2·period, … into the timed region
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, b in names.items():
                    if r & b and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()
        if self.nv is not None and not self.samples:  # a timed region shorter than one period
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def workload(args):
    from paper_1805_09258_b200 import configs

    if args.config == "cfg3":
        w = configs.cfg3()
        B, g = getattr(args, "media_bounces", 1), getattr(args, "hg_g", 0.0)
        if B > 1 or g != 0.0:  # extension: BASELINE cfg3's HG media / multi-bounce media radiance
            import dataclasses

            tag = (f"+hg{g:g}" if g != 0.0 else "") + (f"+{B}-bounce-media" if B > 1 else "")
            w = dataclasses.replace(w, name=f"{w.name}{tag}", media_bounces=B, hg_g=g)
        lights = getattr(args, "lights", "none")
        if lights != "none":  # extension: delta lights (sun = BASELINE cfg3's directional light through
            import dataclasses  # open window cut-outs; lamp = a point light inside the portal room)

            from paper_1805_09258_b200.scene import point_light

            sc = (configs.cfg3_spec_scene() if lights == "sun" else
                  configs.cfg3_scene(lights=[point_light((2.6, 2.2, 1.4), (6.0, 5.0, 4.0))]))
            w = dataclasses.replace(w, name=f"{w.name}+{lights}", scene=sc)
        return w
    if args.config == "cfg2":
        return configs.cfg2(march_step=args.march_step or 4.0)
    if args.config == "cfg1":
        return configs.cfg1(march_step=args.march_step or 4.0)
    if args.config in ("cfg1-spec", "cfg2-spec"):  # extension: the configs as BASELINE.json states them
        import dataclasses

        if args.config == "cfg1-spec":  # point light instead of the emissive square
            w = configs.cfg1(march_step=args.march_step or 0.1)
            return dataclasses.replace(w, name="cfg1-flatland-2d+point-light", scene=configs.cfg1_spec_scene())
        w = configs.cfg2(march_step=args.march_step or 0.1)  # point light, Henyey-Greenstein g = 0.3
        return dataclasses.replace(w, name="cfg2-single-occluder-3d+point-light+hg0.3",
                                   scene=configs.cfg2_spec_scene(), hg_g=0.3)
    if args.config == "cfg4-standin":  # extension stand-in: cfg4's lights and occluders, homogeneous medium
        return configs.cfg4_standin(march_step=args.march_step or 0.1)
    raise SystemExit(f"unknown config {args.config}")


def step_indices(s: int, rank: int, world: int, B: int, N: int):
    start = (s * world + rank) * B
    return (start + np.arange(B)) % N


# ---------------------------------------------------------------------------
# CPU reference arm / baseline
# ---------------------------------------------------------------------------


def cpu_info() -> dict:
    """Host CPU model, the threads used, and the numpy / scipy versions of the CPU arm."""
    import platform

    import scipy

    model = platform.processor() or "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": len(os.sched_getaffinity(0)), "numpy": np.__version__,
            "scipy": scipy.__version__}


def cpu_points(w, n_records: int, start: int = 0):
    """Point indices of a CPU sample: spread evenly over the workload's cache points
    (BASELINE.md §3), offset by `start` so successive samples differ."""
    N = len(w.points)
    stride = max(1, N // max(1, n_records))
    return [(start + k * stride) % N for k in range(n_records)]


def cpu_sample(w, n_records: int, start: int = 0):
    """Oracle records (reference algorithm; brute-force trace over all host threads)."""
    from oracle import volcache_oracle as O

    threads = len(os.sched_getaffinity(0))
    O.use_c_trace(threads)
    ps = O.pack(w.scene)
    t0 = time.perf_counter()
    for i in cpu_points(w, n_records, start):
        rb = O.build_record(ps, w.points[i], w.n_angular, w.march_step, O.seed_seq(w.seed, 401, i), w.n_inner,
                            w.n_light_samples, media_bounces=w.media_bounces, hg_g=w.hg_g)
        for k in range(2):
            O.make_record(w.points[i], rb.L[k], rb.grad[k], rb.hess[k], w.epsilon, ps.scale, ps.max_emission)
    dt = time.perf_counter() - t0
    return dt, threads


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    w = workload(args)
    per = max(1, args.ref_records)
    for s in range(args.warmup):  # warm-up: one record each (page-in, C trace library load)
        cpu_sample(w, 1, start=7919 * s)
    tot = 0.0
    threads = 1
    for s in range(args.steps):  # step s: `per` records spread over the points, offset per step
        dt, threads = cpu_sample(w, per, start=s * 97)
        tot += dt
    value = args.steps * per / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded parity-variant scene, see DESIGN.md)",
        "config": {"workload": w.name, "records_per_step": per, "n_angular": w.n_angular,
                   "march_step": w.march_step, "triangles": len(w.scene.surfaces)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per} record(s) per step of {w.name} spread over its {len(w.points)} points "
                                   f"({args.steps * per} timed): oracle/volcache_oracle.py (numpy restatement) with "
                                   f"the brute-force trace in oracle/trace_c.c on {threads} threads",
                         **cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# cfg5: populate + frozen camera march over ~100k records (the dependent step)
# ---------------------------------------------------------------------------

CFG5_EPS = float(os.environ.get("VOLCACHE_CFG5_EPS", "3e-5"))  # ~96k records at 1920x1080, step 0.01
REC_BYTES_MODEL = 108  # fp32 record: pos 12, value 12, grad 36, axes 36, radii 12


def cfg5_setup(width=1920, height=1080, step=0.01, eps=None):
    from paper_1805_09258_b200 import configs
    from paper_1805_09258_b200.renderer import Camera, RenderSettings

    sc = configs.cfg3_scene()
    c = configs.cfg5_camera(width, height)
    cam = Camera(position=c["position"], look_at=c["look_at"], up=c["up"], fov_degrees=c["fov"], width=width,
                 height=height)
    st = RenderSettings(mode="ours-aniso", epsilon=CFG5_EPS if eps is None else eps, spp=1, march_step=step,
                        n_angular=16384, seed=5, frozen=True)
    return sc, cam, st


def cfg5_march_points(scene, cam, step, rows, cols):
    """Pixel-centre march points of a pixel window (src/renderer.py:290-299), host float64."""
    from paper_1805_09258_b200 import _lib

    r0, nr = rows
    c0, nc = cols
    py, px = np.meshgrid(np.arange(r0, r0 + nr), np.arange(c0, c0 + nc), indexing="ij")
    pos = np.asarray(cam.position, float)
    fwd = np.asarray(cam.look_at, float) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, cam.up)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    th = np.tan(np.radians(cam.fov_degrees) / 2)
    asp = cam.width / cam.height
    u = (px.ravel() + 0.5) / cam.width
    v = (py.ravel() + 0.5) / cam.height
    d = fwd[None] + ((2 * u - 1) * th * asp)[:, None] * right[None] + ((1 - 2 * v) * th)[:, None] * up[None]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.broadcast_to(pos, d.shape).copy()
    ds = __import__("paper_1805_09258_b200").device_scene(scene)
    m = len(d)
    t = np.zeros(m)
    idx = np.zeros(m, np.int32)
    _lib.check(_lib.lib().vc_trace(ds.handle, m, _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), _lib.ptr(idx),
                                   _lib.VC_MEM_HOST, None))
    bmin, bmax = np.asarray(scene.bounds_min, float), np.asarray(scene.bounds_max, float)
    with np.errstate(divide="ignore", invalid="ignore"):
        t1, t2 = (bmin - o) / d, (bmax - o) / d
    t_in = np.maximum(np.nanmax(np.minimum(t1, t2), axis=1), 0.0)
    t_out = np.nanmin(np.maximum(t1, t2), axis=1)
    t_end = np.minimum(t, t_out)
    n = np.maximum(np.floor((t_end - t_in) / step + 0.5), 0).astype(int)
    pts = [o[i] + (t_in[i] + (np.arange(1, n[i] + 1) - 0.5) * step)[:, None] * d[i] for i in range(m)]
    return np.concatenate(pts) if pts else np.zeros((0, 3)), int(n.sum())


def run_cfg5(args):
    import torch

    from paper_1805_09258_b200 import _lib, device_scene
    from paper_1805_09258_b200.renderer import _render_params, populate_cache

    rank, world, local = dist_env()
    if world > 1:
        raise SystemExit("cfg5 bench runs one GPU (multi-GPU populate: dist.populate_sharded)")
    torch.cuda.set_device(local)
    sc, cam, st = cfg5_setup(eps=args.cfg5_eps)
    ds = device_scene(sc)
    L = _lib.lib()
    # warm the scene (BVH, emitter quadrature) with a tiny populate
    from paper_1805_09258_b200.renderer import Camera

    small = Camera(position=cam.position, look_at=cam.look_at, up=cam.up, fov_degrees=cam.fov_degrees, width=8,
                   height=5)
    populate_cache(sc, small, st)
    torch.cuda.synchronize()
    launches0 = L.vc_kernel_launches()
    with ClockSampler(local) as clk_pop:
        t0 = time.perf_counter()
        cs, pst = populate_cache(sc, cam, st)
        torch.cuda.synchronize()
        pop_s = time.perf_counter() - t0
    pop_launches = L.vc_kernel_launches() - launches0
    n_rec = pst["records"]
    # frozen march: device image, inputs (caches, scene) resident
    cam_c = cam._c()
    rp = _render_params(sc, st)
    hs, hm = cs._handles()
    img = torch.zeros((cam.height, cam.width, 3), dtype=torch.float64, device="cuda")
    out = np.zeros(2, np.int64)

    def march(host_img=None):
        ptr = _lib.ptr(host_img) if host_img is not None else _lib.C.c_void_p(img.data_ptr())
        _lib.check(L.vc_render(ds.handle, hs, hm, _lib.C.byref(cam_c), _lib.C.byref(rp), ptr, _lib.ptr(out),
                               _lib.VC_MEM_HOST if host_img is not None else 0, None))

    for _ in range(args.warmup):
        march()
    torch.cuda.synchronize()
    L.vc_profile(1)
    launches0 = L.vc_kernel_launches()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            march()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = L.vc_kernel_launches() - launches0
    kms = np.zeros(12)
    kcnt = np.zeros(12, np.int64)
    L.vc_profile_read(_lib.ptr(kms), _lib.ptr(kcnt), 12)
    L.vc_profile(0)
    hits, misses = int(out[0]), int(out[1])
    steps_total = hits + misses  # march points per frame
    value = steps_total * args.steps / (ms / 1e3)
    # e2e: the public render() call with a host image (D2H of the frame inside the timed region)
    from paper_1805_09258_b200.renderer import render

    t0 = time.perf_counter()
    e2e_n = max(1, args.e2e_steps if args.e2e_steps is not None else 3)  # cfg5: whole frames
    for _ in range(e2e_n):
        image_h, rst = render(sc, cam, st, cache_set=cs)
    e2e_s = (time.perf_counter() - t0) / e2e_n
    # covering records per lookup (single, multiple) on a sample of march points
    sample, _ = cfg5_march_points(sc, cam, st.march_step, (0, cam.height), (0, cam.width)) \
        if args.cfg5_full_sample else cfg5_march_points(sc, cam, st.march_step, (cam.height // 2 - 30, 60),
                                                        (0, cam.width))
    cov = []
    for c in (cs.single, cs.multiple):
        _, cnt = c.interpolate_many(sample)
        cov.append(float(cnt.mean()))
    names = _lib.KERNEL_CLASSES
    march_ms = float(kms[names.index("march")])
    n_march = int(kcnt[names.index("march")])
    # algorithmic bytes per march point: single lookup (12 + Σcov·108 + 12) and, where covered,
    # the multiple lookup; every point of the populated frame is covered by both caches
    bpp = (24 + cov[0] * REC_BYTES_MODEL) + (24 + cov[1] * REC_BYTES_MODEL)
    pk = peaks()
    achieved = bpp * steps_total * args.steps / (march_ms / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("per_class", {}).get("march")
        except Exception:
            traffic = None
    line = {
        "metric": "cfg5 frozen camera-march lookups/s (1920x1080, step 0.01, ~100k records)",
        "value": value, "unit": "lookups/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded cfg3 room, cfg5 camera; no public dataset)",
        "config": {"workload": "cfg5-camera-1920x1080", "width": cam.width, "height": cam.height,
                   "march_step": st.march_step, "epsilon": st.epsilon, "n_angular": 16384, "spp": 1,
                   "records": n_rec, "records_single": pst["records_single"],
                   "records_multiple": pst["records_multiple"], "march_points_per_frame": steps_total,
                   "direct_evaluations_per_frame": misses,
                   "pixel_steps_per_s": value, "mean_covering_single": cov[0], "mean_covering_multiple": cov[1],
                   "l2": "no flush: the frame's record working set (2 caches) is L2-sized by design; "
                         "the roofline below is against HBM",
                   "populate": {"seconds": pop_s, "points_marched": pst["points_marched"],
                                "records_per_s": n_rec / pop_s, "builds": pst["builds"],
                                "builds_per_s": pst["builds"] / pop_s, "windows": pst["windows"],
                                "discarded_builds": pst["discarded_builds"], "kernel_launches": int(pop_launches),
                                "clocks": clk_pop.summary()}},
        "roofline": {"bound": "hbm", "kernel": "march", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                     "bytes_per_march_point": bpp, "march_ms_per_frame": march_ms / max(args.steps, 1),
                     "march_launches": n_march},
        "e2e": {"value": steps_total / e2e_s, "unit": "lookups/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": cam.width * cam.height * 24},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--march-step", type=float, default=None)
    ap.add_argument("--records-per-step", type=int, default=2048)
    ap.add_argument("--cpu-records", type=int, default=4, help="oracle records in the cpu_baseline sample")
    ap.add_argument("--ref-records", type=int, default=4, help="--impl reference: oracle records per timed step")
    ap.add_argument("--media-bounces", type=int, default=1,
                    help="cfg3 extension: media events per gather path (1 = the reference's estimator)")
    ap.add_argument("--hg-g", type=float, default=0.0,
                    help="cfg3 extension: Henyey-Greenstein g of the media scattering events (0 = the reference)")
    ap.add_argument("--lights", default="none", choices=["none", "sun", "lamp"],
                    help="cfg3 extension: delta lights (sun: open windows + directional light; lamp: point light)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None, help="e2e timed steps (default: --steps)")
    ap.add_argument("--cfg5-eps", type=float, default=None, help="cfg5: record-error target ε (default tuned)")
    ap.add_argument("--cfg5-full-sample", action="store_true", help="cfg5: covering counts over the whole frame")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg5":
        return run_cfg5(args)

    import torch
    import torch.distributed as dist

    from paper_1805_09258_b200 import _lib, check_deferred, device_scene, estimate_moments_batch, seed_words
    from paper_1805_09258_b200.records import moment_size, record_size

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args)
    N = len(w.points)
    B = args.records_per_step
    ds = device_scene(w.scene)
    kw = dict(n_angular=w.n_angular, march_step=w.march_step, n_inner=w.n_inner,
              n_light_samples=w.n_light_samples, epsilon=w.epsilon, media_bounces=w.media_bounces,
              hg_g=w.hg_g)
    total_steps = args.warmup + args.steps
    # inputs resident in HBM before timing
    Xs, Ss = [], []
    for s in range(total_steps):
        idx = step_indices(s, rank, world, B, N)
        Xs.append(torch.tensor(w.points[idx], device="cuda"))
        Ss.append(torch.tensor(seed_words(w.seed, 401, idx).astype(np.int32), device="cuda"))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    res = None
    for s in range(args.warmup):
        res = estimate_moments_batch(w.scene, Xs[s], seeds=Ss[s], **kw)
    gathered = None
    if world > 1:  # fixed-size record all-gather over NCCL, warmed once
        gathered = torch.empty(world * res.records.numel(), dtype=res.records.dtype, device="cuda")
        dist.all_gather_into_tensor(gathered, res.records.reshape(-1))
    torch.cuda.synchronize()
    L = _lib.lib()
    L.vc_profile(1)
    launches0 = L.vc_kernel_launches()
    stats_acc = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        step_ev = []
        for s in range(args.warmup, total_steps):
            # device-resident steps queue back to back: the bounds check of every step is read once,
            # after the region (check_deferred below), instead of one host wait per step
            res = estimate_moments_batch(w.scene, Xs[s], seeds=Ss[s], defer_check=True, **kw)
            stats_acc.append(res.stats)
            if os.environ.get("BENCH_STEP_EVENTS"):  # debug: where inside the region the time goes
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                step_ev.append((e, time.perf_counter()))
            if world > 1:  # the exchange before a lookup pass: every rank gets every record
                dist.all_gather_into_tensor(gathered, res.records.reshape(-1))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    check_deferred()  # raises if any timed step saw a point outside the bounds
    launches = L.vc_kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if step_ev:
        print("step end (ms, device | host):", [(round(ev0.elapsed_time(e), 2), round((t - step_ev[0][1]) * 1e3, 2))
                                               for e, t in step_ev], file=sys.stderr)
    kms = np.zeros(12)
    kcnt = np.zeros(12, np.int64)
    L.vc_profile_read(_lib.ptr(kms), _lib.ptr(kcnt), 12)
    L.vc_profile(0)
    st = torch.cat(stats_acc).cpu().numpy()
    tri_fail = int((st[:, 5] != 0).sum())
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    records = B * args.steps * world
    value = records / (ms_max / 1e3)

    # ---- e2e: public API with pinned host buffers, H2D + D2H inside the timed region ----
    e2e_steps = max(1, args.e2e_steps if args.e2e_steps is not None else args.steps)
    Xh = [torch.tensor(w.points[step_indices(s, rank, world, B, N)]).pin_memory().numpy() for s in range(e2e_steps)]
    Sh = [torch.tensor(seed_words(w.seed, 401, step_indices(s, rank, world, B, N)).astype(np.int32))
          .pin_memory().numpy().view(np.uint32) for s in range(e2e_steps)]
    d = ds.dim
    MS, RS = moment_size(d), record_size(d)
    mom_h = torch.empty((B, 2, MS), dtype=torch.float64).pin_memory().numpy()
    rec_h = torch.empty((B, 2, RS), dtype=torch.float64).pin_memory().numpy()
    st_h = torch.empty((B, 8), dtype=torch.int64).pin_memory().numpy()
    prm = _lib.BuildParams()
    prm.n_angular, prm.march_step, prm.n_inner = w.n_angular, w.march_step, w.n_inner
    prm.n_light_samples, prm.epsilon = w.n_light_samples, w.epsilon
    prm.flags = _lib.VC_MEM_HOST | _lib.VC_SEED_WORDS | _lib.VC_MAKE_RECORDS
    prm.media_bounces = w.media_bounces
    prm.hg_g = w.hg_g
    prm.seed_words = 3
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(e2e_steps):
        _lib.check(L.vc_build_records(ds.handle, B, _lib.ptr(Xh[s]), _lib.ptr(Sh[s]), None, _lib.C.byref(prm),
                                      _lib.ptr(mom_h), _lib.ptr(st_h), _lib.ptr(rec_h), None))
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = B * e2e_steps * world / e2e_s
    h2d = B * (d * 8 + 3 * 4)
    d2h = B * (2 * MS * 8 + 8 * 8 + 2 * RS * 8)

    # ---- roofline of the dominant kernel (CUDA events on the launching stream) ----
    pk = peaks()
    K = len(w.scene.surfaces)
    n = w.n_angular
    P_sum = float(st[:, 3].sum())
    E_sum = float(st[:, 0].sum())
    nrec = float(len(st))
    work = {  # algorithmic flops over the timed region, per kernel class
        "gather": P_sum * (6 + w.n_inner * (f_ray(K) + 10)),
        "primary": nrec * n * (F_DIR3 + f_ray(K)),
        "assemble": E_sum * F_ELEM3,
        "make_record": nrec * 2 * F_REC,
    }  # SURVEY.md §8d's W; the triangulation has no flop term there — it is rated on issue below
    names = _lib.KERNEL_CLASSES
    shares = {names[i]: float(kms[i]) for i in range(12) if kcnt[i] > 0}
    # the roofline's kernel is the largest class SURVEY §8d's W has a term for; the triangulation
    # (no flop term in W, ~equal in time to the gather) is rated on its issue rate in per_kernel
    # and named in "largest_by_time" when it leads
    top = max(shares, key=shares.get)
    dom = max((k for k in shares if k in work), key=shares.get)
    dom_i = names.index(dom)
    launches_dom = int(kcnt[dom_i])
    avg_ms = float(kms[dom_i]) / max(launches_dom, 1)
    flops_per_launch = work.get(dom, 0.0) / max(launches_dom, 1)
    achieved = flops_per_launch / (avg_ms / 1e3) / 1e12
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            traffic = tj.get("per_class", tj).get(dom)
        except Exception:
            traffic = None
    # every modelled kernel's fraction, and the whole path: W per record over the step time
    per_kernel = {}
    for k, w_k in work.items():
        if k in shares and shares[k] > 0:
            a = w_k / (shares[k] / 1e3) / 1e12
            per_kernel[k] = {"achieved_tflops": a, "frac": a / pk["fp32_tflops"], "ms": shares[k]}
    # issue-rate bound per kernel class: warp instructions of one 2048-record wave (ncu capture,
    # profiles/ncu_traffic.json "inst_per_class") scaled to the records timed here, over the
    # live CUDA-event time → achieved warp instructions per SM-cycle, against 4
    inst_model = {}
    if tf.exists():
        try:
            inst_model = json.loads(tf.read_text()).get("inst_per_class", {})
        except Exception:
            inst_model = {}
    f_sm = (clk.summary().get("sm_mhz") or pk["sm_max_mhz"]) * 1e6
    for k, inst in inst_model.items():
        if k in shares and shares[k] > 0:
            ipc = inst * (nrec / 2048.0) / (shares[k] / 1e3) / (148 * f_sm)
            per_kernel.setdefault(k, {"ms": shares[k]})
            per_kernel[k]["issue_ipc_per_sm"] = ipc
            per_kernel[k]["issue_frac"] = ipc / ISSUE_PEAK
    w_path = sum(work.values())
    path_achieved = w_path / (ms / 1e3) / 1e12
    roofline = {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": pk["fp32_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["fp32_tflops"], "traffic": traffic,
                "peak_source": f"148 SMs x 128 FP32 lanes x 2 x sm_max_mhz ({pk['source']} clocks)",
                "kernel_ms_share": {k: round(v / sum(shares.values()), 4) for k, v in shares.items()},
                "algorithmic_flops_per_launch": flops_per_launch,
                "largest_by_time": {"kernel": top, "ms": shares[top],
                                    "issue_frac": per_kernel.get(top, {}).get("issue_frac")},
                "per_kernel": per_kernel,
                "path": {"algorithmic_flops_per_record": w_path / nrec, "achieved": path_achieved,
                         "frac": path_achieved / pk["fp32_tflops"]}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded parity-variant scene; no public dataset)",
        "config": {"workload": w.name, "records_per_step": B * world, "records_per_rank_step": B,
                   "n_angular": n, "march_step": w.march_step, "n_inner": w.n_inner, "epsilon": w.epsilon,
                   "triangles": K, "cache_points": N, "parallelism": f"records sharded over {world} GPU(s)",
                   "exchange": ("per step, every rank's records all-gathered over NCCL inside the timed region "
                                f"({world * B * 2 * record_size(ds.dim) * 8} bytes gathered per step)")
                   if world > 1 else "none (1 GPU)",
                   "l2": "no flush: per-step scratch (media samples, directions) is GBs, far above the 126 MB L2",
                   "samples_per_s": value * n, "mean_media_samples_per_record": P_sum / nrec,
                   "mean_elements_evaluated": E_sum / nrec, "triangulation_failures": tri_fail},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
                "d2h_bytes_per_step": d2h * world},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nc = max(1, args.cpu_records)
        dt, threads = cpu_sample(w, nc)
        line["cpu_baseline"] = {
            "value": nc / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{nc} record(s) of {w.name} spread over its {len(w.points)} points, through "
                      f"oracle/volcache_oracle.py (numpy restatement of the reference) with the brute-force trace "
                      f"in oracle/trace_c.c on {threads} host threads ({dt:.1f} s)",
            **cpu_info(),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
