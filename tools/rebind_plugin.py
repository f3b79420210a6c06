"""pytest plugin: run the reference's own test files with the record path rebound to the
B200 engine.  Loaded with `-p rebind_plugin` before the reference's
test modules import their names, so `from volcache.subdivision import estimate_moments`
inside a test module already receives the device drop-in.

Rebinding (the reference symbol → this package):
  volcache.subdivision.estimate_moments, volcache.renderer.estimate_moments → estimate_moments
  volcache.cache.make_record, volcache.renderer.make_record                → make_record
  volcache.cache.interpolate, volcache.renderer.interpolate               → interpolate
  volcache.renderer.populate_cache                                         → populate_cache
The renderer keeps the reference's own CacheSet, so populate_cache / render / CacheSet.compute
inside the reference renderer all reach the device record build through the rebound names.
Used by tools/run_reference_tests.sh on the GPU box (the reference copy is staged into the
git-ignored baseline/_ref by tools/stage_reference.sh; nothing of it is committed).
"""

from __future__ import annotations

import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import volcache.cache as _vc  # noqa: E402
import volcache.renderer as _vr  # noqa: E402
import volcache.subdivision as _vs  # noqa: E402

import paper_1805_09258_b200 as _b200  # noqa: E402

REBOUND = {
    (_vs, "estimate_moments"): _b200.estimate_moments,
    (_vr, "estimate_moments"): _b200.estimate_moments,
    (_vc, "make_record"): _b200.make_record,
    (_vr, "make_record"): _b200.make_record,
    (_vc, "interpolate"): _b200.interpolate,
    (_vr, "interpolate"): _b200.interpolate,
}
for (mod, name), fn in REBOUND.items():
    if hasattr(mod, name):
        setattr(mod, name, fn)
# results come back as the reference's own Moments dataclass (same fields)
_b200.records.use_result_types(moments=_vs.Moments)


def pytest_report_header(config):
    names = ", ".join(sorted({f"{m.__name__}.{n}" for (m, n) in REBOUND}))
    return f"volcache record path rebound to paper_1805_09258_b200 (libvolcache_b200.so): {names}"
