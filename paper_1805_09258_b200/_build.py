"""Build libvolcache_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The shared library is the C-ABI boundary (include/volcache_b200.h); it is placed at
paper_1805_09258_b200/lib/libvolcache_b200.so so it travels with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libvolcache_b200.so"
OBJ = PKG / "build"

CU_SOURCES = ["vc_api.cu", "vc_build.cu", "vc_cache.cu", "vc_populate.cu", "vc_baseline.cu", "vc_path.cu",
              "vc_elements.cu"]
CPP_SOURCES = ["vc_bvh.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + ARCH


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build libvolcache_b200.so")
    return cand


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*")) + [PKG.parent / "include" / "volcache_b200.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile the library; `out`/`defines` build an experiment variant (e.g. -DVC_LB_TRACE=2)."""
    lib = Path(out) if out else LIB
    if not force and out is None and up_to_date():
        return LIB
    obj = OBJ if out is None else OBJ / lib.stem
    obj.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    cuda_inc = str(Path(nvcc).resolve().parent.parent / "include")
    jobs = []
    for s in CU_SOURCES:
        jobs.append([nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / s), "-o", str(obj / (s + ".o"))])
    for s in CPP_SOURCES:
        jobs.append(["g++", "-O3", "-std=c++17", "-fPIC", "-I", cuda_inc, "-c", str(CSRC / s),
                     "-o", str(obj / (s + ".o"))])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = obj / (Path(cmd[-1]).name + ".log")
        log.write_text(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        return r

    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    objs = [str(obj / (s + ".o")) for s in CU_SOURCES + CPP_SOURCES]
    tmp = lib.with_suffix(".so.tmp")
    link = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
