"""Build libmact_cuda.so in-tree with nvcc for sm_100a.

    python -m paper_1009_0854_b200.build [--force] [--verbose]

Every ``csrc/*.cu`` is compiled to an object under ``build/`` and linked into
``paper_1009_0854_b200/libmact_cuda.so`` (static cudart, so the library only
needs the driver at run time).  Objects are rebuilt when a source or any
header under ``csrc/`` or ``include/`` is newer.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# Tuning builds: MACT_NVCC_DEFS="-DMACT_LAB_TP=2048 ..." MACT_LIB_TAG=v2 writes
# libmact_cuda_v2.so (objects under build/mact_v2) without touching the default.
_TAG = os.environ.get("MACT_LIB_TAG", "")
BUILD = ROOT / "build" / ("mact" + (f"_{_TAG}" if _TAG else ""))
LIB = PKG / ("libmact_cuda" + (f"_{_TAG}" if _TAG else "") + ".so")
EXTRA = os.environ.get("MACT_NVCC_DEFS", "").split()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + ARCH


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libmact_cuda.so")


def _newest_header() -> float:
    heads = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in heads), default=0.0)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    hdr = _newest_header()
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = []
    for src in srcs:
        obj = BUILD / (src.stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [cc, *NVCC_FLAGS, *EXTRA, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
        return src.name, r.stderr

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        for name, err in pool.map(compile_one, jobs):
            if verbose and err:
                print(f"--- {name}\n{err}", file=sys.stderr)
    objs = [BUILD / (s.stem + ".o") for s in srcs]
    if force or jobs or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
