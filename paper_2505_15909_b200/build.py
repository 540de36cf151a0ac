"""Build librtnq_b200.so in-tree (sm_100a), with nvcc + g++ only.

    python -m paper_2505_15909_b200.build          # incremental
    python -m paper_2505_15909_b200.build --clean

The library holds the CUDA kernels (csrc/kernels), the extern "C" boundary
(csrc/capi, declared in include/rtnq_capi.h) and the drop-in C++ API
(csrc/dropin, declared in include/rtnq/*.hpp).  It is the only artefact the
product needs; it lands next to this file so gpurun snapshots carry it.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "librtnq_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
          "-I", CSRC]
CUFLAGS = ARCH + COMMON + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
# RTNQ_KERNEL_DEBUG=1 compiles in the int8 kernels' profiling knobs (RTNQ_WGEMM_DEBUG bits used
# by scratch/i4prof.py, i8tl.py, ...); off by default because the checks cost a few % per launch
if os.environ.get("RTNQ_KERNEL_DEBUG"):
    CUFLAGS = CUFLAGS + ["-DRTNQ_KERNEL_DEBUG"]
# experiments only (A/B builds into another library, scratch/*): extra -D flags
CUFLAGS = CUFLAGS + os.environ.get("RTNQ_EXTRA_CUFLAGS", "").split()


def sources():
    out = []
    for sub in ("kernels", "capi", "dropin"):
        d = os.path.join(CSRC, sub)
        if not os.path.isdir(d):
            continue
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(d, f))
    return out


def headers():
    hs = []
    for base in (CSRC, os.path.join(ROOT, "include")):
        for dp, _, fs in os.walk(base):
            hs += [os.path.join(dp, f) for f in fs if f.endswith((".cuh", ".h", ".hpp"))]
    return hs


def _compile(src, verbose):
    obj = os.path.join(OBJ, os.path.relpath(src, CSRC).replace(os.sep, "__") + ".o")
    newest_hdr = max((os.path.getmtime(h) for h in headers()), default=0)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), newest_hdr):
        return obj, ""
    flags = CUFLAGS if src.endswith(".cu") else ARCH + COMMON
    cmd = [NVCC, *flags, "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return obj, (p.stderr if verbose else "")


def build(verbose=False, clean=False):
    if clean and os.path.isdir(OBJ):
        shutil.rmtree(OBJ)
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            sys.stderr.write(log)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart",
               "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, clean=a.clean))
