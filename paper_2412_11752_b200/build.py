"""Builds the CUDA extension in-tree: paper_2412_11752_b200/libdrk_b200.so.

Every translation unit: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
drk_prep.cu / drk_sort.cu / drk_capi.cu use --fmad=false (their fp64 binning
decisions must round like the reference's x86-64 build); drk_raster.cu uses
--fmad=true for its fp32 fast path and rounds its exact fp64 values explicitly
(__dmul_rn / __dadd_rn).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
SOURCES = {"drk_prep.cu": False, "drk_sort.cu": False, "drk_raster.cu": True, "drk_raster_fast.cu": True, "drk_raster_bwd.cu": True,
           "drk_capi.cu": False, "drk_scene.cu": False, "drk_loss.cu": False, "drk_train.cu": False, "drk_mesh.cu": False, "drk_det.cu": False,
           "drk_comm.cu": False}
LIB = os.path.join(HERE, "libdrk_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _deps():
    d = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    return d + [os.path.join(ROOT, "include", "drk_b200.h"), os.path.abspath(__file__)]


def build(verbose: bool = False, extra=None, jobs: int = 4) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = _deps()
    newest_dep = max(os.path.getmtime(d) for d in deps)
    procs, objs = [], []
    for src, fmad in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if not extra and os.path.exists(o) and os.path.getmtime(o) >= max(newest_dep, os.path.getmtime(s)):
            continue
        cmd = [NVCC, *COMMON, f"--fmad={'true' if fmad else 'false'}", *(extra or []), "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), src))
        if len(procs) >= jobs:
            p, name = procs.pop(0)
            if p.wait() != 0:
                raise RuntimeError(f"nvcc failed on {name}")
    for p, name in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {name}")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, extra=sys.argv[1:] or None))
