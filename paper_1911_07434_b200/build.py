"""In-tree build of libfastmusic_b200.so (sm_100a) with nvcc.

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` into ``build/`` and linked
into ``paper_1911_07434_b200/libfastmusic_b200.so`` (git-ignored, travels to the GPU
box with the gpurun snapshot). Objects are rebuilt only when a source or header is
newer. Usage: ``python -m paper_1911_07434_b200.build [--force]``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "fastmusic_b200")
LIB = os.path.join(PKG, "libfastmusic_b200.so")
CU_SOURCES = ["cov_tc.cu", "rmul_tc.cu", "subspace.cu", "smallmat.cu", "final_fallback.cu", "spectrum.cu", "spectrum_tc.cu", "exact.cu", "jacobi.cu",
              "lanczos.cu", "lanczos_batch.cu", "general.cu", "capi.cu"]
CXX_SOURCES = ["facade.cpp", "io.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
EXTRA = os.environ.get("FM_NVCC_FLAGS", "").split()  # experiment switches, e.g. -DFM_COV_MAXNREG=72


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    inc = os.path.join(ROOT, "include")
    for dp, _, fs in os.walk(inc):
        hs += [os.path.join(dp, f) for f in fs if f.endswith((".h", ".hpp"))]
    return hs


def _stale(obj, src, headers):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + headers)


def _compile(src, force, headers):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and not _stale(obj, src, headers):
        return obj, None
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + COMMON + EXTRA + ["-lineinfo", "-Xptxas", "-v", "-c", src, "-o", obj]
    else:
        cmd = [NVCC, "-x", "cu"] + ARCH + COMMON + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = _headers()
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CXX_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, headers), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, srcs):
            if log:
                print(f"== {os.path.basename(s)}\n{log}", file=sys.stderr)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
