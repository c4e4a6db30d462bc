"""In-tree build of the B200 CUDA library (libdaspmm.so) and its C++ test binary.

    python -m paper_2202_08556_b200.build          # incremental
    python -m paper_2202_08556_b200.build --force

Every translation unit is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo so ncu's source page maps
to the kernels. The CUDA runtime is linked statically so the library does not depend
on which libcudart the host process (e.g. torch) loaded first.
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
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libdaspmm.so")
CUSPARSE_LIB = os.path.join(PKG, "libdaspmm_cusparse.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
                 "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]

LIB_SOURCES = ["abi.cu", "features.cu", "select.cu", "graph.cu", "spmm_rb_sr.cu",
               "spmm_rb_pr.cu", "spmm_eb_sr.cu", "spmm_eb_pr.cu", "spmm_lean.cu", "spmm_tma.cu",
               "multi.cu", "spmm_pr_wide.cu", "spmm_tile.cu", "spmm_cm.cu", "coo.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "dispatch.h", "internal.h", "launch_sr.cuh",
           "launch_pr.cuh", "lean.cuh", "tma_gather.cuh", "tile.cuh", "exact_sum.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "daspmm.h")]
    if _mtime(obj) >= max(_mtime(d) for d in deps):
        return obj
    cmd = [NVCC] + CFLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), LIB_SOURCES))
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cusparse(force, verbose)
    return LIB


def build_cusparse(force: bool = False, verbose: bool = False) -> str:
    """The cuSPARSE comparator (bench only; not part of the product library)."""
    src = os.path.join(CSRC, "cusparse_cmp.cu")
    if not os.path.exists(src):
        return ""
    if not force and _mtime(CUSPARSE_LIB) >= _mtime(src):
        return CUSPARSE_LIB
    cmd = [NVCC] + CFLAGS + ["-shared", src, "-o", CUSPARSE_LIB, "-lcusparse", "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cusparse comparator build failed:\n{r.stdout}\n{r.stderr}")
    return CUSPARSE_LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
    sys.exit(0)
