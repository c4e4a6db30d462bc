"""The reference CPU path under its own benchmark protocol (bench.hpp:63-121):
every design-space kernel (spmm, the 8 KernelIds) plus spmm_reference, fp32, timed with
the reference's time_kernel_fn (warmup 2, reps 7, median) at P = 1 and P = all host cores,
on configs[0] (c1: uniform 4096^2, ~1%, N = 32) and the suite's 2^17-row matrices at
N = 32. Runs the unmodified reference headers through oracle/_ref on the host cores of the
machine it runs on (the GPU box when launched under gpurun); records the CPU model.

python tools/cpu_reference_protocol.py > profiles/r02_cpu_reference.json
"""
import ctypes as C
import json
import os
import platform
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

NAMES = ["RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR", "EB+RM+SR", "EB+RM+PR", "EB+CM+SR",
         "EB+CM+PR"]


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def matrices():
    import torch

    from paper_2202_08556_b200 import gen

    dev = "cpu"
    yield "c1_uniform4096_1pct", gen.uniform(4096, 4096, 167_772, seed=1, device=dev), 32
    for name, mk in gen.suite(device=dev, small=True):
        if "s17" in name:
            yield name, mk(), 32


def main():
    R = O.ref()
    if R is None:
        print(json.dumps({"unavailable": "oracle/_ref not built"}))
        return
    cores = os.cpu_count() or 1
    out = {"protocol": "time_kernel_fn: warmup 2, reps 7, median (bench.hpp:63-121), fp32",
           "cpu_model": cpu_model(), "nproc": cores, "results": []}
    for name, (M, K, rp, ci, va), n in matrices():
        rp = rp.numpy().astype(np.int64)
        h = R.ref_csr_from_csr(M, K, rp, ci.numpy().astype(np.int64), va.numpy().astype(np.float64))
        nnz = int(rp[-1])
        x = np.random.default_rng(n).uniform(-1, 1, (K, n)).astype(np.float32).reshape(-1)
        row = {"matrix": name, "M": M, "nnz": nnz, "N": n, "gflops": {}}
        for P in sorted({1, cores}):
            for k in [-1] + list(range(8)):
                label = "spmm_reference" if k < 0 else NAMES[k]
                if k < 0 and P != 1:
                    continue  # spmm_reference is serial
                med, mn, ck = C.c_double(), C.c_double(), C.c_double()
                rc = R.ref_time_spmm_f32(h, k, P, 8, 8 if k < 0 else (4 if k & 1 else 8), x, n, 7,
                                         2, C.byref(med), C.byref(mn), C.byref(ck))
                if rc:
                    row["gflops"][f"{label}@P{P}"] = None
                    continue
                row["gflops"][f"{label}@P{P}"] = round(2 * nnz * n / med.value / 1e9, 4)
        R.ref_csr_free(h)
        out["results"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
