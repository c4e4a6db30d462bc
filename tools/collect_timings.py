"""Collect B200 timings of all eight kernels over a synthetic corpus.

Each sample = (matrix, N): features from the device feature extractor (bit-identical
to extract_features, features.hpp:21-41) and the median device time of each of the
8 kernels (fast mode, make_config defaults W = 8). Output CSV columns follow the
reference's dataset record (dataset.hpp:89-153): matrix_id, nnz, mat_size, std_row,
n_cols, t0..t7, label.

python tools/collect_timings.py --out gpurun_out/timings.csv [--quick]
"""
import argparse
import csv
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402


def corpus(quick: bool):
    rng = np.random.default_rng(2202)
    specs = []
    scales = range(10, 21) if not quick else (10, 14, 17)
    for s in scales:
        for deg in (2, 8, 16, 32) if not quick else (8,):
            if (1 << s) * deg > 40_000_000:
                continue
            specs.append(("uniform", s, deg, None))
            for a in (0.45, 0.57, 0.7):
                specs.append(("rmat", s, deg, a))
        if not quick and s in (12, 14, 16, 17, 18, 20):
            specs.append(("banded", s, 4, None))
            specs.append(("banded", s, 8, None))
            specs.append(("banded", s, 32, None))
        if not quick and s in (11, 12, 13, 14):  # small, denser matrices (c1-like: 4096^2, 1%)
            for deg in (40, 128):
                specs.append(("uniform", s, deg, None))
                specs.append(("rmat", s, deg, 0.45))
    for kind, s, deg, a in specs:
        seed = int(rng.integers(1 << 30))
        n = 1 << s
        name = f"{kind}_s{s}_d{deg}" + (f"_a{a}" if a else "")
        if kind == "uniform":
            yield name, (lambda n=n, deg=deg, seed=seed: gen.uniform(n, n, deg * n, seed=seed))
        elif kind == "banded":
            yield name, (lambda n=n, deg=deg, seed=seed: gen.banded(n, deg, seed=seed))
        else:
            b = c = (1 - a) * 0.4
            d = 1 - a - b - c
            yield name, (lambda s=s, deg=deg, a=a, b=b, c=c, d=d, seed=seed:
                         gen.rmat(s, deg * (1 << s), a, b, c, d, seed=seed))


def time_kernel(fn, flush, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.sum()  # clean lines: the timed call pays no write-back
        torch.cuda._sleep(200_000)  # GPU busy until the call is enqueued (bench._hold)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/timings.csv")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--ns", default="2,4,8,16,32,64,128")
    a = ap.parse_args()
    ns = [int(x) for x in a.ns.split(",")]
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB read sweep
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["matrix_id", "nnz", "mat_size", "std_row", "n_cols"] +
                   [f"t{k}" for k in range(8)] + ["label"])
        for name, mk in corpus(a.quick):
            M, K, rp, ci, va = mk()
            d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
            f = sk.extract_features(d, 0)
            for n in ns:
                B = gen.dense_operand(K, n, seed=n)
                Bcm = B.t().contiguous()
                C = torch.empty(M, n, device="cuda")
                ts = []
                for k in range(8):
                    Bk = Bcm if k & 2 else B
                    ts.append(time_kernel(lambda: sk.spmm_device(k, d, Bk, C, W=8), flush))
                label = int(np.argmin(ts))
                w.writerow([f"{name}", f.nnz, f.mat_size, repr(f.std_row), n] +
                           [repr(t) for t in ts] + [label])
                fh.flush()
                print(name, n, sk.KernelId.from_index(label).name(),
                      " ".join(f"{t*1e6:.1f}" for t in ts), flush=True)
            del d, rp, ci, va
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
