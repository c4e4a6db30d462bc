"""Packed column slices of B (round-2 probe).

tools/experiments/l2cap.cu showed that a column slice of a row-major B with a 512-B row
pitch uses only part of the L2 (a 16-column slice gathers at 3.4 TB/s strided vs 13.4 TB/s
packed, 32 columns 6.6 vs 12.8). This probe times, with the existing kernels, the
N = 32..128 calls as (a) one call on B as given, (b) B packed slice-major
(S x K x w, by torch) then S calls of width w, each on a contiguous K x w slice, writing
C's column slice in place. Prints pack time and pass time separately.

python tools/experiments/packed_slices.py [--only uniform_s20_d16,...] [--ns 32,64,128]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402


def time_fn(fn, flush, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="uniform_s20_d16,powerlaw_s20_d16,banded_s20_b8")
    ap.add_argument("--ns", default="32,64,128")
    ap.add_argument("--widths", default="16,32,64")
    ap.add_argument("--kernels", default="0,4")
    a = ap.parse_args()
    only = set(a.only.split(","))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for name, mk, _ in gen.workload("suite"):
        if name not in only:
            continue
        M, K, rp, ci, va = mk()
        d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
        for n in [int(x) for x in a.ns.split(",")]:
            B = gen.dense_operand(K, n, seed=n)
            C = torch.empty(M, n, device="cuda")
            for k in [int(x) for x in a.kernels.split(",")]:
                t1 = time_fn(lambda: sk.spmm_device(k, d, B, C), flush)
                ref = C.clone()
                line = [f"{name:18s} N={n:4d} k{k}  one call {t1:8.1f}us"]
                for w in [int(x) for x in a.widths.split(",")]:
                    if w >= n:
                        continue
                    S = n // w
                    Bp = torch.empty(S, K, w, device="cuda")

                    def pack():
                        Bp.copy_(B.view(K, S, w).permute(1, 0, 2))

                    def passes():
                        for s in range(S):
                            sk.spmm_device(k, d, Bp[s], C[:, s * w:(s + 1) * w])

                    def both():
                        pack()
                        passes()

                    tp = time_fn(pack, flush)
                    pack()
                    tq = time_fn(passes, flush)
                    tb = time_fn(both, flush)
                    err = (C - ref).abs().max().item()
                    line.append(f"w{w}: pack {tp:6.1f} passes {tq:7.1f} total {tb:7.1f} "
                                f"(err {err:.1e})")
                print(" | ".join(line), flush=True)
        del d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
