"""Quick per-kernel timing probe (development tool; bench.py is the contract).

python tools/probe.py [--small] [--ns 2,8,32,128]
Prints one line per (matrix, N, kernel): time, GFLOP/s, algorithmic GB/s, and the
torch/cuSPARSE time for comparison.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402


def time_fn(fn, reps=10, flush=None):
    ts = []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--ns", default="2,8,32,128")
    ap.add_argument("--kernels", default="0,1,2,3,4,5,6,7")
    ap.add_argument("--W", type=int, default=8)
    ap.add_argument("--only", default="", help="comma list of suite matrix names")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-torch", action="store_true")
    ap.add_argument("--workload", default="suite")
    a = ap.parse_args()
    ns = [int(x) for x in a.ns.split(",")]
    ks = [int(x) for x in a.kernels.split(",")]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    only = set(a.only.split(",")) if a.only else None
    for name, mk, _ in gen.workload(a.workload, small=a.small):
        if only and name not in only:
            continue
        M, K, rp, ci, va = mk()
        d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
        nnz = ci.numel()
        At = torch.sparse_csr_tensor(rp.to(torch.int64), ci.to(torch.int64), va, (M, K))
        for n in ns:
            B = gen.dense_operand(K, n, seed=n)
            Bcm = B.t().contiguous()
            C = torch.empty(M, n, device="cuda")
            byt = gen.algorithmic_bytes(M, nnz, n, d.cols_touched)
            fl = gen.flops(nnz, n)
            t_ref = 1e9 if a.no_torch else time_fn(lambda: torch.sparse.mm(At, B), flush=flush,
                                                    reps=a.reps)
            line = [f"{name:20s} N={n:4d} nnz={nnz:9d} torch/cusparse {t_ref*1e3:8.1f}us "
                    f"{fl/t_ref/1e6:7.1f}GF"]
            for k in ks:
                Bk = Bcm if k & 2 else B
                t = time_fn(lambda: sk.spmm_device(k, d, Bk, C, W=a.W), flush=flush, reps=a.reps)
                line.append(f"k{k} {t*1e3:8.1f}us {fl/t/1e6:7.1f}GF {byt/t/1e6:6.0f}GB/s")
            print(" | ".join(line), flush=True)
        del d, At, rp, ci, va
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
