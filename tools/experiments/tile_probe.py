"""Dense row-panel tiles (tile.cuh) vs the base RB+RM+SR walk: per (matrix, N) the base
and tile times (L2 flushed by a read sweep before each run, median of reps), whether the
results are bit-identical, and the tile fill. DASPMM_TILE toggles the variant through
daspmm_reload_env()."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

flush = torch.ones((256 << 20) // 4, device="cuda")


def t(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def stencil2d(n):
    """5-point Laplacian on an n x n grid (rows sorted by column)."""
    idx = torch.arange(n * n, device="cuda", dtype=torch.int64)
    i, j = idx // n, idx % n
    rows, cols = [], []
    for di, dj in ((-1, 0), (0, -1), (0, 0), (0, 1), (1, 0)):
        ii, jj = i + di, j + dj
        ok = (ii >= 0) & (ii < n) & (jj >= 0) & (jj < n)
        rows.append(idx[ok])
        cols.append((ii * n + jj)[ok])
    return gen._to_csr(torch.cat(rows), torch.cat(cols), n * n, n * n, 5, torch.float32)


mats = [("banded_s14_b8", lambda: gen.banded(1 << 14, 8, seed=14)),
        ("banded_s17_b8", lambda: gen.banded(1 << 17, 8, seed=17)),
        ("banded_s20_b8", lambda: gen.banded(1 << 20, 8, seed=20)),
        ("banded_s20_b32", lambda: gen.banded(1 << 20, 32, seed=21)),
        ("stencil5_1024", lambda: stencil2d(1024)),
        ("uniform_s17_d16", lambda: gen.uniform(1 << 17, 1 << 17, 16 << 17, seed=17))]
for name, mk in mats:
    M, K, rp, ci, va = mk()
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    for n in (2, 4, 8, 16, 32, 64, 128):
        B = gen.dense_operand(K, n, seed=n)
        C0 = torch.empty(M, n, device="cuda")
        C1 = torch.empty(M, n, device="cuda")
        os.environ["DASPMM_TILE"] = "0"
        sk.reload_env()
        tb = t(lambda: sk.spmm_device(0, d, B, C0))
        vb = sk.plan_info(0, d, B, C0)
        os.environ["DASPMM_TILE"] = "1"
        sk.reload_env()
        tt = t(lambda: sk.spmm_device(0, d, B, C1))
        vt = sk.plan_info(0, d, B, C1)
        same = bool(torch.equal(C0, C1))
        print(f"{name:16s} N={n:3d} base {tb:8.1f} us {vb}  tile {tt:8.1f} us {vt}  "
              f"speedup {tb / tt:5.2f}  bit-identical {same}", flush=True)
    # non-finite B under an absent entry: the tile walk must fall back to the CSR replay
    B = gen.dense_operand(K, 32, seed=3)
    B[K // 2, :] = float("inf")
    B[K // 3, 5] = float("nan")
    os.environ["DASPMM_TILE"] = "0"
    sk.reload_env()
    C0 = torch.empty(M, 32, device="cuda")
    C1 = torch.empty(M, 32, device="cuda")
    sk.spmm_device(0, d, B, C0)
    os.environ["DASPMM_TILE"] = "1"
    sk.reload_env()
    sk.spmm_device(0, d, B, C1)
    same = bool(torch.equal(C0.nan_to_num(1.5, 7.0, -7.0), C1.nan_to_num(1.5, 7.0, -7.0))) and \
        bool(torch.equal(C0.isnan(), C1.isnan()))
    print(f"{name:16s} non-finite B: identical to base {same}; nonfinite rows "
          f"{int((~C1.isfinite()).any(1).sum())}", flush=True)
    del d, rp, ci, va
    torch.cuda.empty_cache()
