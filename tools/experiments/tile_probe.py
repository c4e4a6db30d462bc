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
SWEEP = os.environ.get("TILE_SWEEP", "") == "1"
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
        configs = [("default", {})]
        if SWEEP:
            configs += [(f"rl{rl}_u{u}", {"DASPMM_TILE_RL": str(rl), "DASPMM_TILE_U": str(u)})
                        for rl in (1, 8) for u in (2, 4, 8)]
        out = []
        for label, env in configs:
            os.environ["DASPMM_TILE"] = "1"
            for k in ("DASPMM_TILE_RL", "DASPMM_TILE_U"):
                os.environ.pop(k, None)
            os.environ.update(env)
            sk.reload_env()
            tt = t(lambda: sk.spmm_device(0, d, B, C1))
            vt = sk.plan_info(0, d, B, C1)
            same = bool(torch.equal(C0, C1))
            out.append(f"{label} {tt:7.1f}{'' if same else '!'}{'' if vt[0] == 'rb_tile' else '(' + vt[0] + ')'}")
        for k in ("DASPMM_TILE_RL", "DASPMM_TILE_U"):
            os.environ.pop(k, None)
        print(f"{name:16s} N={n:3d} base {tb:7.1f} us {vb[0]:8s} | " + " | ".join(out), flush=True)
    del d, rp, ci, va
    torch.cuda.empty_cache()
