"""Per-call time of the small suite calls (2^14 rows) after an L2 flush, split into what
the event pair sees: DA-SpMM with the optional kernel-id output (an extra H2D copy of the
id), DA-SpMM without it, the chosen kernel through daspmm_spmm, cuSPARSE's best
algorithm, and a one-element fill (the event + launch floor)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
model = sk.load_selector(open(os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                           "b200_selector.txt")).read())
flush = torch.ones((256 << 20) // 4, device="cuda")
tiny = torch.empty(1, device="cuda")


def t(fn, reps=50):
    for _ in range(5):
        fn()
    tot = 0.0
    for _ in range(reps):
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps * 1e3


print(f"floor (1-element fill): {t(lambda: tiny.fill_(1.0)):.2f} us")
for name, mk, _ in gen.workload("suite"):
    if "s14" not in name:
        continue
    M, K, rp, ci, va = mk()
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    for n in (2, 8, 32, 128):
        B = gen.dense_operand(K, n, seed=n)
        C = torch.empty(M, n, device="cuda")
        kout = torch.zeros(1, dtype=torch.int32, device="cuda")
        sk.spmm_selected(d, model, B, C, kernel_out=kout)
        torch.cuda.synchronize()
        kid = int(kout.item())
        a = t(lambda: sk.spmm_selected(d, model, B, C, kernel_out=kout))
        b = t(lambda: sk.spmm_selected(d, model, B, C))
        c = t(lambda: sk.spmm_device(kid, d, B, C)) if not (kid & 2) else float("nan")
        print(f"{name:18s} N={n:3d} k={kid} selected+kout {a:6.2f}  selected {b:6.2f}  "
              f"direct {c:6.2f} us", flush=True)
