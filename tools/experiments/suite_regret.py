"""Selector regret on the suite (BASELINE configs[1]): every one of the 63 (matrix, N)
calls timed on all 8 design points (CM points on a column-major copy of B, as the
selector's training data), against the design point DA-SpMM selects. Prints per call
the selected and the fastest point, and the suite totals (sum of per-call times) for
the selection, the per-call best (an oracle selector) and each static point."""
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
NAMES = ["RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR", "EB+RM+SR", "EB+RM+PR", "EB+CM+SR",
         "EB+CM+PR"]


def t(fn, reps=5):
    for _ in range(2):
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


sel_tot, best_tot = 0.0, 0.0
static = [0.0] * 8
for name, mk, ns in gen.workload("suite"):
    M, K, rp, ci, va = mk()
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    for n in ns:
        B = gen.dense_operand(K, n, seed=1000 + n)
        Bcm = B.t().contiguous()
        C = torch.empty(M, n, device="cuda")
        kout = torch.zeros(1, dtype=torch.int32, device="cuda")
        sk.spmm_selected(d, model, B, C, kernel_out=kout)
        torch.cuda.synchronize()
        ksel = int(kout.item())
        ts = [t(lambda k=k: sk.spmm_device(k, d, Bcm if k & 2 else B, C)) for k in range(8)]
        tsel = t(lambda: sk.spmm_selected(d, model, B, C))
        kb = min(range(8), key=lambda k: ts[k])
        sel_tot += tsel
        best_tot += ts[kb]
        for k in range(8):
            static[k] += ts[k]
        print(f"{name:18s} N={n:3d} selected {NAMES[ksel]:9s} {tsel:8.1f} us  best {NAMES[kb]:9s} "
              f"{ts[kb]:8.1f} us  regret {tsel / ts[kb]:5.2f}", flush=True)
    del d, rp, ci, va
    torch.cuda.empty_cache()
print(f"suite: DA-SpMM {sel_tot / 1e3:.3f} ms, per-call best {best_tot / 1e3:.3f} ms "
      f"({best_tot / sel_tot:.3f} of the selection's time)")
for k in range(8):
    print(f"  static {NAMES[k]:9s} {static[k] / 1e3:8.3f} ms")
