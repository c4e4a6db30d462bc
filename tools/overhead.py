"""Per-call overhead probe: direct kernel launch vs graph-dispatched DA-SpMM vs cuSPARSE
on a small matrix (events around each call, GPU idle before the call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402


def t(fn, reps=50, busy=None):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        if busy is not None:
            busy.zero_()  # keep the GPU busy while the host enqueues the call
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) * 1e3)
    out.sort()
    return out[len(out) // 2]


model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
busy = torch.empty(64 << 20, device="cuda")
M, K, rp, ci, va = gen.uniform(1 << 14, 1 << 14, 16 << 14, seed=1)
d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
B = gen.dense_operand(K, 8, seed=2)
C = torch.empty(M, 8, device="cuda")
kout = torch.zeros(1, dtype=torch.int32, device="cuda")
for busy_flag in (None, busy):
    tag = "busy" if busy_flag is not None else "idle"
    print(tag, "empty torch op      ", round(t(lambda: C.zero_(), busy=busy_flag), 1), "us")
    for k in (0, 1, 4, 5):
        print(tag, f"direct k{k}           ", round(t(lambda: sk.spmm_device(k, d, B, C), busy=busy_flag), 1), "us")
    print(tag, "select only         ", round(t(lambda: sk.select_device(d, model, 8, kout), busy=busy_flag), 1), "us")
    print(tag, "graph DA-SpMM       ", round(t(lambda: sk.spmm_selected(d, model, B, C, kernel_out=kout), busy=busy_flag), 1), "us", int(kout.item()))
