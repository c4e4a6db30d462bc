"""Debug helper: DA-SpMM (graph-dispatched) over the small suite, one call at a time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
for name, mk in gen.suite(small=True):
    M, K, rp, ci, va = mk()
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    for n in (2, 4, 8, 16, 32, 64, 128):
        B = gen.dense_operand(K, n, seed=n)
        C = torch.empty(M, n, device="cuda")
        kout = torch.zeros(1, dtype=torch.int32, device="cuda")
        print(name, n, "...", flush=True, end=" ")
        sk.spmm_selected(d, model, B, C, kernel_out=kout)
        torch.cuda.synchronize()
        print(sk.KernelId.from_index(int(kout.item())).name(), flush=True)
