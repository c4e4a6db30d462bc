"""Per-call cost of the data-aware decision (uncached): the device selector kernel alone
(daspmm_select), the reselect graph (selector + SWITCH + kernel) and the direct launch of
the published choice, each after an L2 read-sweep flush, CUDA events, mean of 20."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

dev = torch.device("cuda", 0)
model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
flush = torch.ones((256 << 20) // 4, device=dev)
st = torch.cuda.current_stream()


def timed(fn, reps=20):
    tot = 0.0
    for _ in range(reps):
        flush.sum()
        torch.cuda._sleep(200_000)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(st)
        fn()
        e.record(st)
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps * 1e3


for scale in (14, 17, 20):
    M, K, rp, ci, va = gen.rmat(scale, 16 << scale, 0.25, 0.25, 0.25, 0.25, seed=3)
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    for n in (4, 32, 128):
        B = gen.dense_operand(K, n, seed=5, device=dev)
        C = torch.empty(M, n, device=dev)
        out = torch.zeros(1, dtype=torch.int32, device=dev)
        sk.select_device(d, model, n, out)
        sk.spmm_selected(d, model, B, C, reselect=True)
        sk.spmm_selected(d, model, B, C)
        t_sel = timed(lambda: sk.select_device(d, model, n, out))
        t_res = timed(lambda: sk.spmm_selected(d, model, B, C, reselect=True))
        t_dir = timed(lambda: sk.spmm_selected(d, model, B, C))
        print(f"s{scale} N={n:4d} select kernel {t_sel:7.2f} us | reselect call {t_res:8.2f} us"
              f" | direct call {t_dir:8.2f} us | difference {t_res - t_dir:7.2f} us", flush=True)
