"""Is the per-call CUDA-event time of a small call inflated by host enqueue gaps?
Times each s14/s17 suite call as bench.py does (read-sweep flush, events around the
DA-SpMM call), then again with a ~100 us device spin after the flush so the GPU is
still busy when the host has finished enqueueing the call. Mean of 20."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

dev = torch.device("cuda", 0)
model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
flush = torch.ones((256 << 20) // 4, device=dev)
st = torch.cuda.current_stream()
mats = [m for m in bench.build_suite(False, 0, 1, "suite") if m["M"] <= (1 << 17)]


def timed(fn, spin, reps=20):
    tot = 0.0
    for _ in range(reps):
        flush.sum()
        if spin:
            torch.cuda._sleep(200_000)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(st)
        fn()
        e.record(st)
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / reps * 1e3


t_plain = t_spin = 0.0
for m in mats:
    dd = m["full"]
    for n in m["ns"]:
        B = gen.dense_operand(m["K"], n, seed=1000 + n, device=dev)
        C = torch.empty(m["M"], n, device=dev)
        sk.spmm_selected(dd, model, B, C)
        a = timed(lambda: sk.spmm_selected(dd, model, B, C), False)
        b = timed(lambda: sk.spmm_selected(dd, model, B, C), True)
        t_plain += a
        t_spin += b
        print(f"{m['name']:18s} N={n:4d} as bench {a:7.2f} us | GPU kept busy {b:7.2f} us", flush=True)
print(f"total as bench {t_plain:.1f} us, GPU kept busy {t_spin:.1f} us")
