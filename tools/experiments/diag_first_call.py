"""Diagnostic: does the bench's per-call event timing of a shallow GPU queue include host
enqueue latency? Times one c1-sized call the bench's way with variants."""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

M, K, rp, ci, va = gen.uniform(4096, 4096, 167_772, seed=1)
d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
B = gen.dense_operand(K, 32, seed=3)
C = torch.empty(M, 32, device="cuda")
kout = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
stream = torch.cuda.current_stream()


def one():
    sk.spmm_selected(d, model, B, C, kernel_out=kout, stream=stream)


def timed(steps, preflush=False, hold=None):
    ts = []
    for _ in range(3):
        flush.zero_(); one()
    torch.cuda.synchronize()
    if preflush:
        flush.zero_()
    for _ in range(steps):
        flush.zero_()
        if hold is not None:
            torch.cuda._sleep(hold)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(stream); one(); e.record(stream)
        ts.append((s, e))
    torch.cuda.synchronize()
    return [round(s.elapsed_time(e) * 1e3, 1) for s, e in ts]


print("plain      ", timed(5))
print("preflush   ", timed(5, preflush=True))
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "200"],
                     stdout=subprocess.DEVNULL)
time.sleep(0.3)
print("with smi   ", timed(5))
print("smi+pre    ", timed(5, preflush=True))
p.terminate()
t0 = time.perf_counter()
for _ in range(1000):
    one()
torch.cuda.synchronize()
print("host us per call", (time.perf_counter() - t0) * 1e3)
