"""Where the e2e step's time goes: the suite's exact transfer sizes (B_i up, C_i down)
pipelined with and without the DA-SpMM calls in between, against the PCIe floor.
  transfers_only  H2D_i on an upload stream, D2H_i on a download stream after H2D_i
  independent     both directions free-running (no per-call dependency)
  bench_e2e       what bench.py times (upload -> compute -> download per call)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402

ns = [2, 4, 8, 16, 32, 64, 128]
sizes = []
for s in (14, 17, 20):
    for _kind in range(3):
        rows = 1 << s
        for n in ns:
            sizes.append((rows * n, rows * n))  # B is K x N, C is M x N (square matrices)
hB = [torch.empty(b, dtype=torch.float32).pin_memory() for b, _ in sizes]
hC = [torch.empty(c, dtype=torch.float32).pin_memory() for _, c in sizes]
dB = [torch.empty(b, device="cuda") for b, _ in sizes]
dC = [torch.zeros(c, device="cuda") for _, c in sizes]
up, down, comp = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
tot = sum(b for b, _ in sizes) * 4 / 1e9
print(f"bytes each way per step: {tot:.3f} GB", flush=True)


def run_multi(k, steps=5):
    """k streams per direction, calls assigned round-robin."""
    ups = [torch.cuda.Stream() for _ in range(k)]
    downs = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    for st in ups + downs:
        st.wait_stream(comp)
    for _ in range(steps):
        for i in range(len(sizes)):
            with torch.cuda.stream(ups[i % k]):
                dB[i].copy_(hB[i], non_blocking=True)
            with torch.cuda.stream(downs[i % k]):
                hC[i].copy_(dC[i], non_blocking=True)
    for st in ups + downs:
        comp.wait_stream(st)
    e.record(comp)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def run(mode, steps=5):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    up.wait_stream(comp)
    down.wait_stream(comp)
    for _ in range(steps):
        for i in range(len(sizes)):
            with torch.cuda.stream(up):
                dB[i].copy_(hB[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
            if mode == "transfers_only":
                down.wait_event(ev)
            with torch.cuda.stream(down):
                hC[i].copy_(dC[i], non_blocking=True)
    comp.wait_stream(up)
    comp.wait_stream(down)
    e.record(comp)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for mode in ("independent", "transfers_only", "independent", "transfers_only"):
    print(f"{mode:16s} {run(mode):8.2f} ms per step", flush=True)
for k in (1, 2, 4, 2, 1):
    print(f"independent x{k} streams per direction {run_multi(k):8.2f} ms per step", flush=True)
