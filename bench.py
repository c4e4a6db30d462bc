"""bench.py — DA-SpMM on B200 (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the synthetic suite — uniform, banded and
power-law (R-MAT, Graph500 skew) CSR matrices with 2^14 / 2^17 / 2^20 rows at
average degree 16 (banded: half-width 8), each multiplied by a dense B of
N = 2, 4, 8, 16, 32, 64, 128 columns, fp32. One *step* runs DA-SpMM — the on-device
selector plus the selected sm_100a kernel, dispatched on the device through a CUDA
graph SWITCH node — once for every (matrix, N) pair of the suite.

  value     suite GFLOP/s = sum(2*nnz*N) / sum(device time), inputs resident in HBM,
            L2 flushed (256 MiB read sweep) before every call, CUDA events per call.
  e2e       same metric through the public API with host operands: pinned-host B ->
            device, DA-SpMM, C -> pinned host, all inside the timed region.
  roofline  HBM roofline of the step: algorithmic bytes (SURVEY §8d:
            4(M+1) + 8 nnz + 4 N K_touched + 4 N M per call) / device time, against
            MEASURED_PEAKS.json hbm_gbs; `dominant` repeats it for the largest call.
  cpu_baseline  the reference's own spmm() (oracle/_ref, unmodified headers) RB+RM+SR
            on all host cores over a bounded sample of the suite.

--gpus N (torchrun): every rank takes an nnz-balanced row panel of every matrix
(partition.hpp cut rule) with B replicated; no collective on the data path; time =
max over ranks. --impl reference: the reference CPU path alone (rank 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NS = (2, 4, 8, 16, 32, 64, 128)
FLUSH_BYTES = 256 << 20


# ------------------------------------------------------------------ helpers
def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms DURING the timed region
    by a separate nvidia-smi process (-lms), so sampling never holds this process's GIL
    while calls are being enqueued."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._path = f"/tmp/daspmm_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self._fh = open(self._path, "w")
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=self._fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)  # first sample lands before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            time.sleep(0.25)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._fh.close()
            try:
                for line in open(self._path):
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 6:
                        self.samples.append(parts)
                os.remove(self._path)
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _key(c):
    """Call label: matrix/N, plus the column slice for an N-split share."""
    k = f'{c["m"]["name"]}/N{c.get("n_full", c["n"])}'
    if c.get("n_full", c["n"]) != c["n"]:
        k += f'[cols {c["cols"][0]}:{c["cols"][1]}]'
    return k


def _flush(buf):
    """Evicts L2 between timed calls with a READ sweep of a buffer twice the L2 size:
    the lines it leaves are clean, so the next call pays no write-back for them (a
    zero-fill would leave up to 126 MB of dirty lines for the timed call to drain).
    Then holds the GPU busy (_hold) so the timed call is enqueued before it can start."""
    buf.sum()
    _hold()


HOLD_CYCLES = 200_000  # ~100 us at 1965 MHz


def _hold():
    """A ~100 us device spin on the launching stream before a timed call's start event,
    so the host's per-call work (operand checks, ctypes, event records) can never land
    inside the event pair on an idle GPU. Measured (tools/experiments/small_call_hold_probe.py,
    profiles/r02e_small_call_probe.txt): the per-call times are the same with and without
    it apart from the first call of a handle, so it is a guard, not a correction. The
    spin touches no memory, so the flushed L2 state is unchanged."""
    import torch

    torch.cuda._sleep(HOLD_CYCLES)


def _max_over_ranks(v: float, dev) -> float:
    """Max of a per-rank scalar over all ranks (device tensor for NCCL, host for gloo)."""
    import torch
    import torch.distributed as dist

    on_dev = dist.get_backend() == "nccl"
    tt = torch.tensor([v], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ workload
def build_suite(small: bool, rank: int, world: int, workload: str = "suite"):
    """Generates the workload's matrices on the current device; returns per-matrix dicts
    holding the rank's row panel as a DeviceCsr (and the N values to run)."""
    import torch

    from paper_2202_08556_b200 import gen, multi
    from paper_2202_08556_b200 import spmmkit as sk

    mats = []
    for name, mk, ns in gen.workload(workload, small=small):
        M, K, rp, ci, va = mk()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        full = sk.DeviceCsr.from_device(M, K, rp, ci, va)
        torch.cuda.synchronize()
        t_handle = (time.perf_counter() - t0) * 1e3
        mats.append(dict(name=name, M=M, K=K, nnz_total=int(ci.numel()), full=full,
                         rp=rp, ci=ci, va=va, ns=ns, handle_ms=t_handle))
    return mats


def _setup_costs(mats):
    """Handle-creation cost per matrix (not in any timed SpMM): device arrays adopted
    (features, empty rows, K_touched, column windows: daspmm_csr_create_device), host int64
    arrays uploaded and validated / compacted on the device (daspmm_csr_create_host),
    shuffled device COO triplets sorted and merged on the device (from_coo),
    extract_features' exact std_row replay, and what the first calls build lazily (COO
    row ids; the row-panel tiles where they pay)."""
    import numpy as np
    import torch

    from paper_2202_08556_b200 import spmmkit as sk

    out = {}
    for m in mats:
        rp = m["rp"].cpu().numpy().astype(np.int64)
        ci = m["ci"].cpu().numpy().astype(np.int64)
        va = m["va"].cpu().numpy()
        a = sk.CsrMatrix(m["M"], m["K"], rp, ci, va, np.float32)
        t_dev = []
        for _ in range(3):  # from device arrays (borrowed): features, windows, K_touched
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hd = sk.DeviceCsr.from_device(m["M"], m["K"], m["rp"], m["ci"], m["va"])
            torch.cuda.synchronize()
            t_dev.append((time.perf_counter() - t0) * 1e3)
            hd.close()
        t_host, t_feat, t_lazy = [], [], []
        B = torch.zeros(m["K"], 32, device="cuda")
        Cb = torch.empty(m["M"], 32, device="cuda")
        for _ in range(3):  # median of 3: single host-side timings vary with the box
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = sk.DeviceCsr.from_host(a)
            torch.cuda.synchronize()
            t_host.append((time.perf_counter() - t0) * 1e3)
            t0 = time.perf_counter()
            sk.extract_features(h, 32)
            t_feat.append((time.perf_counter() - t0) * 1e3)
            # lazily built structures on the first calls (COO row ids, row-panel tiles):
            # first RB+RM+SR and EB+RM+SR calls minus the same calls again
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sk.spmm_device(0, h, B, Cb)
            sk.spmm_device(4, h, B, Cb)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            sk.spmm_device(0, h, B, Cb)
            sk.spmm_device(4, h, B, Cb)
            torch.cuda.synchronize()
            t_lazy.append(((t1 - t0) - (time.perf_counter() - t1)) * 1e3)
            h.close()
        # from shuffled device COO triplets (daspmm_csr_create_coo_device: sort, merge,
        # offsets on the device, then the same handle set-up as from_device)
        rows = torch.repeat_interleave(torch.arange(m["M"], device="cuda"),
                                       (m["rp"][1:] - m["rp"][:-1]).long())
        perm = torch.randperm(rows.numel(), device="cuda")
        cr, cc, cv = rows[perm], m["ci"].long()[perm], m["va"][perm]
        t_coo = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hc = sk.DeviceCsr.from_coo_device(m["M"], m["K"], cr, cc, cv)
            torch.cuda.synchronize()
            t_coo.append((time.perf_counter() - t0) * 1e3)
            hc.close()
        del rows, perm, cr, cc, cv
        t_host, t_feat, t_lazy = sorted(t_host)[1], sorted(t_feat)[1], sorted(t_lazy)[1]
        out[m["name"]] = {"from_device_ms": round(sorted(t_dev)[1], 3),
                          "from_coo_device_ms": round(sorted(t_coo)[1], 3),
                          "from_host_ms": round(t_host, 3),
                          "extract_features_exact_ms": round(t_feat, 3),
                          "first_call_lazy_build_ms": round(t_lazy, 3),
                          "rows": m["M"], "nnz": m["nnz_total"]}
        del a, rp, ci, va
    return out


def shard_calls(mats, ns_override, rank: int, world: int):
    """This rank's share of the workload's (matrix, N) calls (multi.schedule_units):
    large calls split across all ranks by daspmm_multi_plan — nnz-balanced row panels
    with B replicated, or, where it moves fewer bytes per GPU (wide B, e.g. c5 N = 256),
    N-split column slices with A replicated — the rest whole, longest first to the least
    loaded rank. Returns [(matrix, N, handle, (r0, r1), (c0, c1))] and every unit (for the
    whole-job flop count)."""
    import torch

    from paper_2202_08556_b200 import multi

    units = [(m, n) for m in mats for n in (ns_override or m["ns"])]
    costs = [multi.estimate_call_us(m["nnz_total"], n) for m, n in units]
    # DASPMM_SPLIT_FRAC (default 0.5) forces more row splitting, e.g. to exercise the
    # panel path and C assembly on 2 ranks; DASPMM_SPLIT_MODE=rows|cols forces the split.
    assign, split = multi.schedule_units(costs, world,
                                         float(os.environ.get("DASPMM_SPLIT_FRAC", "0.5")))
    force = {"rows": multi.SPLIT_ROWS, "cols": multi.SPLIT_COLS}.get(
        os.environ.get("DASPMM_SPLIT_MODE", ""), multi.SPLIT_AUTO)
    panels = {}
    mine = []
    for i in assign[rank]:
        m, n = units[i]
        if split[i]:
            mode, bounds = multi.plan(m["full"], world, n, force)
            lo, hi = int(bounds[rank]), int(bounds[rank + 1])
            if mode == "cols":
                mine.append((m, n, m["full"], (0, m["M"]), (lo, hi)))
                continue
            if m["name"] not in panels:
                panels[m["name"]] = (m["full"].panel(lo, hi), (lo, hi))
                torch.cuda.synchronize()
            d, rows = panels[m["name"]]
        else:
            d, rows = m["full"], (0, m["M"])
        mine.append((m, n, d, rows, (0, n)))
    return mine, units


def run_ours(args):
    import torch

    from paper_2202_08556_b200 import gen
    from paper_2202_08556_b200 import spmmkit as sk

    world, rank, local = _dist()
    # one process per GPU; ranks beyond the visible devices share them round-robin (only
    # for exercising the multi-rank logic on a 1-GPU box with DASPMM_DIST_BACKEND=gloo)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("DASPMM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    sk.lib()  # fail loudly if the CUDA library is missing
    model = sk.load_selector(open(args.model).read())
    mats = build_suite(args.small, rank, world, args.workload)
    flush = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    ns_override = [int(n) for n in args.ns.split(",")] if args.ns else None
    ns = sorted({n for m in mats for n in (ns_override or m["ns"])})

    # Operands per (matrix, N) call of this rank: B replicated, C the local panel.
    mine, units = shard_calls(mats, ns_override, rank, world)
    calls = []
    for m, n, d, rows, (c0, c1) in mine:
        B = gen.dense_operand(m["K"], n, seed=1000 + n, device=dev)
        w = c1 - c0
        if w != n:  # N-split: this rank's column slice of the replicated-seed B
            B = B[:, c0:c1].contiguous()
        Cp = torch.empty(d.num_rows, w, device=dev)
        kout = torch.zeros(1, dtype=torch.int32, device=dev)
        calls.append(dict(m=m, n=w, n_full=n, cols=(c0, c1), d=d, rows=rows, B=B, C=Cp,
                          kout=kout, flops=gen.flops(d.nnz(), w),
                          bytes=gen.algorithmic_bytes(d.num_rows, d.nnz(), w, d.cols_touched)))
    stream = torch.cuda.current_stream(dev)

    def one(c, report=False):
        # the optional kernel-id output costs a small H2D copy per call (~4 us after an
        # L2 flush), so only the untimed warm-up asks for it
        sk.spmm_selected(c["d"], model, c["B"], c["C"], kernel_out=c["kout"] if report else None,
                         stream=stream)

    def step(times=None):
        for i, c in enumerate(calls):
            _flush(flush)
            if times is None:
                one(c, report=True)
            else:
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record(stream)
                one(c)
                e.record(stream)
                times[i].append((s, e))

    # The clock sampler starts before the warm-up: its start-up pause would otherwise
    # leave the GPU idle (and its clocks relaxed) right before the first timed call.
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        times = [[] for _ in calls]
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            step(times)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_call_ms = [sum(s.elapsed_time(e) for s, e in t) / max(args.steps, 1) for t in times]
    step_ms = sum(per_call_ms)
    if world > 1:
        step_ms = _max_over_ranks(step_ms, dev)
    total_flops = sum(gen.flops(m["nnz_total"], n) for m, n in units)  # all ranks' units
    value = total_flops / (step_ms * 1e-3) / 1e9

    # kernel choices and launch count: after the warm-up every call's decision is
    # published, so a timed call is [EB prologue] + the chosen kernel (no selector node)
    chosen = [int(c["kout"].item()) for c in calls]
    launches_per_step = sum(1 + (1 if k >= 4 else 0) for k in chosen)

    # roofline over this rank's calls
    peak, peak_kind = _peaks()
    my_bytes = sum(c["bytes"] for c in calls)
    achieved = my_bytes / (sum(per_call_ms) * 1e-3) / 1e9
    dom = max(range(len(calls)), key=lambda i: per_call_ms[i])
    dom_ach = calls[dom]["bytes"] / (per_call_ms[dom] * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        key = _key(calls[dom])
        traffic = tr.get(key)
    except Exception:
        pass

    # ---- e2e: host operands through the public API (pinned H2D, DA-SpMM, D2H)
    e2e = parity = warm = overhead = batched = setup = None
    # operands too large to stage in pinned host memory (c5: 68 GB) skip e2e; decided on
    # the largest rank's operands so every rank takes the same branch (_e2e has collectives)
    op_bytes = float(sum(c["B"].numel() + c["C"].numel() for c in calls) * 4)
    if world > 1:
        op_bytes = _max_over_ranks(op_bytes, dev)
    if args.profile_step:
        pass  # --profile-step: only the warm-up and the timed steps (ncu launch lists)
    elif op_bytes > (16 << 30):
        e2e = None
    else:
        e2e = _e2e(calls, one, stream, args, world, total_flops)
    if not args.profile_step:
        parity = _parity_map(calls) if rank == 0 else None
        warm = _warm(calls, one, stream, world, dev, total_flops)
        overhead = _da_overhead(calls, model, stream, flush) if rank == 0 else None
        batched = _batched_small(calls, model, flush, per_call_ms) if rank == 0 else None
        setup = _setup_costs(mats) if rank == 0 and world == 1 else None
    assembly = None
    if world > 1:
        try:
            assembly = _assembly(calls, mats, world, dev)
        except Exception as ex:  # optional measurement: never lose the bench line to it
            assembly = {"error": str(ex)[:200]}
    if args.roofline_table and rank == 0:
        _write_roofline_table(args.roofline_table, calls, per_call_ms, chosen, peak)
    return _report(args, world, rank, mats, calls, ns, step_ms, value, chosen, launches_per_step,
                   per_call_ms, dom, dom_ach, achieved, peak, peak_kind, traffic, clk, e2e, parity,
                   flush, assembly, warm, overhead, batched, setup)


def _batched_small(calls, model, flush, per_call_ms, reps=5, max_nnz=300_000):
    """The small calls of the workload (<= 300K nnz: the 2^14-row matrices) as one CUDA
    graph (spmmkit.SpmmBatch: the chosen kernels' launches, EB prologues included),
    timed cold (L2 flushed before each replay) against the same calls launched one by
    one (their per-call times of the main measurement)."""
    import torch

    from paper_2202_08556_b200 import spmmkit as sk

    idx = [i for i, c in enumerate(calls) if c["d"].nnz() <= max_nnz]
    if not idx:
        return None
    batch = sk.SpmmBatch([(calls[i]["d"], calls[i]["B"], calls[i]["C"]) for i in idx], model)
    batch.run()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        _flush(flush)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        batch.run()
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    ms = tot / reps
    one_by_one = sum(per_call_ms[i] for i in idx)
    # the floor of a one-by-one call: a minimal kernel between the same event pair, after
    # the same flush and hold (launch + event latency with nothing to do)
    floor = 0.0
    for _ in range(reps):
        _flush(flush)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        torch.cuda._sleep(0)
        e.record()
        torch.cuda.synchronize()
        floor += s.elapsed_time(e)
    return {"calls": len(idx), "graph_ms": round(ms, 4),
            "empty_launch_us": round(floor / reps * 1e3, 2),
            "us_per_call": round(ms * 1e3 / len(idx), 2),
            "one_by_one_ms": round(one_by_one, 4),
            "one_by_one_us_per_call": round(one_by_one * 1e3 / len(idx), 2),
            "protocol": "spmmkit.SpmmBatch (one graph launch for all of them), L2 flushed once "
                        f"before each replay, mean of {reps}"}


def _warm(calls, one, stream, world, dev, total_flops, reps=3):
    """The same calls with a warm L2 (no flush; each call run `reps` times back to back,
    the mean of the last reps-1 taken): the figure beside the cold, flushed one."""
    import torch

    per = []
    for c in calls:
        one(c)
        torch.cuda._sleep(HOLD_CYCLES * reps)  # _hold, long enough for all reps' enqueues
        evs = []
        for _ in range(reps):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            one(c)
            e.record(stream)
            evs.append((s, e))
        torch.cuda.synchronize()
        per.append(sum(s.elapsed_time(e) for s, e in evs[1:]) / (reps - 1))
    ms = sum(per)
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    dom = max(range(len(calls)), key=lambda i: per[i])
    return {"value": round(total_flops / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "ms_per_step": round(ms, 4),
            "dominant": {"call": _key(calls[dom]),
                         "ms": round(per[dom], 4)},
            "protocol": f"no L2 flush; each call {reps}x back to back, mean of the last {reps - 1}"}


def _da_overhead(calls, model, stream, flush, reps=3):
    """Uncached DA-SpMM: per call, the device selector (ensemble walk) + SWITCH dispatch +
    the chosen kernel (DASPMM_RESELECT), against the steady-state call that launches the
    published choice directly, and against a plain daspmm_spmm of that kernel. L2 flushed
    before every run; CUDA events on the launching stream."""
    import torch

    from paper_2202_08556_b200 import spmmkit as sk

    def timed(fn):
        tot = 0.0
        for _ in range(reps):
            _flush(flush)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        return tot / reps

    resel, direct, plain = 0.0, 0.0, 0.0
    for c in calls:
        kid = int(c["kout"].item())
        sk.spmm_selected(c["d"], model, c["B"], c["C"], kernel_out=c["kout"], stream=stream,
                         reselect=True)  # builds the reselect graph outside the timing
        resel += timed(lambda: sk.spmm_selected(c["d"], model, c["B"], c["C"], stream=stream,
                                                reselect=True))
        direct += timed(lambda: sk.spmm_selected(c["d"], model, c["B"], c["C"], stream=stream))
        # what DA-SpMM runs on this row-major B: the choice, or its layout twin for CM
        plain += timed(lambda: sk.spmm_device(kid & ~2, c["d"], c["B"], c["C"], stream=stream))
    n = len(calls)
    return {"reselect_ms_per_step": round(resel, 4), "direct_ms_per_step": round(direct, 4),
            "plain_kernel_ms_per_step": round(plain, 4),
            "selector_dispatch_us_per_call": round((resel - direct) / n * 1e3, 2),
            "cached_dispatch_us_per_call": round((direct - plain) / n * 1e3, 2),
            "note": "reselect = device selector walk + graph SWITCH + kernel every call "
                    "(the reference's per-call predict_kernel flow, spmmkit_cli.cpp:239-270); "
                    "direct = published choice launched directly; plain = daspmm_spmm of the "
                    "kernel that runs (a CM choice runs its RM layout twin on the row-major B)"}


def _parity_map(calls):
    """Every timed call checked against the fp64 oracle on sampled rows (oracle/sampled.py:
    random rows + rows straddling EB chunk / CTA boundaries), outside the timed region."""
    import numpy as np

    from oracle import sampled as S

    out, fails, worst = {}, [], 0.0
    for c in calls:
        m = c["m"]
        r0, r1 = c["rows"]
        rp_h = m["rp"][r0:r1 + 1].cpu().numpy().astype(np.int64)
        rp_h = rp_h - rp_h[0]
        rows = S.sample_rows(rp_h, n_random=128, n_boundary=8, seed=c["n"])
        res = S.check(m["rp"], m["ci"], m["va"], m["K"], c["B"], c["C"], rows + r0, row0=r0)
        key = _key(c)
        out[key] = round(res["max_ratio"], 4)
        worst = max(worst, res["max_ratio"])
        if not res["ok"]:
            fails.append(key)
    return {"calls_checked": len(calls), "calls_passed": len(calls) - len(fails),
            "failed": fails, "worst_err_over_bound": round(worst, 4),
            "check": "fp64 oracle on sampled rows (random + EB/CTA boundary rows); "
                     "|y - y64| <= 2 gamma(len+1) sum|a x|",
            "err_over_bound_per_call": out}


def _assembly(calls, mats, world, dev):
    """C assembly, timed apart from the SpMM (optional, only where the output
    must be assembled): the largest row-split call's panels all-gathered into the full C
    on every rank (multi.gather_rows, NCCL over NVLink). Max over ranks."""
    import torch

    from paper_2202_08556_b200 import multi

    split = [c for c in calls if c["rows"] != (0, c["m"]["M"]) or c["n"] != c["n_full"]]
    big = max(split, key=lambda c: c["m"]["M"] * c["n_full"]) if split else None
    name = _key(big) if big else None
    names = [None] * world
    import torch.distributed as dist

    dist.all_gather_object(names, name)
    if len(set(names)) != 1 or name is None:  # every rank must join the same collective
        return None
    full_bytes = big["m"]["M"] * big["n_full"] * 4
    if full_bytes > (8 << 30):  # c5: 34 GB per GPU, more than the SpMM itself moves
        return {"call": name, "ms": None, "bytes_per_rank": full_bytes,
                "skipped": "assembled C above 8 GB per GPU"}
    by_cols = big["n"] != big["n_full"]
    if by_cols:
        bounds = multi.col_split(big["n_full"], world)
        gather = lambda: multi.gather_cols(big["C"], bounds)  # noqa: E731
    else:
        _, cuts = multi.plan(big["m"]["full"], world, big["n_full"], multi.SPLIT_ROWS)
        gather = lambda: multi.gather_rows(big["C"], cuts)  # noqa: E731
    full = gather()  # warm-up (communicator set-up)
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    full = gather()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), dev)
    nbytes = full.numel() * full.element_size()
    out = {"call": name, "ms": round(ms, 4), "bytes_per_rank": nbytes,
           "collective": "all-gather of padded column slices (multi.gather_cols)" if by_cols
           else "all-gather of padded row panels (multi.gather_rows)"}
    # Fused alternative (NCCL runs only, one rank per GPU): the RB+RM+SR panel kernel
    # stores every finished row into all ranks' copies of C (symmetric memory over
    # NVLink); its time includes the SpMM itself. Opt-in (DASPMM_BENCH_FUSED=1): it meets
    # at device-side symmetric-memory barriers, which would spin if one rank failed
    # before them, and it has not yet run on a multi-GPU box — the default multi-GPU
    # bench line must not depend on it.
    if dist.get_backend() == "nccl" and not by_cols and \
            os.environ.get("DASPMM_BENCH_FUSED") == "1":
        try:
            import torch.distributed._symmetric_memory as symm_mem

            r0 = big["rows"][0]
            Cs = symm_mem.empty(big["m"]["M"], big["n"], dtype=torch.float32, device=dev)
            multi.spmm_rows_allgather(big["d"], big["B"], big["m"]["M"], r0, C_full=Cs)
            torch.cuda.synchronize()
            dist.barrier()
            s.record()
            multi.spmm_rows_allgather(big["d"], big["B"], big["m"]["M"], r0, C_full=Cs)
            e.record()
            torch.cuda.synchronize()
            out["fused_spmm_allgather_ms"] = round(_max_over_ranks(s.elapsed_time(e), dev), 4)
            out["fused_equals_nccl"] = bool(torch.equal(Cs, full))
        except Exception as ex:  # never let the optional path break the bench line
            out["fused_spmm_allgather_ms"] = None
            out["fused_error"] = str(ex)[:200]
    return out


def _e2e(calls, one, stream, args, world, total_flops):
    """End to end through the public API with host operands: every call of the step
    copies its B from pinned host memory, runs DA-SpMM and copies its C back. Calls are
    independent, so the step is pipelined the way a user would batch them, one stream per
    PCIe direction beside the compute stream: B_i+1 uploads while call i computes and C_i-1
    downloads (PCIe is full duplex), each buffer reused only after its last reader."""
    import torch

    dev = calls[0]["B"].device
    hostB = [c["B"].cpu().pin_memory() for c in calls]
    hostC = [torch.empty(c["C"].shape, dtype=torch.float32).pin_memory() for c in calls]
    h2d = sum(b.numel() * 4 for b in hostB)
    d2h = sum(h.numel() * 4 for h in hostC)
    up = torch.cuda.Stream(dev)
    down = torch.cuda.Stream(dev)
    landed = [torch.cuda.Event() for _ in calls]   # B_i uploaded
    done = [torch.cuda.Event() for _ in calls]     # C_i computed (B_i consumed)
    drained = [torch.cuda.Event() for _ in calls]  # C_i copied out

    def e2e_step(first=False):
        for i, c in enumerate(calls):
            with torch.cuda.stream(up):
                if not first:
                    up.wait_event(done[i])  # B_i of the previous step is consumed
                c["B"].copy_(hostB[i], non_blocking=True)
                landed[i].record(up)
            stream.wait_event(landed[i])
            if not first:
                stream.wait_event(drained[i])  # C_i of the previous step is out
            one(c)
            done[i].record(stream)
            down.wait_event(done[i])
            with torch.cuda.stream(down):
                hostC[i].copy_(c["C"], non_blocking=True)
            drained[i].record(down)

    e2e_step(first=True)
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5 if args.workload == "suite" else 1))
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    up.wait_stream(stream)  # the first upload starts inside the timed region
    for _ in range(e2e_steps):
        e2e_step()
    stream.wait_event(drained[-1])
    e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s.elapsed_time(e) / e2e_steps
    if world > 1:
        e2e_ms = _max_over_ranks(e2e_ms, dev)
    e2e_value = total_flops / (e2e_ms * 1e-3) / 1e9
    bound = _pcie_bound_ms(dev, h2d, d2h)
    return {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
            "pcie": bound,
            "pipeline": "H2D stream -> DA-SpMM on the compute stream -> D2H stream, "
                        f"{e2e_steps} steps back to back"}


def _pcie_bound_ms(dev, h2d, d2h, mb=512):
    """The link's floor for the e2e step: pinned H2D and D2H rates measured with both
    directions busy at once (512 MB each way), and the step's bytes at those rates."""
    import torch

    n = (mb << 20) // 4
    hb = torch.empty(n, dtype=torch.float32).pin_memory()
    hc = torch.empty(n, dtype=torch.float32).pin_memory()
    db = torch.empty(n, dtype=torch.float32, device=dev)
    dc = torch.zeros(n, dtype=torch.float32, device=dev)
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best_up = best_dn = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(up)
        ev[2].record(down)
        with torch.cuda.stream(up):
            db.copy_(hb, non_blocking=True)
        with torch.cuda.stream(down):
            hc.copy_(dc, non_blocking=True)
        ev[1].record(up)
        ev[3].record(down)
        torch.cuda.synchronize()
        best_up = min(best_up, ev[0].elapsed_time(ev[1]))
        best_dn = min(best_dn, ev[2].elapsed_time(ev[3]))
    gbs_up = (n * 4) / (best_up * 1e-3) / 1e9
    gbs_dn = (n * 4) / (best_dn * 1e-3) / 1e9
    floor = max(h2d / (gbs_up * 1e9), d2h / (gbs_dn * 1e9)) * 1e3
    return {"h2d_gbs": round(gbs_up, 1), "d2h_gbs": round(gbs_dn, 1),
            "floor_ms_per_step": round(floor, 3),
            "protocol": f"{mb} MB pinned each way, both directions at once, best of 3"}


def _report(args, world, rank, mats, calls, ns, step_ms, value, chosen, launches_per_step,
            per_call_ms, dom, dom_ach, achieved, peak, peak_kind, traffic, clk, e2e, parity,
            flush, assembly=None, warm=None, overhead=None, batched=None, setup=None):
    import torch.distributed as dist

    from paper_2202_08556_b200 import spmmkit as sk

    result = {
        "metric": "SpMM GFLOP/s (2*nnz*N/t), DA-SpMM over the synthetic suite",
        "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": ("configs[1] synthetic suite: uniform/banded/power-law, "
                                + ("2^14,2^17" if args.small else "2^14,2^17,2^20")
                                + " rows, deg 16, N=" + ",".join(map(str, ns)))
                               if args.workload == "suite" else
                               f"{args.workload}: " + ", ".join(
                                   f'{m["name"]} M={m["M"]} nnz={m["nnz_total"]}' for m in mats)
                               + " N=" + ",".join(map(str, ns)),
                   "matrices": [m["name"] for m in mats], "ns": ns,
                   "calls_per_step": len(calls), "selector": os.path.basename(args.model),
                   "l2": "flushed before every timed call (read sweep of 256 MiB, clean lines), "
                         "then a ~100 us device spin so the call is enqueued before it starts",
                   "parallelism": (f"{world} GPUs: calls sharded by multi.schedule_units (large calls "
                                   "as nnz-balanced row panels, B replicated; the rest whole, LPT)")
                                  if world > 1 else "1 GPU"},
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "achieved": round(dom_ach, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(dom_ach / peak, 4), "traffic": traffic,
                     "peak_source": peak_kind,
                     # the DRAM bytes ncu measures for this call (profiles/ncu_traffic.json)
                     # moved in its measured time, as a fraction of the same peak
                     "traffic_frac": (round(traffic / (per_call_ms[dom] * 1e-3) / 1e9 / peak, 4)
                                      if traffic else None),
                     "scope": "dominant call (longest of the step): its algorithmic bytes "
                              "(4(M+1)+8nnz+4N*K_touched+4NM) / its mean CUDA-event time",
                     "dominant": {"call": _key(calls[dom]),
                                  "kernel": sk.KernelId.from_index(chosen[dom]).name(),
                                  "ms": round(per_call_ms[dom], 4),
                                  "algorithmic_bytes": calls[dom]["bytes"],
                                  "ceilings_us": _ceilings(calls[dom], traffic, peak)},
                     "suite_aggregate": {"achieved": round(achieved, 1),
                                         "frac": round(achieved / peak, 4),
                                         "scope": "sum algorithmic bytes / sum call time"}},
        "clocks": clk.summary(),
        "selected": {_key(c): sk.KernelId.from_index(k).name()
                     for c, k in zip(calls, chosen)},
        "per_call_ms": {_key(c): round(t, 5)
                        for c, t in zip(calls, per_call_ms)},
        "parity": parity,
        "warm_l2": warm,
        "da_spmm_overhead": overhead,
        "small_calls_batched": batched,
        "setup_cost": setup,
    }
    if assembly is not None:
        result["assembly"] = assembly
    if rank == 0 and not args.no_cusparse:
        result["cusparse"] = _cusparse_compare(calls, flush, per_call_ms, ns)
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = _cpu_baseline(
            mats, [int(n) for n in args.ns.split(",")] if args.ns else None)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _write_roofline_table(path, calls, per_call_ms, chosen, peak):
    """Per-call roofline table: algorithmic bytes and their HBM fraction, and the
    measured ceilings of _ceilings (L2 gather rate, L1 wavefronts); `bound` names the
    largest ceiling, `frac_bound` = that ceiling's time / the measured time."""
    from paper_2202_08556_b200 import spmmkit as sk

    lines = ["| call | kernel | us | algorithmic MB | GB/s | frac HBM | hbm us | l2_gather us "
             "| l1_wavefront us | bound | frac of bound |", "|" + "---|" * 11]
    for c, t, k in zip(calls, per_call_ms, chosen):
        ce = _ceilings(c, None, peak)
        cands = {n: v for n, v in ce.items() if v is not None}
        bname = max(cands, key=cands.get)
        us = t * 1e3
        gbs = c["bytes"] / (t * 1e-3) / 1e9
        lines.append(f'| {c["m"]["name"]}/N{c["n"]} | {sk.KernelId.from_index(k).name()} | '
                     f'{us:.1f} | {c["bytes"] / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.3f} | '
                     f'{ce["hbm"]} | {ce["l2_gather"]} | {ce["l1_wavefront"]} | {bname} | '
                     f'{cands[bname] / us:.2f} |')
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def _ceilings(c, traffic, peak):
    """Lower bounds on one call's time (us), each from a measured B200 rate:
    hbm        algorithmic bytes at the measured HBM copy bandwidth;
    dram       ncu-measured DRAM bytes of the launch (profiles/, B re-reads included) at
               the same bandwidth (null without a capture);
    l2_gather  nnz B-row gathers (4N bytes each, whole 32-B sectors) at the measured random
               L2->SM gather rate for that segment size (tools/gather_bw.cu,
               profiles/gather_bw_r01.json; footprint <= 50 MB);
    l1_wavefront  one L1 wavefront per (nonzero, 128-B line of its B row) at 1 per clock
               per SM (148 SMs x 1.965 GHz) - the LSU floor for small N."""
    import math

    nnz, n = c["d"].nnz(), c["n"]
    seg = max(32, 32 * math.ceil(4 * n / 32))
    rate = None
    try:
        with open(os.path.join(ROOT, "profiles", "gather_bw_r01.json")) as fh:
            g = json.load(fh)["gather"]
        small = [x for x in g if x["footprint_mb"] <= 60]
        best = [x for x in small if x["seg_bytes"] <= seg]
        pick = max(best, key=lambda x: x["seg_bytes"]) if best else min(small, key=lambda x: x["seg_bytes"])
        rate = pick["gbs"] * (seg / pick["seg_bytes"] if pick["seg_bytes"] < seg and pick["seg_bytes"] < 64 else 1.0)
    except Exception:
        pass
    out = {"hbm": round(c["bytes"] / (peak * 1e9) * 1e6, 1),
           "dram": round(traffic / (peak * 1e9) * 1e6, 1) if traffic else None,
           "l2_gather": round(nnz * seg / (rate * 1e9) * 1e6, 1) if rate else None,
           "l1_wavefront": round(nnz * math.ceil(4 * n / 128) / (148 * 1.965e9) * 1e6, 1)}
    return out


CUSPARSE_ALGS = ("DEFAULT", "CSR_ALG1", "CSR_ALG2", "CSR_ALG3", "COO_ALG1", "COO_ALG2",
                 "COO_ALG3", "COO_ALG4")


def _cusparse_compare(calls, flush, our_ms, ns, reps=5):
    """Best cuSPARSE SpMM per call over every CSR and COO algorithm with B and C
    row-major and column-major (PAPER.md:420's baseline set minus the blocked formats),
    on the same matrix, the same L2 flush before every timed run and the same statistic
    as our calls (mean of `reps` runs). Column-major operands are prepared outside the
    timed region; CSR_ALG3's preprocessing too (cmp_create)."""
    import torch

    from paper_2202_08556_b200 import build

    path = build.CUSPARSE_LIB
    if not os.path.exists(path):
        return None
    L = C.CDLL(path)
    L.cmp_create.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 5 + [C.c_int64] * 2 + \
        [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    L.cmp_run.argtypes = [C.c_void_p]
    L.cmp_destroy.argtypes = [C.c_void_p]
    stream = torch.cuda.current_stream()
    best, winner = [], []
    for c in calls:
        d = c["d"]
        rp, ci, va = d.device_arrays()
        rp_t = c["m"]["rp"]
        r0, r1 = c["rows"]
        lens = (rp_t[r0 + 1:r1 + 1] - rp_t[r0:r1]).to(torch.int64)
        coo = torch.repeat_interleave(torch.arange(d.num_rows, device=lens.device,
                                                   dtype=torch.int32), lens)
        n = c["n"]
        out = torch.empty_like(c["C"])
        Bcm = c["B"].t().contiguous()                      # N x K buffer = column-major K x N
        out_cm = torch.empty(n, d.num_rows, device=out.device)  # column-major M x N
        ts = {}
        for order in (0, 1):
            for alg in range(len(CUSPARSE_ALGS)):
                h = C.c_void_p()
                Bp, ldb = (c["B"].data_ptr(), n) if order == 0 else (Bcm.data_ptr(), d.num_cols)
                Cp, ldc = (out.data_ptr(), n) if order == 0 else (out_cm.data_ptr(), d.num_rows)
                if L.cmp_create(d.num_rows, d.num_cols, d.nnz(), rp, ci, coo.data_ptr(), va, Bp,
                                n, ldb, Cp, ldc, order, alg, stream.cuda_stream, C.byref(h)) != 0:
                    continue
                if L.cmp_run(h) != 0:
                    L.cmp_destroy(h)
                    continue
                torch.cuda.synchronize()
                tot = 0.0
                for _ in range(reps):
                    _flush(flush)
                    s = torch.cuda.Event(enable_timing=True)
                    e = torch.cuda.Event(enable_timing=True)
                    s.record(stream)
                    L.cmp_run(h)
                    e.record(stream)
                    torch.cuda.synchronize()
                    tot += s.elapsed_time(e)
                ts[(order, alg)] = tot / reps
                L.cmp_destroy(h)
        if ts:
            k = min(ts, key=ts.get)
            best.append(ts[k])
            winner.append(("row" if k[0] == 0 else "col") + ":" + CUSPARSE_ALGS[k[1]])
        else:
            best.append(float("nan"))
            winner.append(None)
        del Bcm, out_cm, out, coo
    tot_flops = sum(c["flops"] for c in calls)
    cus_ms = sum(best)
    speedups = [b / o for b, o in zip(best, our_ms) if o > 0]
    geo = float(statistics.geometric_mean(speedups)) if speedups else None
    by_n = {}
    for c, b, o in zip(calls, best, our_ms):
        by_n.setdefault(c["n"], []).append(b / o)
    wins = {}
    for w in winner:
        wins[w] = wins.get(w, 0) + 1
    return {"value": round(tot_flops / (cus_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "best_alg_per_call": True,
            "algorithms": [f"{o}:{a}" for o in ("row", "col") for a in CUSPARSE_ALGS],
            "statistic": f"mean of {reps} runs, L2 flushed before each (same as ours)",
            "ms_per_step": round(cus_ms, 4),
            "per_call_ms": {_key(c): round(b, 5)
                            for c, b in zip(calls, best)},
            "winner_per_call": {_key(c): w for c, w in zip(calls, winner)},
            "winner_counts": wins,
            "speedup_geomean": round(geo, 4) if geo else None,
            "speedup_geomean_by_N": {str(n): round(statistics.geometric_mean(v), 4)
                                     for n, v in sorted(by_n.items())}}


# ------------------------------------------------------------------ CPU reference
# Matrices above this many nonzeros are represented by a middle row panel of that size in
# the CPU arm (rows are independent in spmm, spmm.hpp:23-30, so a panel's GFLOP/s is the
# matrix's). It keeps c5 (503M nnz: ~75 GB of host CSR + X + Y) bounded; every matrix of
# the suite, c1, c3 and c4 runs whole.
REF_PANEL_NNZ = 150_000_000


def _ref_sample(mats, ns_override=None):
    """The CPU reference's unit of work: every (matrix, N) pair of the workload."""
    return [(m, n) for m in mats for n in (ns_override or m["ns"])]


def _ref_panel(m):
    import numpy as np

    rp = m["rp"].cpu().numpy().astype(np.int64)
    nnz = int(rp[-1])
    if nnz <= REF_PANEL_NNZ:
        return 0, m["M"]
    mid = np.searchsorted(rp, nnz // 2)
    r0 = int(np.searchsorted(rp, max(0, rp[mid] - REF_PANEL_NNZ // 2)))
    r1 = int(np.searchsorted(rp, min(nnz, rp[r0] + REF_PANEL_NNZ)))
    return r0, max(r1, r0 + 1)


REF_NAMES = ["RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR", "EB+RM+SR", "EB+RM+PR",
             "EB+CM+SR", "EB+CM+PR"]


class _RefArm:
    """The reference's own CPU path (oracle/_ref: its spmm(), P = all host cores, W = 8)
    over the workload, with the reference at its best: every (matrix, N) call runs the
    fastest of the reference's design points for it — the choice its data-aware flow
    (extract_features -> predict_kernel -> spmm) would make with a perfect CPU-trained
    selector (the reference ships no trained model). The choice is made once, by timing
    every design point on the call (CM points only for N <= 16, where column-major
    locality can pay; they need X column-major, laid out once like RM's). Reference CSR
    handles (int64) and X operands are built once, as time_kernel does (bench.hpp:
    125-137); one pass = one spmm() call per pair, each timed alone (wall clock around
    exactly the call, result dropped)."""

    def __init__(self, mats, ns_override=None, select: bool = True):
        import numpy as np

        from oracle import oracle as O

        self.R = O.ref()
        self.cores = os.cpu_count() or 1
        self.handles, self.dense, self.pairs = {}, [], []
        self.panelled = []
        self.choice, self.times, self.nnz, self.rm = [], [], [], []
        if self.R is None:
            return
        R = self.R
        secs = C.c_double()
        for m, n in _ref_sample(mats, ns_override):
            if m["name"] not in self.handles:
                r0, r1 = _ref_panel(m)
                if (r0, r1) != (0, m["M"]):
                    self.panelled.append(m["name"])
                rp = m["rp"].cpu().numpy().astype(np.int64)
                s, e = int(rp[r0]), int(rp[r1])
                ci = m["ci"][s:e].cpu().numpy().astype(np.int64)
                va = m["va"][s:e].cpu().numpy().astype(np.float64)
                self.handles[m["name"]] = (R.ref_csr_from_csr(r1 - r0, m["K"], rp[r0:r1 + 1] - s,
                                                              ci, va), e - s)
                del rp, ci, va
            h, nnz = self.handles[m["name"]]
            x = np.random.default_rng(n).uniform(-1, 1, (m["K"], n)).astype(np.float32)
            d_rm = R.ref_dense_f32(x.reshape(-1), m["K"], n, 0)
            self.dense.append(d_rm)
            d_cm = None
            if select and n <= 16:
                d_cm = R.ref_dense_f32(np.ascontiguousarray(x.T).reshape(-1), m["K"], n, 1)
                self.dense.append(d_cm)
            del x
            best, best_t = 0, float("inf")
            times = [None] * 8
            for k in (range(8) if select else (0,)):
                dk = d_cm if (k >> 1) & 1 else d_rm
                if dk is None:
                    continue
                if R.ref_time_spmm_once_f32(h, dk, k, self.cores, 8, 8, C.byref(secs)):
                    raise RuntimeError(R.ref_last_error().decode())
                times[k] = secs.value
                if secs.value < best_t:
                    best, best_t = k, secs.value
            self.times.append(times)
            self.nnz.append(nnz)
            self.choice.append(best)
            self.rm.append(d_rm)
            self.pairs.append((h, d_cm if (best >> 1) & 1 else d_rm, best, 2 * nnz * n))
        self.flops = sum(f for *_, f in self.pairs)

    def one_pass(self) -> float:
        """Seconds of reference spmm() time for one pass over the workload."""
        secs = C.c_double()
        tot = 0.0
        for h, d, k, _ in self.pairs:
            if self.R.ref_time_spmm_once_f32(h, d, k, self.cores, 8, 8, C.byref(secs)):
                raise RuntimeError(self.R.ref_last_error().decode())
            tot += secs.value
        return tot

    def per_kernel(self):
        """GFLOP/s of each reference design point over the calls it was timed on (one
        run per call at P = all host threads; CM points on N <= 16 only)."""
        out = {}
        for k in range(8):
            fl = sum(f for (*_, f), t in zip(self.pairs, self.times) if t[k] is not None)
            tt = sum(t[k] for t in self.times if t[k] is not None)
            n = sum(1 for t in self.times if t[k] is not None)
            if n:
                out[REF_NAMES[k]] = {"gflops": round(fl / tt / 1e9, 3), "calls": n}
        return out

    def single_thread(self, max_nnz=3_000_000):
        """P = 1 on the calls of matrices up to max_nnz (the 2^14- and 2^17-row ones): the
        chosen design point (one run each) and the serial spmm_reference (the reference's
        time_kernel_fn, reps 3)."""
        secs = C.c_double()
        med, mn, ck = C.c_double(), C.c_double(), C.c_double()
        fl = t_best = t_ref = 0.0
        n = 0
        for (h, d, k, f), nnz in zip(self.pairs, self.nnz):
            if nnz > max_nnz:
                continue
            if self.R.ref_time_spmm_once_f32(h, d, k, 1, 8, 8, C.byref(secs)):
                raise RuntimeError(self.R.ref_last_error().decode())
            t_best += secs.value
            n += 1
            fl += f
        # spmm_reference needs its X row-major: the RM operand of each pair
        for (h, d, k, f), nnz, x_rm in zip(self.pairs, self.nnz, self.rm):
            if nnz > max_nnz:
                continue
            if self.R.ref_time_spmm_dense_reference_f32(h, x_rm, C.byref(secs)):
                raise RuntimeError(self.R.ref_last_error().decode())
            t_ref += secs.value
        if not n:
            return None
        return {"calls": n, "best_point_gflops": round(fl / t_best / 1e9, 3),
                "spmm_reference_gflops": round(fl / t_ref / 1e9, 3) if t_ref else None}

    def choices(self):
        out = {}
        for k in self.choice:
            out[REF_NAMES[k]] = out.get(REF_NAMES[k], 0) + 1
        return out

    def close(self):
        if self.R is None:
            return
        for d in self.dense:
            self.R.ref_dense_free(d)
        for h, _ in self.handles.values():
            self.R.ref_csr_free(h)
        self.dense, self.handles = [], {}


def _cpu_baseline(mats, ns_override=None, passes=3):
    arm = _RefArm(mats, ns_override)
    if arm.R is None:
        return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    arm.one_pass()  # warm-up (first touch of X, the pool's threads)
    secs = sorted(arm.one_pass() for _ in range(passes))[passes // 2]
    v = arm.flops / secs / 1e9
    per_kernel = arm.per_kernel()
    p1 = arm.single_thread()
    arm.close()
    whole = "every matrix whole" if not arm.panelled else \
        f"{', '.join(arm.panelled)} as a middle row panel of {REF_PANEL_NNZ} nnz"
    return {"value": round(v, 4), "unit": "GFLOP/s", "cores": arm.cores, "kind": "reference",
            "sample": f"reference spmm() fp32, P={arm.cores} threads, each of the "
                      f"{len(arm.pairs)} (matrix, N) calls of the workload on its fastest "
                      f"reference design point ({whole}); median of {passes} passes of "
                      f"{secs:.2f} s",
            "kernels": arm.choices(), "per_kernel_all_threads": per_kernel,
            "single_thread_s14_s17": p1, "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """--impl reference: the reference CPU implementation alone (rank 0): every step is one
    pass of the reference's spmm() over the same workload as our arm's step."""
    world, rank, local = _dist()
    if rank != 0:
        return
    import torch

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    if dev == "cuda":
        torch.cuda.set_device(local)
    from paper_2202_08556_b200 import gen

    mats = []
    for name, mk, wns in gen.workload(args.workload, small=args.small, device=dev):
        M, K, rp, ci, va = mk()
        mats.append(dict(name=name, M=M, K=K, nnz_total=int(ci.numel()), rp=rp, ci=ci, va=va,
                         ns=wns))
    ns_override = [int(n) for n in args.ns.split(",")] if args.ns else None
    ns = sorted({n for m in mats for n in (ns_override or m["ns"])})
    arm = _RefArm(mats, ns_override)
    if arm.R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built here"}))
        return
    for m in mats:  # generated operands are no longer needed on the device
        m["rp"] = m["ci"] = m["va"] = None
    for _ in range(args.warmup):
        arm.one_pass()
    step_s = [arm.one_pass() for _ in range(max(args.steps, 1))]
    secs = statistics.median(step_s)
    value = arm.flops / secs / 1e9
    whole = "every matrix whole" if not arm.panelled else \
        f"{', '.join(arm.panelled)} as a middle row panel of {REF_PANEL_NNZ} nnz"
    arm.close()
    out = {"impl": "reference",
           "metric": "SpMM GFLOP/s (2*nnz*N/t), DA-SpMM over the synthetic suite",
           "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic",
           "config": {"workload": f"{args.workload} (reference CPU, {whole})", "ns": ns,
                      "calls_per_step": len(arm.pairs)},
           "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": arm.cores,
                            "kind": "reference",
                            "sample": f"reference spmm() fp32, P={arm.cores} threads, one pass "
                                      f"over {len(arm.pairs)} (matrix, N) calls per step, each on "
                                      f"its fastest reference design point ({whole}), median "
                                      f"over steps",
                            "kernels": arm.choices()}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default=os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                                    "b200_selector.txt"))
    ap.add_argument("--small", action="store_true", help="2^14 and 2^17 matrices only")
    ap.add_argument("--workload", default="suite", choices=["suite", "c1", "c3", "c4", "c5"],
                    help="BASELINE.json config (default: configs[1] suite, the headline)")
    ap.add_argument("--ns", default="")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cusparse", action="store_true")
    ap.add_argument("--profile-step", action="store_true",
                    help="only the warm-up and the timed steps (for ncu launch lists); "
                         "implies --no-cpu --no-cusparse")
    ap.add_argument("--roofline-table", default="",
                    help="also write a per-call roofline table (markdown) to this path")
    args = ap.parse_args()
    if args.profile_step:
        args.no_cpu = args.no_cusparse = True
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
