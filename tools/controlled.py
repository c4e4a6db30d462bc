"""Controlled one-factor experiments on the B200 (the reference's
controlled.hpp:123-189 and acceptance criterion 7, acceptance_test.cpp:391-483).

Each experiment varies one input property and races the two kernels that differ only in
the matching loop choice, the other two pinned to RB / RM / SR (controlled.hpp:132-150):

  rb-eb  skew (R-MAT a = 0.25 .. 0.7, size and nnz fixed) -> varied = std_row,
         ratio = t(RB+RM+SR) / t(EB+RM+SR)
  rm-cm  N (matrix fixed)                                 -> ratio = t(RB+CM+SR) / t(RB+RM+SR)
  sr-pr  nnz (scale, skew and N fixed)                    -> ratio = t(RB+RM+PR) / t(RB+RM+SR)

Rising ratios mean the contrast kernel gains as the property grows. Rows report the
minimum over reps (controlled.hpp:165-170); the verdict is the reference's
trend_verdict (controlled.hpp:60-71). Sizes are B200-scale (2^20 rows) instead of the
reference's CPU-scale 2^8.

python tools/controlled.py [--out profiles/r01_controlled.csv] [--scale 20]
"""
import argparse
import csv
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402


def trend_verdict(ratios, tau=0.10):
    """controlled.hpp:60-71: a step counts as movement only outside a +-tau band."""
    if len(ratios) < 2:
        return "flat"
    up = down = False
    for prev, cur in zip(ratios, ratios[1:]):
        if cur > prev * (1 + tau):
            up = True
        elif cur < prev * (1 - tau):
            down = True
    return "mixed" if up and down else "rising" if up else "falling" if down else "flat"


def min_time(fn, flush, reps):
    for _ in range(2):
        fn()
    best = float("inf")
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    return best


def run(kind, scale, reps, flush):
    deg = 16
    nnz = deg << scale
    if kind == "rb-eb":
        points = [(a, 8, nnz) for a in (0.25, 0.45, 0.57, 0.70)]
        ka, kb = 0, 4
    elif kind == "rm-cm":
        points = [(0.45, n, nnz) for n in (2, 8, 32, 128)]
        ka, kb = 0, 2
    else:
        points = [(0.45, 8, z) for z in (nnz // 8, nnz // 4, nnz // 2, nnz)]
        ka, kb = 0, 1
    rows = []
    for a, n, z in points:
        b = c = d = (1.0 - a) / 3.0
        M, K, rp, ci, va = gen.rmat(scale, z, a, b, c, d, seed=31)
        dcsr = sk.DeviceCsr.from_device(M, K, rp, ci, va)
        f = sk.extract_features(dcsr, n)
        B = gen.dense_operand(K, n, seed=7321 ^ n)
        Bcm = B.t().contiguous()
        C = torch.empty(M, n, device="cuda")
        ta = min_time(lambda: sk.spmm_device(ka, dcsr, Bcm if ka & 2 else B, C), flush, reps)
        tb = min_time(lambda: sk.spmm_device(kb, dcsr, Bcm if kb & 2 else B, C), flush, reps)
        varied = f.std_row if kind == "rb-eb" else (n if kind == "rm-cm" else ci.numel())
        ratio = ta / tb if kind == "rb-eb" else tb / ta
        rows.append(dict(varied=varied, time_a_s=ta, time_b_s=tb, ratio=ratio))
        del dcsr, rp, ci, va
        torch.cuda.empty_cache()
    verdict = trend_verdict([r["ratio"] for r in rows])
    return rows, verdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/controlled.csv")
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    names = {"rb-eb": ("std_row", "rb_over_eb"), "rm-cm": ("n_cols", "cm_over_rm"),
             "sr-pr": ("nnz", "pr_over_sr")}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["experiment", "varied_name", "varied", "time_a_s", "time_b_s", "ratio_name",
                    "ratio", "verdict"])
        for kind in ("rb-eb", "rm-cm", "sr-pr"):
            rows, verdict = run(kind, a.scale, a.reps, flush)
            for r in rows:
                w.writerow([kind, names[kind][0], f"{r['varied']:.6g}", f"{r['time_a_s']:.6g}",
                            f"{r['time_b_s']:.6g}", names[kind][1], f"{r['ratio']:.4g}", verdict])
            print(kind, verdict, [round(r["ratio"], 3) for r in rows], flush=True)


if __name__ == "__main__":
    main()
