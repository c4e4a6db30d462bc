"""Controlled one-factor experiments on the B200: CLI over
paper_2202_08556_b200.controlled (the reference's controlled.hpp:123-189 and acceptance
criterion 7, acceptance_test.cpp:391-483).

python tools/controlled.py [--out profiles/r02_controlled.csv] [--scale 20] [--reps 7]
"""
import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_08556_b200 import controlled as ce  # noqa: E402

trend_verdict = ce.trend_verdict  # kept for callers of the round-1 tool


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/controlled.csv")
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    timer = ce._Timer()
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["experiment", "varied_name", "varied", "time_a_s", "time_b_s", "ratio_name",
                    "ratio", "verdict"])
        for d in ce.ControlledDimension:
            t = ce.run_controlled(ce.b200_spec(d, a.scale, a.reps), timer)
            for r in t.rows:
                w.writerow([ce.dimension_name(d), t.varied_name, f"{r.varied:.6g}",
                            f"{r.time_a:.6g}", f"{r.time_b:.6g}", t.ratio_name,
                            f"{r.ratio:.4g}", t.verdict])
            print(ce.dimension_name(d), t.verdict, [round(r.ratio, 3) for r in t.rows], flush=True)


if __name__ == "__main__":
    main()
