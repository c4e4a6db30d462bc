"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel
family: launches, total time and share.

python tools/launch_summary.py launches.csv [--ours] [--step]
  --ours  only this library's kernels
  --step  only the kernels an SpMM call launches (design-point kernels, EB prologues,
          the selector), not handle creation / lazy set-up (features, column windows,
          COO row ids, tiles, the exact std_row replay)"""
import csv
import io
import re
import sys
from collections import defaultdict


def main():
    raw = open(sys.argv[1]).read()
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        fam = re.sub(r"\(.*", "", name)
        fam = re.sub(r"^void ", "", fam)
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3}.get(unit.strip(), 1.0)
        agg[fam][0] += 1
        agg[fam][1] += v * scale
    if "--ours" in sys.argv or "--step" in sys.argv:  # only this library's kernels
        agg = {k: v for k, v in agg.items() if k.startswith("daspmm::")}
    if "--step" in sys.argv:
        setup = ("k_row_terms", "k_cols_touched", "k_popcount", "k_fine_spans", "k_coo_rows",
                 "k_tile_spans", "k_tile_fill", "k_std_sequential", "k_ingest", "k_rebase",
                 "k_rows_unsorted", "k_tile_windows", "k_spans_init")
        agg = {k: v for k, v in agg.items() if not any(f"::{n}" in k for n in setup)}
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for fam, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{fam[:70]:70s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    main()
