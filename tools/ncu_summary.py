"""Summarise an ncu --set full report: key throughput metrics, stall reasons and the
hottest source lines. python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--lines 12]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    path = sys.argv[1]
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 12
    h, u, vals = raw(path)
    for v in vals:
        print("-" * 100)
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:62s} {v[i]:>24s} {u[i]}")
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("stalls/issue:", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    try:
        rows = list(csv.reader(io.StringIO(src)))
        hdr = None
        for i, r in enumerate(rows):
            if "Source" in r and any(c.startswith("Warp Stall Sampling") for c in r):
                hdr = i
                break
        if hdr is None:
            return
        H = rows[hdr]
        si = H.index("Source")
        cols = [j for j, c in enumerate(H) if c.startswith("Warp Stall Sampling (All")]
        if not cols:
            return
        ci = cols[0]
        body = [r for r in rows[hdr + 1:] if len(r) > ci and r[ci].replace(".", "").isdigit()]
        body.sort(key=lambda r: -float(r[ci]))
        tot = sum(float(r[ci]) for r in body) or 1.0
        print(f"top SASS by warp-stall samples ({H[ci]}):")
        for r in body[:nlines]:
            print(f"  {100*float(r[ci])/tot:5.1f}%  {r[si].strip()[:110]}")
    except Exception as e:  # source page layout differs across ncu versions
        print("source page unavailable:", e)


if __name__ == "__main__":
    main()
