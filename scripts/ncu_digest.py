"""Digest an ncu --set full report on the GPU box (reports are too large to bring back):
writes <out>.md (headline metrics + stall reasons, as ncu_summary.py full) and
<out>.sass.txt (the 40 SASS instructions with the most stall samples, with execution
counts, and the share of samples / instructions per 32-instruction block).
Usage: python scripts/ncu_digest.py REPORT.ncu-rep OUT_PREFIX
"""
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402


def sass(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ia, isrc = h.index("Address"), h.index("Source")
    ism, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot_s = sum(f(r[ism]) for r in data if len(r) > ism) or 1.0
    tot_e = sum(f(r[iex]) for r in data if len(r) > iex) or 1.0
    lines = [f"# SASS hot spots: {os.path.basename(rep)} ({len(data)} instructions, "
             f"{tot_s:.0f} samples, {tot_e:.3e} warp instructions)", "", "## top instructions by stall samples"]
    top = sorted(range(len(data)), key=lambda i: -f(data[i][ism]))[:40]
    for i in sorted(top):
        r = data[i]
        lines.append(f"{i:6d} {r[ia][-6:]} smp {100 * f(r[ism]) / tot_s:5.2f}% exe {100 * f(r[iex]) / tot_e:5.2f}% "
                     f"n={r[iex]:>12}  {r[isrc][:90]}")
    lines += ["", "## 32-instruction blocks with >= 1% of samples or instructions"]
    for b in range(0, len(data), 32):
        s = sum(f(r[ism]) for r in data[b:b + 32]) / tot_s
        e = sum(f(r[iex]) for r in data[b:b + 32]) / tot_e
        if s >= 0.01 or e >= 0.01:
            lines.append(f"block {b // 32:5d} @{data[b][ia][-6:]}  samples {100 * s:5.1f}%  instructions {100 * e:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    rep, prefix = sys.argv[1], sys.argv[2]
    ncu_summary.full(rep, prefix + ".md")
    sass(rep, prefix + ".sass.txt")
