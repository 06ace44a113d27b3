"""Summarise ncu output into small committed files under profiles/.

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, total device time and share (cold-cache,
      serialised: compare SHARES, not absolutes)
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md>
      headline metrics + stall reasons of the captured kernel
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list summary: {path.split('/')[-1]}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: shares, not absolutes)",
             "", "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {ms:.2f} | {ms / tot:.3f} |")
    lines.append(f"| **total** | {sum(a[0] for a in agg.values())} | {tot:.2f} | 1.000 |")
    open(out, "w").write("\n".join(lines) + "\n")


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "lts__t_requests_op_atom.sum", "lts__t_requests_op_red.sum"]
    lines = [f"# ncu --set full summary: {path.split('/')[-1]}", "", "| metric | value | unit |", "|---|---|---|"]
    for k in keys:
        if k in d:
            lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
    st = []
    for k, v in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    lines += ["", "| stall reason (pc samples) | share |", "|---|---:|"]
    for v, k in sorted(st, reverse=True)[:10]:
        lines.append(f"| {k} | {v / tot:.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
