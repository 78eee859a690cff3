"""Summarise ncu outputs of one gpurun call into a markdown table for profiles/.

  python tools/ncu_summary.py gpurun_out/<tag> [--launches-per-step N] > profiles/<round>_ncu_<tag>.md

Reads <dir>/launches.csv (gpu__time_duration.sum per launch; the LAST N
launches are one relay step) and every <dir>/full_*.ncu-rep (--set full).
"""
import collections
import csv
import glob
import io
import os
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
]


def launches(path, per_step):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(lines)
    h = next(r)
    rows = list(r)
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    last = rows[-per_step:] if per_step else rows
    agg = collections.defaultdict(lambda: [0, 0.0])
    for x in last:
        name = x[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "").split("<")[0]
        agg[name][0] += 1
        agg[name][1] += float(x[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    out = ["| kernel | launches | time (us, ncu cold-cache serialised) | share |", "|---|---|---|---|"]
    for n, (c, v) in sorted(agg.items(), key=lambda t: -t[1][1]):
        out.append(f"| {n} | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    out.append(f"| **total** | {len(last)} | {tot / 1e3:.1f} | |")
    return "\n".join(out)


def full(path):
    p = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    r = list(csv.reader(io.StringIO(p.stdout)))
    if len(r) < 3:
        return f"(no data in {os.path.basename(path)})"
    h, units, data = r[0], r[1], r[2:]
    name_i = h.index("Kernel Name")
    cols = []
    for key, label in RAW:
        if key in h:
            cols.append((h.index(key), label, units[h.index(key)]))
    out = ["| launch | " + " | ".join(f"{l} ({u})" if u else l for _, l, u in cols) + " |",
           "|---" * (len(cols) + 1) + "|"]
    for i, x in enumerate(data):
        out.append(f"| {x[name_i].split('(')[0][-40:]} #{i} | " + " | ".join(x[c] for c, _, _ in cols) + " |")
    return "\n".join(out)


def main():
    d = sys.argv[1]
    per_step = 0
    if "--launches-per-step" in sys.argv:
        per_step = int(sys.argv[sys.argv.index("--launches-per-step") + 1])
    print(f"# ncu summary: {d}\n")
    lp = os.path.join(d, "launches.csv")
    if os.path.exists(lp):
        print(f"## Launch list of one relay step (last {per_step or 'all'} launches)\n")
        print(launches(lp, per_step))
        print()
    for f in sorted(glob.glob(os.path.join(d, "full_*.ncu-rep"))):
        print(f"## `ncu --set full`: {os.path.basename(f)}\n")
        print(full(f))
        print()


if __name__ == "__main__":
    main()
