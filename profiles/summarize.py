"""Summarise ncu outputs into markdown: launch-list shares and key --set full metrics.

    python profiles/summarize.py launches <launches.csv>
    python profiles/summarize.py full <report.ncu-rep>
"""

import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
            agg[r[ki].split("(")[0][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "Block Size", "Grid Size",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Executed Instructions",
        "Dynamic Shared Memory Per Block"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seen = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] in WANT:
            seen.setdefault((r[ki].split("(")[0][:60], r[mi]), f"{r[vi]} {r[ui]}".strip())
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if rr:
        hh = rr[0]
        cols = [c for c in hh if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")]
        for r in rr[2:]:
            name = r[hh.index("Kernel Name")].split("(")[0][:60]
            for c in cols:
                seen.setdefault((name, c), f"{r[hh.index(c)]} {rr[1][hh.index(c)]}")
    kernels = list(dict.fromkeys(k for k, _ in seen))
    for k in kernels:
        print(f"### `{k}`\n")
        print("| metric | value |\n|---|---|")
        for (kk, m), v in seen.items():
            if kk == k:
                print(f"| {m} | {v} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
