"""Summarise an ncu source page (SASS) by execution-count blocks: samples, stall reasons."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
show = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
if kfilter:
    cmd += ["-k", f"regex:{kfilter}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
stc = [k for k in h if k.startswith("stall_") and "Not" not in k]
f = lambda r, k: float(r[idx[k]] or 0)
c = collections.Counter(); st = collections.Counter(); ins = collections.Counter()
for r in data:
    e = int(f(r, "Instructions Executed"))
    c[e] += 1; st[e] += f(r, "Warp Stall Sampling (All Samples)"); ins[e] += e
tot = sum(st.values())
print("instructions", sum(ins.values()), "samples", tot)
print("| exec count | #instr | instr executed | samples | share | top stalls |")
print("|---|---|---|---|---|---|")
for e, v in sorted(st.items(), key=lambda x: -x[1])[:12]:
    agg = collections.Counter()
    for r in data:
        if int(f(r, "Instructions Executed")) == e:
            for k in stc:
                agg[k] += f(r, k)
    tops = ", ".join(f"{k[6:]} {int(x)}" for k, x in agg.most_common(3))
    print(f"| {e} | {c[e]} | {ins[e]} | {int(v)} | {100*v/tot:.1f}% | {tops} |")
if show:
    for r in data:
        if int(f(r, "Instructions Executed")) == show:
            top = max(stc, key=lambda k: f(r, k))
            print(int(f(r, "Warp Stall Sampling (All Samples)")), r[idx["Source"]][:72], top[6:])
