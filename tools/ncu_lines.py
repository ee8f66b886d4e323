"""Per-source-line instruction counts and stall samples from an ncu report (ncu -i ...
--page source --print-source cuda,sass --csv).  Usage: ncu_lines.py REP [kernel-regex] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"]
if kre:
    cmd += ["-k", f"regex:{kre}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "-" and r[0].isdigit():
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            rows.append((fname, int(r[0]), r[1][:90], float(r[ie] or 0), float(r[sm] or 0)))
        except ValueError:
            pass
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total instr {ti:.0f} samples {ts:.0f}")
for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{f}:{ln:<4} ins {100*ins/ti:5.1f}%  smp {100*smp/ts:5.1f}%  {src.strip()}")
