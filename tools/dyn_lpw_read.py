import csv, sys
for l in sys.argv[1:]:
    rows = list(csv.reader(open(f"gpurun_out/lrm_{l}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    v = [(r[ki][:14], float(r[vi]) / 1000) for r in rows[hi + 1:]]
    dyn = [x for k, x in v if "k_dyn" in k]
    sp = [x for k, x in v if "spec" in k]
    print("LPW", l, "home dyn us", sorted(dyn[:8])[4], "resample dyn us", sorted(dyn[8:])[4], "spec", sorted(sp)[len(sp) // 2])
