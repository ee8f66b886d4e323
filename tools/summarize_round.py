"""Summaries of a round profile capture (tools/profile_round.sh R) for profiles/:
    python tools/summarize_round.py R
reads gpurun_out/R_* and writes profiles/R_launches.md, R_plr_launches.md,
R_ncu_full.md, R_ncu_full_large.md, R_ncu_full_plr_update.md, R_traffic.json and copies
the bench / reference / bandwidth lines."""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r2x"
G = "gpurun_out"
P = os.environ.get("AMZ_PROFILES_DIR", "profiles")


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("amz::", "").replace("at::", "").replace("(anonymous namespace)::", "")
    return name[:70]


def launch_csv(path):
    """rows of an ncu --csv --log-file launch list (metric gpu__time_duration.sum etc.)."""
    if not os.path.exists(path):
        return []
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    if not rows:
        return []
    h = rows[0]
    return [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]


def launches_md(path, title):
    rows = [r for r in launch_csv(path) if r.get("Metric Name") == "gpu__time_duration.sum"]
    if not rows:
        return ""
    agg = {}
    for r in rows:
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
        if r["Metric Unit"] == "ms":
            v = float(r["Metric Value"]) * 1e3
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + v)
    tot = sum(t for _, t in agg.values())
    out = [f"### {title}", "", f"source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none; "
           "cold-cache, serialised launches: compare shares, not absolutes)", "",
           "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t / n:.2f} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(out) + "\n"


METRICS = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "Executed Ipc Active",
           "Issue Slots Busy", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Instructions",
           "Block Size", "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
           "Static Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]


def ncu_rows(rep, page):
    if not os.path.exists(rep):
        return []
    try:
        txt = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True,
                             timeout=600).stdout
    except Exception:
        return []
    lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    return rows


def full_md(rep, title):
    det = ncu_rows(rep, "details")
    raw = ncu_rows(rep, "raw")
    if not det:
        return "", {}
    h = det[0]
    ix = {k: i for i, k in enumerate(h)}
    per = {}
    order = []
    for r in det[1:]:
        if len(r) < ix["Metric Value"] + 1:
            continue
        key = (r[ix["ID"]], short(r[ix["Kernel Name"]]))
        if key not in per:
            per[key] = {}
            order.append(key)
        name = r[ix["Metric Name"]]
        if name in METRICS and name not in per[key]:
            per[key][name] = f'{r[ix["Metric Value"]]} {r[ix["Metric Unit"]]}'.strip()
    traffic = {}
    if raw:
        hr = raw[0]
        jx = {k: i for i, k in enumerate(hr)}
        for r in raw[2:]:
            if len(r) != len(hr):
                continue
            key = (r[jx["ID"]], short(r[jx["Kernel Name"]]))
            if key in per:
                for m in RAW:
                    if m in jx:
                        per[key][m] = r[jx[m]] + " " + raw[1][jx[m]]
                try:
                    rd = float(r[jx["dram__bytes_read.sum"]].replace(",", ""))
                    wr = float(r[jx["dram__bytes_write.sum"]].replace(",", ""))
                    unit = raw[1][jx["dram__bytes_read.sum"]]
                    unit_w = raw[1][jx["dram__bytes_write.sum"]]
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                    us = float(r[jx["gpu__time_duration.sum"]].replace(",", ""))
                    tu = raw[1][jx["gpu__time_duration.sum"]]
                    us = us / 1e3 if tu in ("nsecond", "ns") else (us * 1e3 if tu in ("msecond", "ms") else us)
                    traffic[key] = {"read": int(rd * scale.get(unit, 1)), "write": int(wr * scale.get(unit_w, 1)),
                                    "us": round(us, 2)}
                except (KeyError, ValueError):
                    pass
    out = [f"## {title}", "", f"source: `{rep}` (ncu --set full --clock-control none --import-source on)", ""]
    for key in order:
        out += [f"### `{key[1]}` (launch id {key[0]})", "", "| metric | value |", "|---|---|"]
        for m in METRICS + RAW:
            if m in per[key]:
                out.append(f"| {m} | {per[key][m]} |")
        out.append("")
    return "\n".join(out) + "\n", traffic


def main():
    os.makedirs(P, exist_ok=True)
    for suf in ("bench.json", "bench_ref.json", "bw.json"):
        src = f"{G}/{R}_{suf}"
        if os.path.exists(src) and os.path.getsize(src):
            shutil.copy(src, f"{P}/{R}_{suf}")
    md = launches_md(f"{G}/{R}_launches.csv", f"{R}: configs[1] bench step (bench.py --steps 3 --warmup 3)")
    md += "\n" + launches_md(f"{G}/{R}_large_launches.csv", f"{R}: 65536 x 256 rollout (tools/rollout_large.py)")
    open(f"{P}/{R}_launches.md", "w").write(md)
    pl = ""
    for m in ("plr_2048", "accel_2048", "plr_16384"):
        pl += launches_md(f"{G}/{R}_plr_{m}.csv", f"{R}: tools/plr_profile.py {m.replace('_', ' ')} (8 iterations)") + "\n"
    open(f"{P}/{R}_plr_launches.md", "w").write(pl)
    traffic = {}
    for rep, name, title in ((f"{G}/{R}_full.ncu-rep", "ncu_full", "configs[1] step kernels"),
                             (f"{G}/{R}_large_full.ncu-rep", "ncu_full_large", "65536 x 256 rollout kernels"),
                             (f"{G}/{R}_plr_update_full.ncu-rep", "ncu_full_plr_update", "PLR|| 2048 buffer update")):
        text, tr = full_md(rep, title)
        if text:
            open(f"{P}/{R}_{name}.md", "w").write(text)
        traffic[name] = {f"{k[1]} #{k[0]}": v for k, v in tr.items()}
    json.dump(traffic, open(f"{P}/{R}_traffic_raw.json", "w"), indent=1)
    # the per-launch DRAM traffic bench.py reports as roofline.traffic
    out = {"source": f"ncu --set full ({G}/{R}_full.ncu-rep: bench.py config 2; {R}_large_full.ncu-rep: "
                     "tools/rollout_large.py 65536), dram__bytes_read.sum + dram__bytes_write.sum per launch"}

    def pick(group, pat):
        for k, v in traffic.get(group, {}).items():
            if re.search(pat, k):
                return k.rsplit(" #", 1)[0], v
        return None, None

    for key, group, cfg, alg, pats in (
            ("k_env_rollout", "ncu_full", "configs[1] 4096 x 256", 36 * 4096 * 256, (r"k_dyn<", r"k_render")),
            ("large_batch_rollout", "ncu_full_large", "65536 x 256", 36 * 65536 * 256, (r"k_dyn<", r"k_render"))):
        ks = {}
        for pat in pats:
            name, v = pick(group, pat)
            if name:
                ks[name] = v
        if ks:
            out[key] = {"config": cfg, "kernels": ks, "dram_bytes": sum(v["read"] + v["write"] for v in ks.values()),
                        "algorithmic_bytes": alg}
    name, v = pick("ncu_full", r"k_gae_score")
    if name:
        out["k_gae_score4"] = dict(v, config="configs[1]", algorithmic_bytes=33 * 4096 * 256, kernel=name)
    json.dump(out, open(f"{P}/{R}_traffic.json", "w"), indent=1)
    print("wrote", sorted(f for f in os.listdir(P) if f.startswith(R)))


if __name__ == "__main__":
    main()
