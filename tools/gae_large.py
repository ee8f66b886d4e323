"""GAE + MaxMC/PVL timing at HBM-sized batches for one kernel selection (set by the
AMZ_GAE_KERNEL / AMZ_GAE_M / AMZ_GAE_U env vars, read once per process).  Prints one
JSON line per batch size with the device time, algorithmic GB/s and an output digest
(so runs with different kernels can be compared bit for bit)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

T = 256
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6552.0) if os.path.exists("MEASURED_PEAKS.json") else 6552.0


def digest(*xs):
    h = 0
    for x in xs:
        h ^= int(x.contiguous().view(torch.int64).sum().item()) & ((1 << 63) - 1)
    return h


flush = torch.empty(32 << 20, dtype=torch.int64, device="cuda")
for B in [int(b) for b in (sys.argv[1:] or ["16384", "65536", "262144"])]:
    g = torch.Generator(device="cuda")
    g.manual_seed(B)
    r = (torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64) < 0.01).double()
    v = torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64)
    if os.environ.get("GAE_V32"):  # the policy's float32 values (gae_and_scores' f32 entry)
        v = v.float()
    d = torch.rand((T, B), generator=g, device="cuda") < 0.01
    last = torch.rand((B,), generator=g, device="cuda", dtype=torch.float64).to(v.dtype)
    res = {}
    for fn in ("maxmc", "pvl"):
        ts = []
        for it in range(6):
            flush.fill_(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            o = amz.gae_and_scores(r, v, d, last, 0.995, 0.95, score_fn=fn)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = sum(ts) / len(ts)
        gbs = (29 if v.dtype == torch.float32 else 33) * B * T / (ms * 1e-3) / 1e9
        res[fn] = {"ms": round(ms, 4), "GBs": round(gbs, 1), "frac": round(gbs / peak, 3),
                   "digest": digest(*[x for x in o.values() if torch.is_tensor(x)])}
    print(json.dumps({"B": B, "kernel": os.environ.get("AMZ_GAE_KERNEL", "0"), "m": os.environ.get("AMZ_GAE_M"),
                      "v32": bool(os.environ.get("GAE_V32")), **res}), flush=True)
