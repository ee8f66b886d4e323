"""Large-batch (HBM-sized) DR reset + RESAMPLE rollout, the roofline point of the env
step: ``python tools/rollout_large.py [B] [iters]``.  Prints one JSON line with the
rollout's device time and algorithmic GB/s (36 B per env-step); run under
ncu with ``-k regex:"k_dyn|k_render"`` to capture the launches."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_12716_b200 as amz  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
T = 256
p = amz.StaticParams()
env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, B), generator=g, dtype=torch.uint8, device="cuda")
flush = torch.empty(32 << 20, dtype=torch.int64, device="cuda")
ts = []
for i in range(iters):
    res = env.reset(amz.RngStream.from_seed(i), p)
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tr, cur = amz.rollout_actions(env, res, acts, p)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts[1:])[len(ts[1:]) // 2] if len(ts) > 1 else ts[0]
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6552.0) if os.path.exists("MEASURED_PEAKS.json") else 6552.0
gbs = 36 * B * T / (ms * 1e-3) / 1e9
print(json.dumps({"lanes": B, "T": T, "rollout_ms": ms, "GBs": gbs, "frac": gbs / peak,
                  "env_steps_per_s": B * T / (ms * 1e-3), "all_ms": ts}))
