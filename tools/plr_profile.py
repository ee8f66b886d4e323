"""Run a few PLR iterations (for ncu launch lists):
    python tools/plr_profile.py [plr|accel|perp|accel_perp] [n]
plr/accel: ParallelPLR (PLR|| / ACCEL||) with n new lanes; perp: SequentialPLR."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR, SequentialPLR  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "plr"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
T = 256
accel = AccelConfig(20, 4) if mode in ("accel", "accel_perp") else None
cfg = PlrConfig(buffer_size=4000, staleness_coef=0.5, replay_rate=0.8 if accel else 0.5)
if mode.endswith("perp"):
    plr = SequentialPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(7), accel)
    L = n
else:
    plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(7), accel)
    L = plr.L
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, L), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, L), generator=g, device="cuda", dtype=torch.float64) * 0.2
last = torch.rand((L,), generator=g, device="cuda", dtype=torch.float64) * 0.2
for it in range(8):
    r = plr.iteration(it, acts, vals, last)
torch.cuda.synchronize()
print("size", plr.buffer.size())
