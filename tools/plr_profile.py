"""Run a few parallel PLR / ACCEL iterations (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

accel = len(sys.argv) > 1 and sys.argv[1] == "accel"
n, T = 2048, 256
plr = ParallelPLR(n, amz.StaticParams(), PlrConfig(buffer_size=4000), amz.RngStream.from_seed(7),
                  AccelConfig(20, 4) if accel else None)
L = plr.L
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, L), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, L), generator=g, device="cuda", dtype=torch.float64) * 0.2
last = torch.rand((L,), generator=g, device="cuda", dtype=torch.float64) * 0.2
for it in range(6):
    r = plr.iteration(it, acts, vals, last)
torch.cuda.synchronize()
print("size", plr.buffer.size(), "replay", r.n_replay)
