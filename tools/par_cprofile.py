"""cProfile of the host side of PLR|| iterations (where the ~320 us of enqueue goes):
    python tools/par_cprofile.py [n_iters]"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

T, n = 256, 2048
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
plr = ParallelPLR(n, amz.StaticParams(), PlrConfig(buffer_size=4000, staleness_coef=0.5), amz.RngStream.from_seed(7))
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, plr.L), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, plr.L), generator=g, device="cuda", dtype=torch.float64)
last = torch.rand((plr.L,), generator=g, device="cuda", dtype=torch.float64)
for it in range(4):
    plr.iteration(it, acts, vals, last)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for it in range(4, 4 + iters):
    plr.iteration(it, acts, vals, last)
    if it % 8 == 0:
        torch.cuda.synchronize()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
