import cProfile, pstats, sys, io
import torch
sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz
from paper_2311_12716_b200.buffer import PlrConfig
from paper_2311_12716_b200.plr import SequentialPLR
n, T = 4096, 256
plr = SequentialPLR(n, amz.StaticParams(), PlrConfig(buffer_size=4000, staleness_coef=0.3), amz.RngStream.from_seed(11))
g = torch.Generator(device="cuda"); g.manual_seed(1)
acts = torch.randint(0, 3, (T, n), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, n), generator=g, device="cuda", dtype=torch.float64)
last = torch.rand((n,), generator=g, device="cuda", dtype=torch.float64)
for it in range(8): plr.iteration(it, acts, vals, last)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for it in range(8, 48):
    plr.iteration(it, acts, vals, last)
pr.disable()
torch.cuda.synchronize()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
