"""Median device time of one PLR buffer sample (K=4000, 2048 draws); argv[1] is a label."""
import sys, statistics, torch
sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz
torch.cuda.set_device(0)
torch.zeros(1, device="cuda:0")
from paper_2311_12716_b200.buffer import PlrConfig, LevelBuffer
buf = LevelBuffer(PlrConfig(buffer_size=4000))
lv = amz.sample_levels(amz.RngStream(3, (0,)), 4096, amz.StaticParams(), device="cuda:0")
buf.update(lv, torch.rand(4096, device="cuda:0", dtype=torch.float64) * (torch.rand(4096, device="cuda:0") > 0.3), torch.zeros(4096, device="cuda:0", dtype=torch.float64), 1)
ts = []
for i in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = buf.sample(amz.RngStream(5, (i,)), 2048, 10 + i); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
print(sys.argv[1], "sample us median", statistics.median(ts[5:]), "slots digest", int(out["slots"].sum()))
