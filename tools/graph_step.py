"""Device-timed DR-iteration graph step, L2 flushed before each (as bench.py's headline);
diagnostic for graph-structure changes: python tools/graph_step.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
flush = torch.empty(32 << 20, dtype=torch.int64, device="cuda")
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98)
gen = torch.Generator(device="cuda")
gen.manual_seed(1234)
g.inputs[0]["actions"].copy_(torch.randint(0, 3, (T, B), generator=gen, device="cuda", dtype=torch.uint8))
g.inputs[0]["values"].copy_(torch.rand((T, B), generator=gen, device="cuda", dtype=torch.float64))
g.capture()
for _ in range(5):
    g.step()
res = []
for rep in range(3):
    ts = []
    for i in range(50):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    res.append(round(sum(ts) / len(ts), 1))
print("graph step us (mean of 50, x3):", res)
