"""After the host CPU rewrites the pinned feed, is the slow-PCIe-read period a matter of
time or of traffic?  (diagnostic)"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True,
                     copy_mode="engine")
g.capture()
acts = torch.randint(0, 3, (T, B), dtype=torch.uint8)
vals = torch.rand(T, B)
last = torch.rand(B)


def blocks(n=6, k=20):
    out = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            g.step()
        b.record()
        torch.cuda.synchronize()
        out.append(round(a.elapsed_time(b) / k * 1000))
    return out


for _ in range(300):
    g.step()
torch.cuda.synchronize()
print("settled", blocks())
for wait in (0.0, 0.1, 0.5, 2.0, 0.0):
    g.host_inputs["actions"].copy_(acts)
    g.host_inputs["values"].copy_(vals)
    g.host_inputs["last"].copy_(last)
    time.sleep(wait)
    print(f"rewrite, idle {wait} s, then us/step by block of 20:", blocks())
