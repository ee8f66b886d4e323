"""Steady-state e2e step time per H2D path (kernel / copy engine), alternating, after a
long warm-up (diagnostic)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True,
                     copy_mode="kernel")
g.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
g.host_inputs["values"].copy_(torch.rand(T, B))
g.host_inputs["last"].copy_(torch.rand(B))
g.capture()


def run(ce, k):
    g.copy_engine = ce
    g._pending_h2d = False
    for _ in range(3):
        g.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        g.step()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


for k in (8, 8, 50, 200, 8, 8):
    print(k, "kernel", run(False, k), "engine", run(True, k))

# when does the step speed up?  blocks of 20 steps from a fresh graph
g2 = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(1), T,
                      amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True,
                      copy_mode=sys.argv[1] if len(sys.argv) > 1 else "kernel")
g2.capture()
torch.cuda.synchronize()
import time  # noqa: E402

time.sleep(2.0)
t0 = time.perf_counter()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
ev[0].record()
for blk in range(40):
    for _ in range(20):
        g2.step()
    ev[blk + 1].record()
torch.cuda.synchronize()
print(g2.copy_mode, "per-step us by block of 20:", [round(ev[i].elapsed_time(ev[i + 1]) * 50) for i in range(40)])
