"""Does the input CONTENT change the e2e step time?  (diagnostic)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True,
                     copy_mode="kernel")
g.capture()


def fill(kind):
    if kind == "random":
        g.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
        g.host_inputs["values"].copy_(torch.rand(T, B))
        g.host_inputs["last"].copy_(torch.rand(B))
    else:
        g._host_raw.zero_()


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


fill("zero")
run(False, 600)
for kind in ("random", "zero", "random", "zero", "random"):
    fill(kind)
    print(kind, [("kernel", run(False, 100), "engine", run(True, 100)) for _ in range(3)])
