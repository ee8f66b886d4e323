"""DRIterationGraph(host_io, overlap) with the step's kernels removed / kept (diagnostic)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256


def mk(no_kernels):
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                          amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True)
    gr.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
    gr.host_inputs["values"].copy_(torch.rand(T, B))
    gr.host_inputs["last"].copy_(torch.rand(B))
    if no_kernels:
        gr._kernels = lambda inp, after=None: (after() if after else None, torch.cuda._sleep(int(no_kernels)))
    return gr.capture()


def timeit(gr, k=30):
    for _ in range(5):
        gr.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        gr.step()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k, 4)


print("copy + sleep(~0.13 ms)", timeit(mk(250_000)))
print("copy + tiny sleep", timeit(mk(100)))
print("copy + real kernels", timeit(mk(0)))
