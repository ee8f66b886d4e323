"""Where does the e2e step's time go?  (diagnostic)
device-only graph vs host_io graphs with the H2D as the SM copy kernel (ctas) or as a
copy-engine memcpy, and each copy alone."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256


def mk(host_io, ctas=64, ce=False, split=1):
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                          amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=host_io, overlap=host_io,
                          copy_ctas=ctas, copy_mode="kernel")
    if host_io:
        gr.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
        gr.host_inputs["values"].copy_(torch.rand(T, B))
        gr.host_inputs["last"].copy_(torch.rand(B))
    return gr.capture()


def timeit(fn, k=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


g0 = mk(False)
print("device-only graph us", timeit(g0.step))
for ctas in (8, 16, 24, 32, 48, 64):
    g = mk(True, ctas)
    t = timeit(g.step)
    print(f"host_io kernel copy ctas={ctas} us", t, "copy alone us", timeit(lambda: g._h2d(0)))
g = mk(True, 32)
g.overlap = False
print("(graphs captured for overlap, replayed without the copy) us", timeit(lambda: g.graphs[0].replay()))
