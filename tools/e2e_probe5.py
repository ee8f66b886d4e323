"""e2e step with the H2D as SM copy kernel vs copy-engine memcpys over 1/2/4 streams,
pipelined one step ahead (diagnostic)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256


def mk(**kw):
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                          amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True, **kw)
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


for rep in range(2):
    for kw in (dict(copy_mode="kernel", copy_ctas=16), dict(copy_mode="kernel", copy_ctas=32), dict(copy_mode="engine", copy_streams=1),
               dict(copy_mode="engine", copy_streams=2), dict(copy_mode="engine", copy_streams=4)):
        g = mk(**kw)
        cur = torch.cuda.current_stream()

        def copy_only(g=g):
            g._issue_copy(0)
            cur.wait_event(g._copied[0])
        print(rep, kw, "step us", timeit(g.step), "copy alone us", timeit(copy_only))
