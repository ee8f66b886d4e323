"""Replay time of the DR-iteration graph alone (no copies beside it): device inputs f64 /
f32, and the host-io graph (its result read-back kernel at the end).  Diagnostic."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256


def mk(vdt, host_io):
    g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                         amz.StaticParams(), 0.995, 0.98, value_dtype=vdt, host_io=host_io, overlap=host_io)
    acts = torch.randint(0, 3, (T, B), dtype=torch.uint8)
    if host_io:
        g.host_inputs["actions"].copy_(acts)
    g.inputs[0]["actions"].copy_(acts.cuda())
    if host_io:
        g.inputs[1]["actions"].copy_(acts.cuda())
    return g.capture()


def t(fn, k=40):
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


for vdt in (torch.float64, torch.float32):
    g = mk(vdt, False)
    print(vdt, "device-io graph", t(lambda: g.graphs[0].replay()))
    h = mk(vdt, True)
    print(vdt, "host-io graph (no copies)", t(lambda: h.graphs[0].replay()))
