"""Does host<->device traffic slow the DR-iteration graph, and why?  (diagnostic)
The graph is replayed N times on the main stream while a side stream runs a copy load."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32)
g.capture()
N = 20
nb = 5259264
hbig = amz.pinned_empty((nb,), torch.uint8)
hsmall = amz.pinned_empty((1 << 16,), torch.uint8)
dbig = torch.empty(nb, dtype=torch.uint8, device="cuda")
dsrc = torch.empty(nb, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
main = torch.cuda.current_stream()


hw = amz.pinned_empty((nb,), torch.uint8)
hw.copy_(torch.randint(0, 3, (nb,), dtype=torch.uint8))  # written by the CPU (dirty in its caches)
hz = amz.pinned_empty((nb,), torch.uint8)
hz.zero_()


def loads():
    yield "none", lambda: None
    yield "CE H2D 5.3MB cpu-written", lambda: dbig.copy_(hw, non_blocking=True)
    yield "CE H2D 5.3MB zeroed", lambda: dbig.copy_(hz, non_blocking=True)
    yield "kernel H2D cpu-written", lambda: _lib.call("amz_copy_h2d", dbig.data_ptr(), hw.data_ptr(), nb, 32,
                                                      torch.cuda.current_stream().cuda_stream)
    yield "CE H2D 5.3MB", lambda: dbig.copy_(hbig, non_blocking=True)
    yield "CE H2D 64KB x80", lambda: [dbig[i << 16:(i + 1) << 16].copy_(hsmall, non_blocking=True) for i in range(80)]
    yield "CE D2H 5.3MB", lambda: hbig.copy_(dbig, non_blocking=True)
    yield "CE D2D 5.3MB", lambda: dbig.copy_(dsrc, non_blocking=True)
    yield "kernel H2D 5.3MB", lambda: _lib.call("amz_copy_h2d", dbig.data_ptr(), hbig.data_ptr(), nb, 32,
                                                torch.cuda.current_stream().cuda_stream)


for name, fn in loads():
    for _ in range(3):
        g.graphs[0].replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        torch.cuda._sleep(2000)
        c0.record()
        for _ in range(3 * N):
            fn()
        c1.record()
    a.record(main)
    for _ in range(N):
        g.graphs[0].replay()
    b.record(main)
    torch.cuda.synchronize()
    print(f"{name:26s} graph us {a.elapsed_time(b) / N * 1000:7.1f}   load per op us {c0.elapsed_time(c1) / (3 * N) * 1000:7.1f}")
