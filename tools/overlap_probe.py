"""Does the kernel H2D copy overlap a concurrent graph branch?  (diagnostic)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402

n = 5259264
h = amz.pinned_empty((n,), torch.uint8)
h.copy_(torch.randint(0, 3, (n,), dtype=torch.uint8))
d = torch.empty(n, dtype=torch.uint8, device="cuda")
x = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timeit(fn, k=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k, 4)


def copyk(st, ctas):
    _lib.call("amz_copy_h2d", d.data_ptr(), h.data_ptr(), n, ctas, st.cuda_stream)


s = torch.cuda.Stream()
for ctas in (32, 64, 148):
    for other in ("sleep", "fill"):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            cur = torch.cuda.current_stream()
            side = torch.cuda.Stream(priority=-5)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                copyk(side, ctas)
            if other == "sleep":
                torch.cuda._sleep(250_000)  # ~0.13 ms on one SM
            else:
                for _ in range(6):
                    x.add_(1.0)  # memory-bound kernels over all SMs, ~0.13 ms
            cur.wait_stream(side)
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga, stream=s):
            copyk(torch.cuda.current_stream(), ctas)
        gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb, stream=s):
            if other == "sleep":
                torch.cuda._sleep(250_000)
            else:
                for _ in range(6):
                    x.add_(1.0)
        print(f"ctas {ctas} {other}: copy alone {timeit(ga.replay)} other alone {timeit(gb.replay)} "
              f"both {timeit(g.replay)}")
