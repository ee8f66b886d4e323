"""Does capturing a host->device copy into a CUDA graph change the source's copy rate?"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

n = 5259264
d = torch.empty(n, dtype=torch.uint8, device="cuda")


def rate(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(20 * n / (a.elapsed_time(b) * 1e-3) / 1e9, 1)


h = amz.pinned_empty((n,), torch.uint8)
h[: n // 2].view(torch.float32).copy_(torch.rand(n // 8))
print("eager before capture", rate(lambda: d.copy_(h, non_blocking=True)))
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    d.copy_(h, non_blocking=True)
print("graph replay", rate(g.replay))
print("eager after capture", rate(lambda: d.copy_(h, non_blocking=True)))
h2 = amz.pinned_empty((n,), torch.uint8)
print("other buffer eager", rate(lambda: d.copy_(h2, non_blocking=True)))
# a kernel-containing graph reading a device buffer filled from h
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=s):
    d.copy_(h, non_blocking=True)
    d.add_(1)
print("graph copy+kernel", rate(g2.replay))
from paper_2311_12716_b200 import _lib  # noqa: E402
h3 = amz.pinned_empty((n,), torch.uint8)
h3.copy_(torch.randint(0, 3, (n,), dtype=torch.uint8))
for ctas in (16, 32, 64, 128):
    def kc():
        _lib.call("amz_copy_h2d", d.data_ptr(), h3.data_ptr(), n, ctas, torch.cuda.current_stream().cuda_stream)
    g4 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g4, stream=s):
        kc()
    print("kernel copy ctas", ctas, "eager", rate(kc), "graph", rate(g4.replay))
print("check", bool((d.cpu() == h3).all()))
