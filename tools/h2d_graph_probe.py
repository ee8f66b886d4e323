"""H2D copy rate of pinned (amz_host_alloc) memory: untouched vs written by the host,
eager and inside a captured graph:  python tools/h2d_graph_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

n = 5 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")


def rate(h, label):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    a.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    print(label, "GB/s", round(20 * n / (a.elapsed_time(b) * 1e-3) / 1e9, 1))


h = amz.pinned_empty((n,), torch.uint8)
rate(h, "untouched")
h.zero_()
rate(h, "zeroed")
h.copy_(torch.randint(0, 3, (n,), dtype=torch.uint8))
rate(h, "random bytes")
t = torch.empty(n, dtype=torch.uint8, pin_memory=True)
t.copy_(torch.randint(0, 3, (n,), dtype=torch.uint8))
rate(t, "torch pinned, random bytes")
h2 = amz.pinned_empty((n,), torch.uint8)
h2.numpy()[:] = 7
rate(h2, "numpy-filled")
