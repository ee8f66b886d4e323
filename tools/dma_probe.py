"""Why do copy-engine reads of CPU-written pinned pages run slow?  (diagnostic)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

nb = 5259264
d = torch.empty(nb, dtype=torch.uint8, device="cuda")


def ce(h, k=20):
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


h = amz.pinned_empty((nb,), torch.uint8)
print("fresh (alloc-time memset)", ce(h))
h.fill_(3)
print("after CPU fill", ce(h))
junk = torch.empty(1 << 29, dtype=torch.uint8)
junk.fill_(1)
s = int(junk[:: 4096].sum())
print("after evicting the CPU caches (512 MB written)", ce(h))
h2 = amz.pinned_empty((nb,), torch.uint8)
h2.fill_(5)
print("fresh + CPU fill", ce(h2))
x = int(h2[::64].sum())
print("after CPU read of it", ce(h2))
tp = torch.empty(nb, dtype=torch.uint8).pin_memory()
tp.fill_(7)
print("torch pin_memory + fill", ce(tp))
