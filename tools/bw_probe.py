"""HBM bandwidth of write-only (fill_), read-only (sum) and copy (read+write) streams on
this B200, 1 GiB buffers, CUDA events, best of 10 -- the denominators behind the
rollout's roofline (its traffic is ~90% writes)."""
import json

import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
for name, fn, nbytes in (("write_fill", lambda: a.fill_(3), n), ("read_sum", lambda: a.view(torch.int64).sum(), n),
                         ("copy", lambda: b.copy_(a), 2 * n)):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[name + "_GBs"] = nbytes / (best * 1e-3) / 1e9
print(json.dumps(out))
