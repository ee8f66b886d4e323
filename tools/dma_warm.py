"""Is the PCIe read rate low right after an idle period (link power state)?  (diagnostic)"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402

nb = 5259264
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
h = amz.pinned_empty((nb,), torch.uint8)
h.fill_(3)
torch.cuda.synchronize()
for mode in ("ce", "kernel", "ce"):
    time.sleep(1.0)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
    evs[0].record()
    for i in range(40):
        if mode == "ce":
            d.copy_(h, non_blocking=True)
        else:
            _lib.call("amz_copy_h2d", d.data_ptr(), h.data_ptr(), nb, 32, torch.cuda.current_stream().cuda_stream)
        evs[i + 1].record()
    torch.cuda.synchronize()
    print(mode, "after 1 s idle, per-copy us:", [round(evs[i].elapsed_time(evs[i + 1]) * 1000) for i in range(40)])
