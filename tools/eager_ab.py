"""Eager per-call config-2 step, back to back (no spin, no flush): device time per step
and host enqueue per step (diagnostic, for A/B of library builds via AMZ_LIB_PATH)."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.Workload(4096, 256, 0, 0, torch.device("cuda", 0))
for i in range(5):
    wl.step(i)
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for i in range(50):
        wl.step(100 + i)
    host = (time.perf_counter() - t0) / 50 * 1e6
    b.record()
    torch.cuda.synchronize()
    print(os.environ.get("AMZ_LIB_PATH", "default"), "b2b us/step", round(a.elapsed_time(b) / 50 * 1000, 1),
          "host us/step", round(host, 1))
