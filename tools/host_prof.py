"""Host-side enqueue cost of one bench step (bench.Workload.step) under cProfile."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload(4096, 256, 7, 0, dev)
for i in range(5):
    wl.step(i)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(200):
    wl.step(100 + i)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue per step: {(t1 - t0) / 200 * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    wl.step(1000 + i)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
