import sys, time
sys.path.insert(0, ".")
import torch
import bench
dev = torch.device("cuda", 0)
wl = bench.Workload(4096, 256, 0, 0, dev)
for i in range(5): wl.step(i)
torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
ts = []
for i in range(20):
    flush.fill_(1)
    t = time.perf_counter(); wl.step(100 + i); ts.append(time.perf_counter() - t)
torch.cuda.synchronize()
print("cpu per step us", sorted(ts)[10] * 1e6)
# GPU-only timing without flush, back-to-back
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(20): wl.step(200 + i)
b.record(); torch.cuda.synchronize(); print("back-to-back ms/step", a.elapsed_time(b) / 20)
