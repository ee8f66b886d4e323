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

# per-call host cost (no profiler): reset, rollout_actions, gae_and_scores
amz = wl.amz
res = wl.env.reset(wl.root.fold_in(0), wl.p)
traj, _ = amz.rollout_actions(wl.env, res, wl.actions, wl.p, out=wl.out)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for i in range(N):
    res = wl.env.reset(wl.root.fold_in(i), wl.p)
t1 = time.perf_counter()
for i in range(N):
    amz.rollout_actions(wl.env, res, wl.actions, wl.p, out=wl.out)
t2 = time.perf_counter()
for i in range(N):
    amz.gae_and_scores(traj.rewards, wl.values, traj.dones, wl.last, 0.995, 0.95, out=wl.gout)
t3 = time.perf_counter()
torch.cuda.synchronize()
print(f"reset {(t1 - t0) / N * 1e6:.1f} us  rollout {(t2 - t1) / N * 1e6:.1f} us  gae {(t3 - t2) / N * 1e6:.1f} us")
