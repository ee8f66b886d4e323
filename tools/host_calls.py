"""Host-side cost (us per call, GPU kept busy so launches never wait) of the public calls
a PLR-perp iteration makes (diagnostic)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import LevelBuffer, PlrConfig  # noqa: E402

n, T = 4096, 256
P = amz.StaticParams()
root = amz.RngStream.from_seed(3)
env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, n)), amz.HOME)
buf = LevelBuffer(PlrConfig(buffer_size=4000))
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, n), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, n), generator=g, device="cuda", dtype=torch.float64)
last = torch.rand((n,), generator=g, device="cuda", dtype=torch.float64)
lv = amz.sample_levels(root, n, P)
start = env.reset_to_levels(root, lv, P)
traj, _ = amz.rollout_actions(env, start, acts, P)
o = amz.gae_and_scores(traj.rewards, vals, traj.dones, last, 0.995, 0.98)
buf.update(lv, o["scores"], o["max_returns"], 0)
torch.cuda.synchronize()


def cost(name, fn, k=50):
    torch.cuda._sleep(20_000_000)
    t0 = time.perf_counter()
    for i in range(k):
        fn(i)
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    print(f"{name:28s} {dt:7.1f} us")


cost("fold_in+seed_prefix", lambda i: root.fold_in(i).fold_in(1).seed_prefix())
cost("decision (numpy)", lambda i: buf.decision(root.fold_in(i).fold_in(0)))
cost("sample_levels", lambda i: amz.sample_levels(root.fold_in(i), n, P))
cost("reset_to_levels", lambda i: env.reset_to_levels(root.fold_in(i), lv, P))
cost("rollout_actions", lambda i: amz.rollout_actions(env, start, acts, P))
cost("gae_and_scores", lambda i: amz.gae_and_scores(traj.rewards, vals, traj.dones, last, 0.995, 0.98))
cost("buffer.update", lambda i: buf.update(lv, o["scores"], o["max_returns"], i + 1))
cost("buffer.sample", lambda i: buf.sample(root.fold_in(i), n, i + 100))
renv = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, n)), amz.RESAMPLE)
renv.reset(root, P)
res0 = renv.reset(root, P)
torch.cuda.synchronize()
cost("DR reset (RESAMPLE)", lambda i: renv.reset(root.fold_in(i), P))
cost("rollout RESAMPLE", lambda i: amz.rollout_actions(renv, res0, acts, P))
cost("flush fill_ 256MB", lambda i: vals.fill_(0.5))
