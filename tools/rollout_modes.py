"""Time the fused rollout in HOME vs RESAMPLE mode (dynamics-only vs with resampling)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = 256
p = amz.StaticParams()
for mode in (amz.HOME, amz.RESAMPLE):
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
    acts = torch.randint(0, 3, (T, B), dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(8):
        res = env.reset(amz.RngStream.from_seed(i), p)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tr, cur = amz.rollout_actions(env, res, acts, p)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        solved = int((tr.rewards > 0).sum())
    print(mode, B, "ms", sorted(ts)[len(ts) // 2], "solved episodes", solved, "dones", int(tr.dones.sum()))
