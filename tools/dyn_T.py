"""k_dyn HOME/RESAMPLE time vs T (fixed B) to split per-step cost from fixed overhead."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = amz.StaticParams()
for mode in (amz.HOME, amz.RESAMPLE):
    for T in (32, 64, 128, 256, 512):
        env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
        acts = torch.randint(0, 3, (T, B), dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(6):
            res = env.reset(amz.RngStream.from_seed(i), p)
            torch.cuda.synchronize()
            tr, cur = amz.rollout_actions(env, res, acts, p)
        torch.cuda.synchronize()
