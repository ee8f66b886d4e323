"""DR reset (+ the first rollout's timeout levels) time per lane count (diagnostic;
AMZ_RESET_WARP=1 selects the warp-per-level kernel)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

P = amz.StaticParams()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for B in (4096, 65536):
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    env.reset(amz.RngStream.from_seed(0), P)
    ts = []
    for i in range(20):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        env.reset(amz.RngStream.from_seed(i), P)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    print(B, "reset us (median)", round(sorted(ts)[10], 1))
