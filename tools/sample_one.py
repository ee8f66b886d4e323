"""One batched DR level generation (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402

p = amz.StaticParams()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for _ in range(3):
    lv = amz.sample_levels(amz.RngStream(1, (0,)), n, p)
torch.cuda.synchronize()
print("ok", lv.shape)
