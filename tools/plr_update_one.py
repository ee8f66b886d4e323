"""One all-insert PLR update (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import LevelBuffer, PlrConfig  # noqa: E402

K, n = 4000, 4096
p = amz.StaticParams()
pool = amz.sample_levels(amz.RngStream(1, (0,)), K + n, p)
rng = np.random.default_rng(0)
buf = LevelBuffer(PlrConfig(buffer_size=K))
sc0 = torch.from_numpy(rng.uniform(0, 1, K) * (rng.uniform(size=K) < 0.5)).cuda()
buf.update(pool[:K], sc0, sc0, 0)
sc = torch.from_numpy(rng.uniform(0.2, 1, n)).cuda()
buf.update(pool[K:], sc, sc, 1)
torch.cuda.synchronize()
print("ok")
