"""Micro-benchmark of the PLR buffer update: all-insert, all-dup and mixed candidate batches."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import LevelBuffer, PlrConfig  # noqa: E402

K, n = 4000, 4096
p = amz.StaticParams()
pool = amz.sample_levels(amz.RngStream(1, (0,)), 40000, p)
rng = np.random.default_rng(0)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


buf = LevelBuffer(PlrConfig(buffer_size=K))
init = pool[:K]
sc0 = torch.from_numpy(rng.uniform(0, 1, K) * (rng.uniform(size=K) < 0.5)).cuda()
buf.update(init, sc0, sc0, 0)
st = buf.export()
it = [1]


def reload():
    buf.load(st)


def run(levels, scores):
    reload()
    torch.cuda.synchronize()
    it[0] += 1
    return timed(lambda: buf.update(levels, scores, scores, it[0]), reps=1)


new = pool[K:K + n]
dup_idx = torch.from_numpy(rng.integers(0, K, n)).cuda()
dups = init[dup_idx]
for name, lv, sc in [
    ("all-new zero scores", new, torch.zeros(n, dtype=torch.float64, device="cuda")),
    ("all-new positive", new, torch.from_numpy(rng.uniform(0.2, 1, n)).cuda()),
    ("all-dup", dups, torch.from_numpy(rng.uniform(0, 1, n)).cuda()),
    ("mixed new|dup", torch.cat([new[: n // 2], dups[: n // 2]]),
     torch.from_numpy(np.concatenate([rng.uniform(0, 1, n // 2) * (rng.uniform(size=n // 2) < 0.25),
                                      rng.uniform(0, 1, n // 2)])).cuda()),
]:
    ms = [run(lv, sc) for _ in range(3)]
    print(f"{name:24s} {sorted(ms)[1]*1e3:9.1f} us")
