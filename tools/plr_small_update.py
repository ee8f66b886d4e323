"""Fixed cost of the PLR buffer update: a full K=4000 buffer updated with n candidates
(new levels or in-place re-scores), kernel time by CUDA events and (with
AMZ_LIB_PATH=tools/libamaze_stats.so) the phase cycle counters.  Diagnostic."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.buffer import LevelBuffer, PlrConfig  # noqa: E402

P = amz.StaticParams()
K = 4000
pool = amz.sample_levels(amz.RngStream(1, (0,)), 12000, P)
buf = LevelBuffer(PlrConfig(buffer_size=K))
rng = np.random.default_rng(0)
buf.update(pool[:K], torch.from_numpy(rng.uniform(0, 1, K)), torch.zeros(K, dtype=torch.float64), 0)
torch.cuda.synchronize()
try:
    fn = _lib.lib().amz_debug_plr_stats
    stats = (ctypes.c_ulonglong * 40)()
except AttributeError:
    fn = None
it = 1
for kind, n in (("new", 4), ("new", 64), ("inplace", 4), ("inplace", 4096), ("new", 4096)):
    ts = []
    for rep in range(5):
        if kind == "new":
            idx = rng.integers(K, 12000, n)
        else:
            idx = rng.integers(0, K, n)
        lv = pool[torch.from_numpy(idx).cuda()]
        sc = torch.from_numpy(rng.uniform(0, 1, n))
        if fn:
            fn(stats, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        buf.update(lv, sc, sc, it)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
        it += 1
    line = f"{kind} n={n}: {sorted(ts)[2]:.1f} us"
    if fn:
        fn(stats, 1)
        line += f"  cyc A {stats[34]} B {stats[11]} C {stats[12]} epi {stats[35]} rebuild {stats[18]}x{stats[9]} warp0 {stats[16]} A-marks {stats[36]},{stats[37]},{stats[38]}"
        if len(sys.argv) > 1:
            names = ["seq", "seq_inplace", "bulk_runs", "bulk_cands", "insert_calls", "insert_passes", "run_cands",
                     "relevant", "calls", "cache_rebuilds", "batched", "cyc_B", "cyc_C", "batch_steps", "cyc_batch"]
            line += "\n   " + str({k: int(stats[i]) for i, k in enumerate(names)})
    print(line)
