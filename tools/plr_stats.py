"""Per-update statistics of k_plr_update (built with -DAMZ_PLR_STATS):
    AMZ_LIB_PATH=tools/libamaze_stats.so python tools/plr_stats.py [plr|accel] [n]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "plr"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
T = 256
accel = AccelConfig(20, 4) if mode == "accel" else None
cfg = PlrConfig(buffer_size=4000, staleness_coef=0.5, replay_rate=0.8 if accel else 0.5)
plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(7), accel)
L = plr.L
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, L), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, L), generator=g, device="cuda", dtype=torch.float64) * 0.2
last = torch.rand((L,), generator=g, device="cuda", dtype=torch.float64) * 0.2
fn = _lib.lib().amz_debug_plr_stats
buf = (ctypes.c_ulonglong * 40)()
names = ["seq", "seq_inplace", "bulk_runs", "bulk_cands", "insert_calls", "insert_passes", "run_cands", "relevant",
         "calls", "cache_rebuilds", "batched", "cyc_B", "cyc_C", "batch_steps", "cyc_batch", "cyc_inplace_scan", "cyc_warp0", "warp0_sections", "cyc_rebuild", "cyc_insert_runs", "cyc_scalar", "n_scalar", "cyc_scalar_pre", "cyc_inplace_body", "cyc_fill", "n_fill", "cyc_evict_argmin", "n_evict", "cyc_evict_full", "n_evict_acc", "probes_gread", "probes", "cyc_probe_eval", "n_probe_eval_or_bulk_nocache", "cyc_A", "cyc_epilogue", "x36", "x37", "x38", "bulk_invalidating"]
for it in range(6):
    fn(buf, 1)
    r = plr.iteration(it, acts, vals, last)
    torch.cuda.synchronize()
    fn(buf, 1)
    sc = r.scores
    print(it, {k: int(buf[i]) for i, k in enumerate(names)}, "zero scores", int((sc == 0).sum()), "of", sc.numel())
