"""Phase clocks of k_plr_sample (library built with -DAMZ_PLR_STATS):
    AMZ_LIB_PATH=tools/libamaze_stats.so python tools/samp_clk.py"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.buffer import LevelBuffer, PlrConfig  # noqa: E402

buf = LevelBuffer(PlrConfig(buffer_size=4000, staleness_coef=0.5))
lv = amz.sample_levels(amz.RngStream(1, (0,)), 4000, amz.StaticParams())
sc = torch.rand(4000, dtype=torch.float64, device="cuda")
buf.update(lv, sc, sc, 0)
names = ["start", "-", "-", "-", "weights", "pairwise sum", "P", "cumsum || uniforms", "normalize", "draws", "mark"]
clk = (ctypes.c_longlong * 16)()
for it in range(1, 4):
    buf.sample(amz.RngStream(5, (it,)), 2048, it)
    torch.cuda.synchronize()
    _lib.lib().amz_debug_samp_clk(clk)
    print({names[k]: clk[k] - clk[k - 1] for k in range(1, 11)}, "total cycles", clk[10] - clk[0])
