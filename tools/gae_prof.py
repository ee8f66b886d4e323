"""Per-CTA phase clocks of k_gae_score4 (needs tools/_prof/libamaze_b200.so built with -DAMZ_GAE_PROF)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200._lib as _l  # noqa: E402

_l.LIB_PATH = __import__("os").environ.get("GAE_PROF_LIB", "tools/_prof/libamaze_b200.so")
import paper_2311_12716_b200 as amz  # noqa: E402

B, T = 4096, 256
g = torch.Generator(device="cuda")
g.manual_seed(1)
r = (torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64) < 0.01).double()
v = torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64)
d = torch.rand((T, B), generator=g, device="cuda") < 0.004
last = torch.rand((B,), generator=g, device="cuda", dtype=torch.float64)
flush = torch.empty(32 << 20, dtype=torch.int64, device="cuda")
for it in range(3):
    flush.fill_(it)
    out = amz.gae_and_scores(r, v, d, last, 0.995, 0.95)
    torch.cuda.synchronize()
buf = np.zeros((4096, 8), dtype=np.int64)
_l.lib().amz_debug_gae_prof(ctypes.c_void_p(buf.ctypes.data))
b = buf[: B // 8]
names = ["load", "fwd(w0)", "prep(w1-3)", "rev(w1)", "pass3+final"]
ph = [b[:, 1] - b[:, 0], b[:, 2] - b[:, 1], b[:, 3] - b[:, 1], b[:, 4] - b[:, 3], b[:, 6] - b[:, 5]]
for n, x in zip(names, ph):
    print(f"{n:12s} med {int(np.median(x)):6d}  max {int(x.max()):6d} cycles")
print("total (0->6) med", int(np.median(b[:, 6] - b[:, 0])), "max", int((b[:, 6] - b[:, 0]).max()))
