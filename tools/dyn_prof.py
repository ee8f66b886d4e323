"""Per-warp phase timing of k_dyn (needs tools/_prof/libamaze_b200.so built with -DAMZ_DYN_PROF)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200._lib as _l  # noqa: E402

_l.LIB_PATH = "tools/_prof/libamaze_b200.so"
import paper_2311_12716_b200 as amz  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = 256
p = amz.StaticParams()
for mode in (amz.HOME, amz.RESAMPLE):
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
    acts = torch.randint(0, 3, (T, B), dtype=torch.uint8, device="cuda")
    res = env.reset(amz.RngStream.from_seed(1), p)
    torch.cuda.synchronize()
    zero = np.zeros((65536, 8), dtype=np.uint64)
    _l.lib().amz_debug_dyn_prof_reset(ctypes.c_void_p(zero.ctypes.data))
    tr, cur = amz.rollout_actions(env, res, acts, p)
    torch.cuda.synchronize()
    buf = np.zeros((65536, 8), dtype=np.uint64)
    _l.lib().amz_debug_dyn_prof(ctypes.c_void_p(buf.ctypes.data))
    nw = B // 4
    b = buf[:nw]
    sm = (b[:, 0] >> np.uint64(56)).astype(int)
    t = (b & np.uint64((1 << 56) - 1)).astype(np.int64)
    pro, loop, epi = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2]
    # per-SM span: clock64 is per-SM, so compare within an SM
    spans = []
    for s in np.unique(sm):
        m = sm == s
        spans.append(t[m, 3].max() - t[m, 0].min())
    print(mode, "warps", nw, "prologue cyc med/max", int(np.median(pro)), int(pro.max()),
          "loop med/max", int(np.median(loop)), int(loop.max()), "epi med/max", int(np.median(epi)), int(epi.max()),
          "SM span med/max", int(np.median(spans)), int(max(spans)))
    ev, smp, tbl, q = [b[:, k].astype(np.int64) for k in (4, 5, 6, 7)]
    w = int(np.argmax(loop))
    print("   event cyc med/max", int(np.median(ev)), int(ev.max()), "sampler med/max", int(np.median(smp)), int(smp.max()),
          "table med/max", int(np.median(tbl)), int(tbl.max()), "sampled levels med/max", int(np.median(q & 0xFFFFFFFF)), int((q & 0xFFFFFFFF).max()))
    nsmp, nev, nfin = q & 0xFFFFFFFF, (q >> 32) & 0xFFFF, q >> 48
    b2 = np.zeros((65536, 8), dtype=np.uint64)
    if hasattr(_l.lib(), "amz_debug_dyn_prof2"):
        _l.lib().amz_debug_dyn_prof2(ctypes.c_void_p(b2.ctypes.data))
    b2 = b2[:nw].astype(np.int64)
    print("   slowest warp sub-phases: pre-sample", int(b2[w, 0]), "key", int(b2[w, 1]), "board+record", int(b2[w, 2]))
    print("   slowest warp: loop", int(loop[w]), "events", int(ev[w]), "sampler", int(smp[w]), "table", int(tbl[w]),
          "sampled", int(nsmp[w]), "event steps", int(nev[w]), "lane ends", int(nfin[w]))
    print("   event steps med/max", int(np.median(nev)), int(nev.max()), "lane ends med/max", int(np.median(nfin)), int(nfin.max()))
