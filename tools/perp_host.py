"""Host enqueue time vs device time of PLR-perp / ACCEL-perp iterations (diagnostic)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import SequentialPLR  # noqa: E402

n, T = 4096, 256
for accel in (None, AccelConfig(20, 4)):
    plr = SequentialPLR(n, amz.StaticParams(), PlrConfig(buffer_size=4000, staleness_coef=0.3), amz.RngStream.from_seed(11),
                        accel)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    acts = torch.randint(0, 3, (T, n), generator=g, device="cuda", dtype=torch.uint8)
    vals = torch.rand((T, n), generator=g, device="cuda", dtype=torch.float64)
    last = torch.rand((n,), generator=g, device="cuda", dtype=torch.float64)
    for it in range(8):
        plr.iteration(it, acts, vals, last)
    torch.cuda.synchronize()
    hs, ds, dec = [], [], []
    for it in range(8, 28):
        t0 = time.perf_counter()
        plr.decide(it)
        dec.append(time.perf_counter() - t0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)  # keep the GPU busy: pure host enqueue time
        a.record()
        t0 = time.perf_counter()
        plr.iteration(it, acts, vals, last)
        hs.append(time.perf_counter() - t0)
        b.record()
        torch.cuda.synchronize()
        ds.append(a.elapsed_time(b))
    print("accel" if accel else "plr", "host enqueue us", round(1e6 * sum(hs) / len(hs)), "of which decide us",
          round(1e6 * sum(dec) / len(dec)), "device us", round(1e3 * sum(ds) / len(ds)))
