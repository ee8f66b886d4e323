"""Host enqueue time vs device time of PLR|| / ACCEL|| iterations (diagnostic)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

T = 256
for n, accel in ((2048, None), (2048, AccelConfig(20, 4)), (16384, None)):
    plr = ParallelPLR(n, amz.StaticParams(), PlrConfig(buffer_size=4000, staleness_coef=0.5), amz.RngStream.from_seed(7),
                      accel)
    L = plr.L
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    acts = torch.randint(0, 3, (T, L), generator=g, device="cuda", dtype=torch.uint8)
    vals = torch.rand((T, L), generator=g, device="cuda", dtype=torch.float64)
    last = torch.rand((L,), generator=g, device="cuda", dtype=torch.float64)
    for it in range(4):
        plr.iteration(it, acts, vals, last)
    torch.cuda.synchronize()
    hs, ds = [], []
    for it in range(4, 14):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(5_000_000)
        a.record()
        t0 = time.perf_counter()
        plr.iteration(it, acts, vals, last)
        hs.append(time.perf_counter() - t0)
        b.record()
        torch.cuda.synchronize()
        ds.append(a.elapsed_time(b))
    print(n, "accel" if accel else "plr", "host enqueue us", round(1e6 * sum(hs) / len(hs)), "device us",
          round(1e3 * sum(ds) / len(ds)))
