"""Probe the end-to-end DRIterationGraph step time for copy layouts:
    python tools/e2e_probe.py [B]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = 256
for vdt in (torch.float32, torch.float64):
    for overlap, cs in ((False, 1), (True, 1), (True, 2)):
        gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0),
                              T, amz.StaticParams(), 0.995, 0.98, value_dtype=vdt, host_io=True, overlap=overlap,
                              copy_streams=cs).capture()
        for _ in range(5):
            gr.step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30):
            gr.step()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 30
        print(f"{str(vdt):14s} overlap={overlap} streams={cs} ms/step={ms:.4f} H2D GB/s if copy-bound="
              f"{gr._nbytes / (ms * 1e-3) / 1e9:.1f}")
        del gr
# raw H2D rate, 1 and 2 streams
n = 5 << 20
h = amz.pinned_empty((n,), torch.uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2):
    ss = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * n // k:(i + 1) * n // k].copy_(h[i * n // k:(i + 1) * n // k], non_blocking=True)
    torch.cuda.synchronize()
    print("raw H2D streams", k, "GB/s", 20 * n / (time.perf_counter() - t0) / 1e9)
