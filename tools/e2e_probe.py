"""Probe the end-to-end DRIterationGraph step time (valid synthetic inputs, as bench.py):
    python tools/e2e_probe.py [B]
Prints ms/step for: device-resident inputs, host I/O without overlap, host I/O with the
next step's copy overlapped (1 and 2 copy streams), and the raw pinned H2D rate."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = 256
g = torch.Generator(device="cuda")
g.manual_seed(1)
acts = torch.randint(0, 3, (T, B), generator=g, device="cuda", dtype=torch.uint8)
vals = torch.rand((T, B), generator=g, device="cuda", dtype=torch.float64)
last = torch.rand((B,), generator=g, device="cuda", dtype=torch.float64)


def run(gr, n=30):
    for _ in range(5):
        gr.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        gr.step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for vdt in (torch.float32, torch.float64):
    for host_io, overlap, cs in ((False, False, 1), (True, False, 1), (True, True, 1), (True, True, 2)):
        gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0),
                              T, amz.StaticParams(), 0.995, 0.98, value_dtype=vdt, host_io=host_io, overlap=overlap,
                              copy_streams=cs)
        if host_io:
            gr.host_inputs["actions"].copy_(acts.cpu())
            gr.host_inputs["values"].copy_(vals.to(vdt).cpu())
            gr.host_inputs["last"].copy_(last.to(vdt).cpu())
        else:
            gr.inputs[0]["actions"].copy_(acts)
            gr.inputs[0]["values"].copy_(vals.to(vdt))
            gr.inputs[0]["last"].copy_(last.to(vdt))
        gr.capture()
        print(f"{str(vdt):14s} host_io={host_io} overlap={overlap} streams={cs} ms/step={run(gr):.4f}")
        del gr
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
