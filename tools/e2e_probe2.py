"""Where the host-I/O DRIterationGraph step time goes (diagnostic)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                      amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=False)
gr.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
gr.host_inputs["values"].copy_(torch.rand(T, B))
gr.host_inputs["last"].copy_(torch.rand(B))
gr.capture()


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("graph step", timeit(gr.step))
print("eager h2d", timeit(lambda: gr._h2d(0)))
print("eager kernels", timeit(lambda: gr._kernels(gr.inputs[0])))
print("eager d2h", timeit(lambda: gr.host_result.copy_(gr.res, non_blocking=True)))
print("host_raw pinned", gr._host_raw.is_pinned(), "result pinned", gr.host_result.is_pinned())
g2 = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.graph(g2, stream=s):
    gr._h2d(0)
print("graph h2d only", timeit(g2.replay))
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3, stream=s):
    gr.host_result.copy_(gr.res, non_blocking=True)
print("graph d2h only", timeit(g3.replay))
import paper_2311_12716_b200 as amz2  # noqa: E402
n = gr._nbytes
fresh_d = torch.empty(n, dtype=torch.uint8, device="cuda")
fresh_h = amz2.pinned_empty((n,), torch.uint8)
print("host_raw -> fresh device", timeit(lambda: fresh_d.copy_(gr._host_raw, non_blocking=True)))
print("fresh host -> raw[0]", timeit(lambda: gr._raw[0].copy_(fresh_h, non_blocking=True)))
print("fresh host -> fresh device", timeit(lambda: fresh_d.copy_(fresh_h, non_blocking=True)))
print("ptrs", hex(gr._host_raw.data_ptr()), hex(fresh_h.data_ptr()), gr._host_raw.stride(), gr._host_raw.is_contiguous(),
      gr._host_raw.storage_offset(), gr._host_raw.dtype, gr._host_raw.shape)
