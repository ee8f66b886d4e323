"""Which of the step's kernels slows down (or slows the copy) when the H2D copy kernel
runs beside it?  (diagnostic)"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402
from paper_2311_12716_b200.gae import gae_and_scores  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                      amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True)
gr.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
gr.host_inputs["values"].copy_(torch.rand(T, B))
gr.host_inputs["last"].copy_(torch.rand(B))
gr.capture()
gr.step()
torch.cuda.synchronize()
lanes = gr.benv._ensure(gr.p)
o, inp = gr.out, gr.inputs[0]


def reset():
    _lib.call("amz_env_reset_dr_iter", lanes.handle, ctypes.byref(gr.root_pfx), _lib.ptr(gr.it_dev),
              _lib.ptr(o["reset_view"]), _lib.ptr(o["reset_dir"]), lanes.stream())


def roll():
    _lib.call("amz_env_rollout_iter", lanes.handle, gr.T, _lib.ptr(inp["actions"]), ctypes.byref(gr.root_pfx),
              _lib.ptr(gr.it_dev), _lib.ptr(o["view"]), _lib.ptr(o["dir"]), _lib.ptr(o["rewards"]),
              _lib.ptr(o["dones"]), _lib.ptr(o["final_view"]), _lib.ptr(o["final_dir"]), lanes.stream())


def gae():
    gae_and_scores(o["rewards"], inp["values"], o["dones"], inp["last"], gr.gamma, gr.lam, out=gr.gae)


def timeit(fn, k=30):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


s = torch.cuda.Stream()
for ctas in (16, 32, 64):
    for name, fns in (("reset", [reset]), ("rollout", [roll]), ("gae", [gae]), ("rollout x2", [roll, roll]),
                      ("reset+rollout+gae", [reset, roll, gae])):
        def body(fns=fns):
            for f in fns:
                f()
        gk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gk, stream=s):
            body()
        gc = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gc, stream=s):
            gr._h2d(0)
        gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb, stream=s):
            cur = torch.cuda.current_stream()
            side = torch.cuda.Stream(priority=-5)
            side.wait_stream(cur)
            gr.copy_ctas = ctas
            gr._h2d(0, side)
            body()
            cur.wait_stream(side)
        gr.copy_ctas = ctas
        print(f"ctas {ctas} {name}: kernels {timeit(gk.replay)} copy {timeit(gc.replay)} both {timeit(gb.replay)}")
