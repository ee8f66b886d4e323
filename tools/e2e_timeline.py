"""Timeline of the pipelined e2e step: copy start/end and graph start/end per step,
from CUDA events (diagnostic).  python tools/e2e_timeline.py [kernel|ce]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402

B, T = 4096, 256
mode = sys.argv[1] if len(sys.argv) > 1 else "kernel"
kw = dict(copy_mode="kernel", copy_ctas=32) if mode.startswith("kernel") else dict(copy_mode="engine", copy_streams=1)
g = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RngStream.from_seed(0), T,
                     amz.StaticParams(), 0.995, 0.98, value_dtype=torch.float32, host_io=True, overlap=True, **kw)
g.host_inputs["actions"].copy_(torch.randint(0, 3, (T, B), dtype=torch.uint8))
g.host_inputs["values"].copy_(torch.rand(T, B))
g.host_inputs["last"].copy_(torch.rand(B))
if mode.endswith("nod2h"):  # diagnostic: the graphs without the result read-back
    g.host_io = False
    g.capture()
    g.host_io = True
else:
    g.capture()
import time  # noqa: E402

time.sleep(2.0)  # the freshly written pinned feed settles (see bench.py)
for _ in range(300):
    g.step()
torch.cuda.synchronize()


def timeit(fn, k=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


print("graph alone us", timeit(lambda: g.graphs[0].replay()), "copy kernel alone us", timeit(lambda: g._h2d(0)),
      "CE copy alone us", timeit(lambda: g._raw[0].copy_(g._host_raw, non_blocking=True)))
N = 12
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
t0 = ev()
cs0, cs1, gs0, gs1 = [ev() for _ in range(N)], [ev() for _ in range(N)], [ev() for _ in range(N)], [ev() for _ in range(N)]
cur = torch.cuda.current_stream()
orig = g._issue_copy
step_i = [0]


def issue(k):
    c = g._cs[0]
    c.wait_event(g._used[k])
    cs0[step_i[0]].record(c)
    if g.copy_engine:
        with torch.cuda.stream(c):
            g._raw[k].copy_(g._host_raw, non_blocking=True)
    else:
        g._h2d(k, c)
    cs1[step_i[0]].record(c)
    g._copied[k].record(c)


g._issue_copy = issue
t0.record()
for i in range(N):
    step_i[0] = i
    k = g._step_count % 2
    cur.wait_event(g._copied[k])
    issue(k ^ 1)
    gs0[i].record(cur)
    g.graphs[k].replay()
    gs1[i].record(cur)
    g._used[k].record(cur)
    g._step_count += 1
torch.cuda.synchronize()
for i in range(N):
    f = lambda e: round(t0.elapsed_time(e) * 1000)  # noqa: E731
    print(f"step {i}: copy(next) {f(cs0[i])}-{f(cs1[i])} ({f(cs1[i]) - f(cs0[i])})  graph {f(gs0[i])}-{f(gs1[i])} "
          f"({f(gs1[i]) - f(gs0[i])})")
