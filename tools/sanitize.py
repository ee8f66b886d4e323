"""Small invocations of every hot-path kernel for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck):  compute-sanitizer --tool racecheck python tools/sanitize.py
Covers: smoke() (DR reset + RESAMPLE rollout + GAE/MaxMC vs the oracle), the HOME and
large-LPW rollout variants, float32-value GAE, the PLR buffer (update incl. insert runs,
bulk in-place runs and the sequential path; sample; top-q; digest), PLR||/ACCEL||
and PLR-perp iterations, the captured DR iteration, single steps, level metrics."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, LevelBuffer, PlrConfig  # noqa: E402
from paper_2311_12716_b200.graph import DRIterationGraph  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR, SequentialPLR  # noqa: E402

which = sys.argv[1:] or ["smoke", "rollout", "gae", "plr", "graph", "misc"]
p = amz.StaticParams()
T = 40
if "smoke" in which:
    __graft_entry__.smoke()
if "rollout" in which:
    for mode in (amz.HOME, amz.RESAMPLE):
        for B in (96, 3000):  # k_dyn<4,4> and (AMZ_DYN_LPW) variants
            env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
            res = env.reset(amz.RngStream.from_seed(1), p)
            acts = torch.randint(0, 3, (T, B), dtype=torch.uint8, device="cuda")
            tr, cur = amz.rollout_actions(env, res, acts, p)
            tr, cur = amz.rollout_actions(env, cur, acts, p)
    torch.cuda.synchronize()
    print("rollout ok")
if "gae" in which:
    for B in (40, 13000):
        r = torch.zeros((T, B), dtype=torch.float64, device="cuda")
        d = torch.rand((T, B), device="cuda") < 0.05
        r[d] = 0.5
        v = torch.rand((T, B), dtype=torch.float64, device="cuda")
        for vv in (v, v.float()):
            last = vv[-1].clone()
            for fn in ("maxmc", "pvl"):
                amz.gae_and_scores(r, vv, d, last, 0.995, 0.95, score_fn=fn)
    torch.cuda.synchronize()
    print("gae ok")
if "plr" in which:
    buf = LevelBuffer(PlrConfig(buffer_size=300))
    lv = amz.sample_levels(amz.RngStream(1, (0,)), 700, p)
    for it in range(4):
        sc = (torch.rand(700, dtype=torch.float64, device="cuda") * 4).floor() / 4
        buf.update(lv[(it * 200):(it * 200 + 500)], sc[:500], sc[:500], it)
        buf.update(buf.export()["levels"][:300], sc[:300], sc[:300], it)  # in-place bulk runs
        buf.sample(amz.RngStream(2, (it,)), 64, it)
        buf.digest()
    for accel in (None, AccelConfig(20, 4)):
        plr = ParallelPLR(64, p, PlrConfig(buffer_size=100), amz.RngStream.from_seed(3), accel)
        seq = SequentialPLR(64, p, PlrConfig(buffer_size=100, replay_rate=0.7), amz.RngStream.from_seed(4), accel)
        for it in range(4):
            L = plr.L
            plr.iteration(it, torch.randint(0, 3, (T, L), dtype=torch.uint8, device="cuda"),
                          torch.rand((T, L), dtype=torch.float64, device="cuda") * 0.2,
                          torch.rand((L,), dtype=torch.float64, device="cuda") * 0.2)
            seq.iteration(it, torch.randint(0, 3, (T, 64), dtype=torch.uint8, device="cuda"),
                          torch.rand((T, 64), dtype=torch.float64, device="cuda") * 0.2,
                          torch.rand((64,), dtype=torch.float64, device="cuda") * 0.2)
    torch.cuda.synchronize()
    print("plr ok")
if "graph" in which:
    gr = DRIterationGraph(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 128)), amz.RngStream.from_seed(5),
                          T, p, 0.995, 0.98, host_io=True).capture()
    for _ in range(3):
        gr.step()
    torch.cuda.synchronize()
    print("graph ok")
if "misc" in which:
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 64))
    env = amz.AutoResetWrapper(benv, amz.RESAMPLE)
    res = env.reset(amz.RngStream.from_seed(6), p)
    st, ex = res.state, res.extras
    for t in range(5):
        r = env.step(None, st, torch.randint(0, 3, (1, 64), device="cuda"), p, ex)
        st, ex = r.state, r.extras
    amz.level_metrics(amz.sample_levels(amz.RngStream(7, (0,)), 200, p), p)
    torch.cuda.synchronize()
    print("misc ok")
