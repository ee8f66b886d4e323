"""Memory-safety and race checks without compute-sanitizer (closed on this GPU pool: see
profiles/r2_sanitizer.md).
  * guard bands: every output the kernels write is a view into a larger buffer filled
    with a canary pattern; after the call the bytes before and after must be untouched
    (catches out-of-bounds writes of the rollout, render, GAE/score, level generation,
    mutation, PLR sample/export/digest paths);
  * determinism: repeated runs, and the two render implementations (quad tiles vs the
    per-observation legacy kernel, selected per process by AMZ_RENDER_LEGACY), must give
    bit-identical results -- a shared-memory race or a missing barrier shows up as
    run-to-run differences long before it corrupts a parity case."""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, LevelBuffer, PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAD = 4096  # guard bytes on each side


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


class Guarded:
    """Tensors carved out of canary-filled byte buffers."""

    def __init__(self):
        self.bufs = []

    def __call__(self, shape, dtype):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        raw = torch.full((n + 2 * PAD,), 0xA5, dtype=torch.uint8, device="cuda")
        self.bufs.append((raw, n))
        return raw[PAD:PAD + n].view(dtype).view(shape)

    def check(self):
        torch.cuda.synchronize()
        for raw, n in self.bufs:
            assert bool((raw[:PAD] == 0xA5).all()), "write before the start of an output"
            assert bool((raw[PAD + n:] == 0xA5).all()), "write past the end of an output"


@pytest.mark.parametrize("B,T,mode", [(100, 37, "resample"), (4096, 21, "resample"), (33, 9, "home"),
                                      (20000, 6, "resample")])
def test_rollout_and_score_outputs_stay_in_bounds(B, T, mode):
    g = Guarded()
    p = amz.StaticParams()
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)),
                               amz.RESAMPLE if mode == "resample" else amz.HOME)
    res = env.reset(amz.RngStream.from_seed(4), p)
    out = {"view": g((T, B, 5, 5), torch.uint8), "dir": g((T, B), torch.uint8), "rewards": g((T, B), torch.float64),
           "dones": g((T, B), torch.bool), "final_view": g((B, 5, 5), torch.uint8), "final_dir": g((B,), torch.uint8)}
    acts = torch.randint(0, 3, (T, B), dtype=torch.uint8, device="cuda")
    tr, cur = amz.rollout_actions(env, res, acts, p, out=out)
    gout = {"advantages": g((T, B), torch.float64), "returns": g((T, B), torch.float64),
            "scores": g((B,), torch.float64), "max_returns": g((B,), torch.float64)}
    vals = torch.rand((T, B), dtype=torch.float64, device="cuda")
    amz.gae_and_scores(tr.rewards, vals, tr.dones, vals[-1].clone(), 0.995, 0.98, out=gout)
    g.check()


def test_level_and_buffer_outputs_stay_in_bounds():
    g = Guarded()
    p = amz.StaticParams()
    lv = amz.sample_levels(amz.RngStream(1, (0,)), 777, p)
    mut = amz.mutate_levels(amz.RngStream(1, (3,)), lv, 20, p)
    buf = LevelBuffer(PlrConfig(buffer_size=500))
    sc = torch.rand(777, dtype=torch.float64, device="cuda")
    buf.update(lv, sc, sc, 0)
    buf.update(mut, sc, sc, 1)
    buf.digest(out=g((1,), torch.int64))
    seed = amz.RngStream(2, (1,)).seed_prefix()
    outs = [g((300,), torch.int32), g((300, 8), torch.int32), g((300,), torch.float64), g((300,), torch.float64)]
    import ctypes

    from paper_2311_12716_b200 import _lib

    _lib.call("amz_plr_sample", buf.handle, ctypes.byref(seed), 300, 0.3, _lib.ptr(buf.lut), 2,
              *(_lib.ptr(o) for o in outs), _lib.stream_handle("cuda"))
    g.check()


@pytest.mark.parametrize("n", [17, 4096, 16500])
def test_level_generation_and_dr_reset_stay_in_bounds(n):
    """Both level samplers (one warp per level below 16384, one thread per level from
    there: k_sample_levels_w / _t, k_env_reset_dr / _t) write only their outputs."""
    import ctypes

    from paper_2311_12716_b200 import _lib

    g = Guarded()
    p = amz.StaticParams()
    seed = amz.RngStream(1, (0,)).seed_prefix()
    out = g((n, 8), torch.int32)
    _lib.call("amz_sample_levels", ctypes.byref(p.c_struct()), ctypes.byref(seed), ctypes.c_uint32(0), None, n,
              _lib.ptr(out), _lib.stream_handle("cuda"))
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, n))
    lanes = benv._ensure(p)
    view, dirs = g((n, 5, 5), torch.uint8), g((n,), torch.int64)
    wrap = amz.RngStream(7, (1,)).seed_prefix()
    _lib.call("amz_env_reset_dr", lanes.handle, ctypes.byref(seed), ctypes.byref(wrap), _lib.ptr(view), _lib.ptr(dirs),
              lanes.stream())
    g.check()


def _rollout_digest(B, T, seed):
    p = amz.StaticParams()
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    acts = torch.randint(0, 3, (T, B), generator=g, dtype=torch.uint8, device="cuda")
    tr, cur = amz.rollout_actions(env, res, acts, p)
    return [x.cpu().numpy().copy() for x in (tr.obs["view"], tr.obs["dir"], tr.rewards, tr.dones, cur.obs["view"])]


def test_rollouts_are_deterministic():
    for B, T in ((4096, 64), (30000, 16)):
        a = _rollout_digest(B, T, 9)
        b = _rollout_digest(B, T, 9)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_render_implementations_agree():
    """quad-tile render (default) == legacy per-observation render, bit for bit."""
    code = ("import sys, hashlib; sys.path.insert(0, %r); from tests.test_gpu_guards import _rollout_digest; "
            "h = hashlib.sha256(); [h.update(x.tobytes()) for x in _rollout_digest(5000, 33, 3)]; "
            "print(h.hexdigest())") % ROOT
    outs = []
    for legacy in ("0", "1"):
        env = dict(os.environ, AMZ_RENDER_LEGACY=legacy)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


def test_plr_iterations_are_deterministic():
    def run():
        plr = ParallelPLR(700, amz.StaticParams(), PlrConfig(buffer_size=900), amz.RngStream.from_seed(2),
                          AccelConfig(20, 4))
        rng = np.random.default_rng(0)
        for it in range(4):
            L = plr.L
            plr.iteration(it, torch.from_numpy(rng.integers(0, 3, (12, L)).astype(np.uint8)).cuda(),
                          torch.from_numpy(np.round(rng.uniform(0, 0.3, (12, L)), 2)).cuda(),
                          torch.from_numpy(rng.uniform(0, 0.3, L)).cuda())
        return {k: v.cpu().numpy() for k, v in plr.buffer.export().items()}

    a, b = run(), run()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
