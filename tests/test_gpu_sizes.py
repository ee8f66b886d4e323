"""CUDA path vs the numpy oracle over the size/shape edge cases the fast paths branch on:
odd lane counts (no vector/TMA stores), small/large view sizes and grids, occlusion,
T not a multiple of the kernels' chunk sizes, GAE pairwise plans with several leaves,
and the large-batch kernel variants."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import amaze_np as onp  # noqa: E402

import paper_2311_12716_b200 as amz  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _oparams(p):
    return onp.Params(p.height, p.width, p.max_episode_steps, p.agent_view_size, p.wall_budget, p.see_through_walls)


CASES = [
    # (B, T, params, mode)
    (37, 41, amz.StaticParams(), amz.RESAMPLE),
    (37, 70, amz.StaticParams(), amz.HOME),
    (300, 67, amz.StaticParams(see_through_walls=False), amz.RESAMPLE),
    (64, 90, amz.StaticParams(height=9, width=9, wall_budget=25, agent_view_size=3, max_episode_steps=40),
     amz.RESAMPLE),
    (96, 60, amz.StaticParams(agent_view_size=7, max_episode_steps=30), amz.RESAMPLE),
    (40, 50, amz.StaticParams(height=11, width=15, wall_budget=40, agent_view_size=9, max_episode_steps=20,
                              see_through_walls=False), amz.RESAMPLE),
    (128, 33, amz.StaticParams(max_episode_steps=5), amz.RESAMPLE),  # many resets per lane
]


@pytest.mark.parametrize("B,T,p,mode", CASES)
def test_fused_rollout_vs_oracle(B, T, p, mode):
    seed = 3
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    acts = np.random.default_rng(B + T).integers(0, 3, (T, B)).astype(np.uint8)
    tr, cur = amz.rollout_actions(env, res, torch.from_numpy(acts).cuda(), p)
    oenv = onp.AutoReset(B, _oparams(p), "home" if mode == amz.HOME else "resample")
    view, dirs, rew, dn, fobs = onp.rollout(oenv, oenv.reset(seed), acts)
    assert np.array_equal(tr.obs["view"].cpu().numpy(), view)
    assert np.array_equal(tr.obs["dir"].cpu().numpy(), dirs.astype(np.uint8))
    assert np.array_equal(tr.rewards.cpu().numpy(), rew)
    assert np.array_equal(tr.dones.cpu().numpy(), dn)
    assert np.array_equal(cur.obs["view"].cpu().numpy(), fobs["view"])


@pytest.mark.parametrize("B,T,p,mode", CASES[:4])
def test_step_api_vs_oracle(B, T, p, mode):
    seed = 4
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B))
    env = amz.AutoResetWrapper(benv, mode)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    oenv = onp.AutoReset(B, _oparams(p), "home" if mode == amz.HOME else "resample")
    oenv.reset(seed)
    acts = np.random.default_rng(7).integers(0, 3, (T, B))
    state, extras = res.state, res.extras
    for t in range(T):
        r = env.step(None, state, torch.from_numpy(acts[t]).cuda().reshape(1, B), p, extras)
        obs, rew, done, info = oenv.step(acts[t])
        assert np.array_equal(r.observation["view"].reshape(B, p.agent_view_size, -1).cpu().numpy(), obs["view"]), t
        assert np.array_equal(r.reward.reshape(B).cpu().numpy(), rew), t
        assert np.array_equal(r.done.reshape(B).cpu().numpy(), done), t
        assert np.array_equal(r.info["time"].reshape(B).cpu().numpy(), info["time"]), t
        state, extras = r.state, r.extras


def test_large_batch_kernels_vs_oracle():
    """4 x 148 x 32 lanes selects the large-batch dynamics kernel; 40000 lanes the
    single-warp GAE kernel; checked on a lane subset through the oracle."""
    p = amz.StaticParams()
    B, T, seed = 148 * 8 * 16 + 64, 40, 9
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    acts = np.random.default_rng(1).integers(0, 3, (T, B)).astype(np.uint8)
    tr, _ = amz.rollout_actions(env, res, torch.from_numpy(acts).cuda(), p)
    # lanes [B-256, B): an oracle env over exactly those global lanes
    lo = B - 256
    oenv = onp.AutoReset(256, onp.Params(), "resample", lane_offset=lo)
    view, dirs, rew, dn, _ = onp.rollout(oenv, oenv.reset(seed), acts[:, lo:])
    assert np.array_equal(tr.obs["view"][:, lo:].cpu().numpy(), view)
    assert np.array_equal(tr.rewards[:, lo:].cpu().numpy(), rew)
    assert np.array_equal(tr.dones[:, lo:].cpu().numpy(), dn)


@pytest.mark.parametrize("T,B", [(1, 5), (7, 33), (8, 64), (129, 17), (300, 40), (1000, 9), (256, 40000),
                                 (200, 16400), (256, 13000)])
def test_gae_scores_shapes(T, B):
    rng = np.random.default_rng(T * 7 + B)
    r = np.where(rng.uniform(size=(T, B)) < 0.05, rng.uniform(size=(T, B)), 0.0)
    v = rng.uniform(-1, 1, (T, B))
    d = rng.uniform(size=(T, B)) < 0.05
    last = rng.uniform(size=B)
    prior = rng.uniform(size=B) * (rng.uniform(size=B) < 0.3)
    for fn in ("maxmc", "pvl"):
        o = amz.gae_and_scores(*(torch.from_numpy(x).cuda() for x in (r, v, d, last)), 0.99, 0.9,
                               torch.from_numpy(prior).cuda(), fn)
        adv, ret = onp.gae(r, v, d, last, 0.99, 0.9)
        sc, mx, _ = onp.lane_scores(v, adv, r, d, prior, fn)
        assert np.array_equal(o["advantages"].cpu().numpy(), adv)
        assert np.array_equal(o["returns"].cpu().numpy(), ret)
        assert np.array_equal(o["scores"].cpu().numpy(), sc)
        assert np.array_equal(o["max_returns"].cpu().numpy(), mx)


def test_dr_levels_valid_and_distributed():
    """1000 DR levels pass MazeLevel invariants; wall counts spread over 0..60."""
    p = amz.StaticParams()
    lv = amz.sample_levels(amz.RngStream(11, (0,)), 4000, p)
    amz.check_levels(lv, p)
    host = amz.amaze.to_host_levels(lv, p)
    walls = np.array([h.n_interior_walls() for h in host])
    assert walls.min() == 0 and walls.max() == 60 and abs(walls.mean() - 30) < 1.5


@pytest.mark.gpu
@pytest.mark.parametrize("T,B", [(256, 4096), (256, 12288), (200, 16400), (256, 40000), (256, 13000), (129, 17),
                                 (300, 40)])
def test_gae_scores_f32_values(T, B):
    """Values as the policy's float32 (agents/ppo.py:96 widens them with .double()): the
    f32 entry equals the f64 path on the widened values, bit for bit, on every kernel."""
    rng = np.random.default_rng(T * 11 + B)
    r = np.where(rng.uniform(size=(T, B)) < 0.05, rng.uniform(size=(T, B)), 0.0)
    v32 = rng.uniform(-1, 1, (T, B)).astype(np.float32)
    d = rng.uniform(size=(T, B)) < 0.05
    last32 = rng.uniform(size=B).astype(np.float32)
    prior = rng.uniform(size=B) * (rng.uniform(size=B) < 0.3)
    v, last = v32.astype(np.float64), last32.astype(np.float64)
    adv, ret = onp.gae(r, v, d, last, 0.99, 0.9)
    for fn in ("maxmc", "pvl"):
        o = amz.gae_and_scores(torch.from_numpy(r).cuda(), torch.from_numpy(v32).cuda(), torch.from_numpy(d).cuda(),
                               torch.from_numpy(last32).cuda(), 0.99, 0.9, torch.from_numpy(prior).cuda(), fn,
                               with_stats=True)
        sc, mx, _ = onp.lane_scores(v, adv, r, d, prior, fn)
        assert np.array_equal(o["advantages"].cpu().numpy(), adv)
        assert np.array_equal(o["returns"].cpu().numpy(), ret)
        assert np.array_equal(o["scores"].cpu().numpy(), sc)
        assert np.array_equal(o["max_returns"].cpu().numpy(), mx)
        o64 = amz.gae_and_scores(torch.from_numpy(r).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(d).cuda(),
                                 torch.from_numpy(last).cuda(), 0.99, 0.9, torch.from_numpy(prior).cuda(), fn,
                                 with_stats=True)
        for k in ("episodes", "mean_return", "max_return", "solved_rate"):
            assert torch.equal(o["stats"][k], o64["stats"][k]), k
