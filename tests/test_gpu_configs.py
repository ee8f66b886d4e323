"""Parity at the BASELINE.json configurations themselves (not just small cases):
  * configs[1] headline: 4096 lanes x 256 steps RESAMPLE rollout + GAE/MaxMC, every
    output vs the oracle;
  * the HBM-roofline point: 65536 lanes x 256 steps (k_dyn<8,4>, k_gae_score7) on lane
    windows spread over the batch (the oracle keys lanes by global index, so a window
    is exact);
  * configs[4]: a 32768-lane PLR|| iteration (16384 new | 16384 replay) vs the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import amaze_np as onp  # noqa: E402
from oracle import plr_np  # noqa: E402
from tests.helpers import records_to_rows, tensor_rows  # noqa: E402

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import PlrConfig  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402

GAMMA, LAM = 0.995, 0.98


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rollout_and_score(B, T, seed, aseed):
    p = amz.StaticParams()
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    rng = np.random.default_rng(aseed)
    acts = rng.integers(0, 3, (T, B)).astype(np.uint8)
    vals = rng.uniform(0, 1, (T, B))
    last = rng.uniform(0, 1, B)
    tr, cur = amz.rollout_actions(env, res, torch.from_numpy(acts).cuda(), p)
    o = amz.gae_and_scores(tr.rewards, torch.from_numpy(vals).cuda(), tr.dones, torch.from_numpy(last).cuda(), GAMMA,
                           LAM)
    return acts, vals, last, tr, cur, o


def _check_window(seed, acts, vals, last, tr, cur, o, lo, hi):
    oenv = onp.AutoReset(hi - lo, onp.Params(), "resample", lane_offset=lo)
    obs0 = oenv.reset(seed)
    view, dirs, rew, dn, fobs = onp.rollout(oenv, obs0, acts[:, lo:hi])
    assert np.array_equal(tr.obs["view"][:, lo:hi].cpu().numpy(), view)
    assert np.array_equal(tr.obs["dir"][:, lo:hi].cpu().numpy(), dirs.astype(np.uint8))
    assert np.array_equal(tr.rewards[:, lo:hi].cpu().numpy(), rew)
    assert np.array_equal(tr.dones[:, lo:hi].cpu().numpy(), dn)
    assert np.array_equal(cur.obs["view"][lo:hi].cpu().numpy(), fobs["view"])
    adv, ret = onp.gae(rew, vals[:, lo:hi], dn, last[lo:hi], GAMMA, LAM)
    sc, mx, _ = onp.lane_scores(vals[:, lo:hi], adv, rew, dn, np.zeros(hi - lo))
    assert np.array_equal(o["advantages"][:, lo:hi].cpu().numpy(), adv)
    assert np.array_equal(o["returns"][:, lo:hi].cpu().numpy(), ret)
    assert np.array_equal(o["scores"][lo:hi].cpu().numpy(), sc)
    assert np.array_equal(o["max_returns"][lo:hi].cpu().numpy(), mx)


def test_headline_config_full_batch():
    """configs[1]: 4096 x 256, every lane and step."""
    B, T, seed = 4096, 256, 0
    acts, vals, last, tr, cur, o = _rollout_and_score(B, T, seed, 1)
    _check_window(seed, acts, vals, last, tr, cur, o, 0, B)


def test_hbm_point_65536_lanes_windows():
    B, T, seed = 65536, 256, 3
    acts, vals, last, tr, cur, o = _rollout_and_score(B, T, seed, 2)
    for lo, hi in ((0, 384), (32640, 33024), (65152, 65536)):
        _check_window(seed, acts, vals, last, tr, cur, o, lo, hi)


def test_config5_parallel_plr_32768_lanes():
    """configs[4] shape on one rank: 16384 new | 16384 replay lanes, K = 4000."""
    n, T, K, seed = 16384, 6, 4000, 5
    cfg = PlrConfig(buffer_size=K, staleness_coef=0.5, replay_rate=0.5)
    ocfg = plr_np.PlrConfig(buffer_size=K, staleness_coef=0.5, replay_rate=0.5)
    plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(seed), gamma=0.999, lam=0.95)
    ref = plr_np.LevelBuffer(K)
    rng = np.random.default_rng(8)
    p = onp.Params()
    for it in range(2):
        L = plr.L
        acts = rng.integers(0, 3, (T, L)).astype(np.uint8)
        vals = rng.uniform(0, 0.3, (T, L))
        last = rng.uniform(0, 0.3, L)
        res = plr.iteration(it, torch.from_numpy(acts).cuda(), torch.from_numpy(vals).cuda(),
                            torch.from_numpy(last).cuda())
        levels, prior, n_rep, _ = plr_np.compose_lanes(ref, seed, (), it, n, p, ocfg)
        env = onp.AutoReset(L, p, "home")
        obs = env.reset_to_levels(seed, (it, 4), onp.unpack_levels(levels, p))
        _, _, rew, dn, _ = onp.rollout(env, obs, acts)
        adv, _ = onp.gae(rew, vals, dn, last, 0.999, 0.95)
        sc, mx, _ = onp.lane_scores(vals, adv, rew, dn, prior, "maxmc")
        ref.update(levels, sc, mx, it)
        assert res.n_replay == n_rep
        assert np.array_equal(tensor_rows(res.levels), records_to_rows(levels))
        assert np.array_equal(res.scores.cpu().numpy(), sc)
        st = plr.buffer.export()
        size = int(st["meta"][0])
        assert size == ref.size and int(st["meta"][1]) == ref.next_seq
        assert np.array_equal(st["score"][:size].cpu().numpy(), ref.score[:size])
        assert np.array_equal(st["seq"][:size].cpu().numpy(), ref.seq[:size])
        assert np.array_equal(st["last_sampled"][:size].cpu().numpy(), ref.last_sampled[:size])
        assert np.array_equal(tensor_rows(st["levels"][:size]), records_to_rows(ref.levels[:size]))


@pytest.mark.parametrize("B", [512, 20000])
def test_successive_rollouts_reuse_the_env_counters(B):
    """One env, several reset + rollout rounds of different lengths: the render's per-group
    counters and (B > 18944) the persistent dynamics' work queue re-zero themselves between
    launches, so every round equals the oracle."""
    p = amz.StaticParams()
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    for rnd, T in enumerate((37, 256, 5, 100)):
        seed = 40 + rnd
        res = env.reset(amz.RngStream.from_seed(seed), p)
        rng = np.random.default_rng(seed)
        acts = rng.integers(0, 3, (T, B)).astype(np.uint8)
        vals = rng.uniform(0, 1, (T, B))
        last = rng.uniform(0, 1, B)
        tr, cur = amz.rollout_actions(env, res, torch.from_numpy(acts).cuda(), p)
        o = amz.gae_and_scores(tr.rewards, torch.from_numpy(vals).cuda(), tr.dones, torch.from_numpy(last).cuda(),
                               GAMMA, LAM)
        for lo, hi in ((0, 160), (B - 160, B)):
            _check_window(seed, acts, vals, last, tr, cur, o, lo, hi)
