"""CUDA path vs the reference (golden fixtures) and vs the oracle -- bit-exact.

Every call goes through the C ABI (libamaze_b200.so) via the drop-in Python layer."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import amaze_np as onp  # noqa: E402
from oracle import corc  # noqa: E402
from tests.helpers import records_to_rows, rows_to_records, tensor_rows  # noqa: E402

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.level import records_to_tensor  # noqa: E402

LEVEL_CASES = ["default", "seed12345", "budget0", "budget1", "budget119", "small9", "bigseed"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", LEVEL_CASES)
def test_sample_levels_bit_exact(golden, name):
    z = golden("levels")
    H, W, budget, seed, n = (int(x) for x in z[f"lv_{name}_meta"])
    p = amz.StaticParams(height=H, width=W, wall_budget=budget)
    got = amz.sample_levels(amz.RngStream(seed, (0,)), n, p)
    assert np.array_equal(tensor_rows(got), z[f"lv_{name}"])


@pytest.mark.parametrize("name", ["default", "budget0", "budget119", "small9"])
@pytest.mark.parametrize("edits", [1, 20])
def test_mutate_levels_bit_exact(golden, name, edits):
    z = golden("levels")
    H, W, budget, seed, n = (int(x) for x in z[f"lv_{name}_meta"])
    p = amz.StaticParams(height=H, width=W, wall_budget=budget)
    parents = records_to_tensor(rows_to_records(z[f"lv_{name}"]))
    got = amz.mutate_levels(amz.RngStream(seed, (7,)), parents, edits, p)
    assert np.array_equal(tensor_rows(got), z[f"mut{edits}_{name}"])


def test_single_level_dropins(golden):
    z = golden("levels")
    p = amz.StaticParams()
    lv = amz.sample_random_level(amz.RngStream(0, (0, 5)), p)
    assert tensor_rows(amz.amaze.to_device_levels([lv], p))[0].tolist() == z["lv_default"][5].tolist()
    mut = amz.mutate_level(amz.RngStream(0, (7, 5)), lv, 20, p)
    assert tensor_rows(amz.amaze.to_device_levels([mut], p))[0].tolist() == z["mut20_default"][5].tolist()


def _make_env(z, name):
    na, ne, nv, T, seed, aseed, home, st = (int(x) for x in z[f"{name}_meta"])
    p = amz.StaticParams(see_through_walls=bool(st))
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(na, ne, nv))
    env = amz.AutoResetWrapper(benv, amz.HOME if home else amz.RESAMPLE)
    return env, p, (na, ne, nv, T, seed, aseed, home)


def _reset(env, p, z, name, golden, seed, home):
    if home:
        assets = records_to_tensor(rows_to_records(golden("views")["asset_levels"]))
        return env.reset_to_levels(amz.RngStream.from_seed(seed), assets, p)
    return env.reset(amz.RngStream.from_seed(seed), p)


@pytest.mark.parametrize("name", ["cfg1", "hier", "occl", "home"])
def test_step_api_matches_reference(golden, name):
    z = golden("rollouts")
    env, p, (na, ne, nv, T, seed, aseed, home) = _make_env(z, name)
    res = _reset(env, p, z, name, golden, seed, home)
    B = na * ne * nv
    assert np.array_equal(res.observation["view"].reshape(B, 5, 5).cpu().numpy(), z[f"{name}_view0"])
    assert np.array_equal(res.observation["dir"].reshape(B).cpu().numpy(), z[f"{name}_dir0"])
    acts = torch.from_numpy(z[f"{name}_actions"].astype(np.int64)).cuda()
    state, extras = res.state, res.extras
    views, dirs, rews, dones, solved, times = [], [], [], [], [], []
    for t in range(T):
        r = env.step(None, state, acts[t].reshape(na, ne * nv), p, extras)
        assert r.observation["view"].shape == (na, ne * nv, 5, 5)
        assert r.observation["dir"].dtype == torch.int64 and r.reward.dtype == torch.float64
        assert r.done.dtype == torch.bool and r.info["time"].dtype == torch.int64
        views.append(r.observation["view"].reshape(B, 5, 5)); dirs.append(r.observation["dir"].reshape(B))
        rews.append(r.reward.reshape(B)); dones.append(r.done.reshape(B))
        solved.append(r.info["solved"].reshape(B)); times.append(r.info["time"].reshape(B))
        state, extras = r.state, r.extras
    assert np.array_equal(torch.stack(views).cpu().numpy(), z[f"{name}_view"])
    assert np.array_equal(torch.stack(dirs).cpu().numpy(), z[f"{name}_dir"])
    assert np.array_equal(torch.stack(rews).cpu().numpy(), z[f"{name}_reward"])
    assert np.array_equal(torch.stack(dones).cpu().numpy(), z[f"{name}_done"])
    assert np.array_equal(torch.stack(solved).cpu().numpy(), z[f"{name}_solved"])
    assert np.array_equal(torch.stack(times).cpu().numpy(), z[f"{name}_time"])
    assert np.array_equal(tensor_rows(env.benv.lane_levels_tensor(state)), z[f"{name}_final_levels"])


@pytest.mark.parametrize("name", ["cfg1", "hier", "occl", "home"])
def test_fused_rollout_matches_reference(golden, name):
    z = golden("rollouts")
    env, p, (na, ne, nv, T, seed, aseed, home) = _make_env(z, name)
    res = _reset(env, p, z, name, golden, seed, home)
    B = na * ne * nv
    acts = torch.from_numpy(z[f"{name}_actions"]).cuda()
    # two chunks to exercise the cursor / step counter carry-over
    t1 = T // 3
    tr1, cur = amz.rollout_actions(env, res, acts[:t1], p)
    tr2, cur = amz.rollout_actions(env, cur, acts[t1:], p)
    view = torch.cat([tr1.obs["view"], tr2.obs["view"]]).cpu().numpy()
    dirs = torch.cat([tr1.obs["dir"], tr2.obs["dir"]]).cpu().numpy()
    want_view = np.concatenate([z[f"{name}_view0"][None], z[f"{name}_view"][:-1]])
    want_dir = np.concatenate([z[f"{name}_dir0"][None], z[f"{name}_dir"][:-1]]).astype(np.uint8)
    assert np.array_equal(view, want_view)
    assert np.array_equal(dirs, want_dir)
    assert np.array_equal(torch.cat([tr1.rewards, tr2.rewards]).cpu().numpy(), z[f"{name}_reward"])
    assert np.array_equal(torch.cat([tr1.dones, tr2.dones]).cpu().numpy(), z[f"{name}_done"])
    assert np.array_equal(cur.obs["view"].cpu().numpy(), z[f"{name}_view"][-1])
    assert np.array_equal(cur.obs["dir"].cpu().numpy(), z[f"{name}_dir"][-1])
    assert np.array_equal(tensor_rows(env.benv.lane_levels_tensor(cur.state)), z[f"{name}_final_levels"])
    del B


def test_views_match_reference(golden):
    z = golden("views")
    for st in (0, 1):
        p = amz.StaticParams(see_through_walls=bool(st))
        lv = records_to_tensor(rows_to_records(z["st_levels"]))
        benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, lv.shape[0]))
        res = benv.reset_to_levels(None, lv, p)
        poses = torch.from_numpy(z["st_poses"]).cuda()
        table = res.state.state_table()
        table[:, 0:3] = poses.to(torch.int32)
        res.state.set_state_table(table)
        obs = res.state.observe()
        assert np.array_equal(obs["view"].cpu().numpy(), z[f"st_view_st{st}"])
        al = records_to_tensor(rows_to_records(z["asset_levels"]))
        benv2 = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, al.shape[0]))
        r2 = benv2.reset_to_levels(None, al, p)
        assert np.array_equal(r2.observation["view"][0].cpu().numpy(), z[f"asset_view_st{st}"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_gae_and_scores_bit_exact(golden, tag):
    z = golden("scores")
    g, lam = (float(x) for x in z[f"sc_{tag}_gl"])
    r, v, d, last, prior = (torch.from_numpy(z[k]).cuda() for k in ("sc_r", "sc_v", "sc_d", "sc_last", "sc_prior"))
    adv, ret = amz.compute_gae(r, v, d, last, g, lam)
    assert np.array_equal(adv.cpu().numpy(), z[f"sc_{tag}_adv"])
    assert np.array_equal(ret.cpu().numpy(), z[f"sc_{tag}_ret"])
    for fn in ("maxmc", "pvl"):
        for disc in (0, 1):
            o = amz.gae_and_scores(r, v, d, last, g, lam, prior, fn, bool(disc), with_stats=True)
            assert np.array_equal(o["scores"].cpu().numpy(), z[f"sc_{tag}_{fn}_{disc}_score"]), (fn, disc)
            assert np.array_equal(o["max_returns"].cpu().numpy(), z[f"sc_{tag}_{fn}_{disc}_maxret"])

            class Cfg:
                score_fn, maxmc_discounted = fn, bool(disc)

            class Tr:
                rewards, values, dones = r, v, d

            s, m = amz.lane_scores(Tr, adv, prior, Cfg, gamma=g)
            assert np.array_equal(s.cpu().numpy(), z[f"sc_{tag}_{fn}_{disc}_score"])
            assert np.array_equal(m.cpu().numpy(), z[f"sc_{tag}_{fn}_{disc}_maxret"])
    st = amz.per_lane_episode_stats(r, d, g)
    for k in ("episodes", "mean_return", "max_return", "solved_rate"):
        assert np.array_equal(st[k].cpu().numpy(), z[f"sc_{tag}_stats_{k}"]), k


def test_known_answers():
    assert amz.score_pvl(np.array([0.5, -0.2, 0.3])) == 0.26666666666666666
    assert amz.score_maxmc(np.full(7, 0.2), 1.0) == pytest.approx(0.8)
    assert amz.score_maxmc(np.full(3, 2.0), 1.0) == -1.0  # unclamped, like the reference
    adv, _ = amz.compute_gae(np.ones((3, 1)), np.zeros((3, 1)), np.zeros((3, 1), bool), np.zeros(1), 1.0, 1.0)
    assert adv[:, 0].tolist() == [3.0, 2.0, 1.0]


def test_bare_step_on_terminal_lanes_raises():
    p = amz.StaticParams(max_episode_steps=2)
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 8))
    res = benv.reset(amz.RngStream(3, (0,)), p)
    a = torch.zeros((1, 8), dtype=torch.int64, device="cuda")
    r1 = benv.step(None, res.state, a, p)
    r2 = benv.step(None, r1.state, a, p)
    assert bool(r2.done.all())
    before = r2.state.state_table().clone()
    with pytest.raises(amz.ContractViolation):
        benv.step(None, r2.state, a, p)
    assert torch.equal(before, r2.state.state_table())  # untouched, as step_batch raises first
    with pytest.raises(amz.ShapeError):
        benv.step(None, r2.state, torch.zeros((1, 7), dtype=torch.int64, device="cuda"), p)


def test_invalid_actions_are_noops():
    """step_batch treats unknown action codes as no-ops that still advance time."""
    p = amz.StaticParams()
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 16))
    res = benv.reset(amz.RngStream(4, (0,)), p)
    before = res.state.state_table().clone()
    r = benv.step(None, res.state, torch.full((1, 16), 7, dtype=torch.int64, device="cuda"), p)
    after = r.state.state_table()
    assert torch.equal(before[:, :3], after[:, :3])
    assert bool((after[:, 3] == 1).all())


@pytest.mark.parametrize("B,T", [(1000, 300), (4096, 64)])
def test_large_rollout_vs_oracle(B, T):
    """Full RESAMPLE rollout vs the numpy oracle at a size the oracle finishes quickly."""
    p = amz.StaticParams()
    seed = 21
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), amz.RESAMPLE)
    res = env.reset(amz.RngStream.from_seed(seed), p)
    acts_np = np.random.default_rng(5).integers(0, 3, (T, B)).astype(np.uint8)
    tr, cur = amz.rollout_actions(env, res, torch.from_numpy(acts_np).cuda(), p)
    oenv = onp.AutoReset(B, onp.Params(), "resample")
    obs0 = oenv.reset(seed)
    view, dirs, rew, dn, fobs = onp.rollout(oenv, obs0, acts_np)
    assert np.array_equal(tr.obs["view"].cpu().numpy(), view)
    assert np.array_equal(tr.obs["dir"].cpu().numpy(), dirs.astype(np.uint8))
    assert np.array_equal(tr.rewards.cpu().numpy(), rew)
    assert np.array_equal(tr.dones.cpu().numpy(), dn)
    assert np.array_equal(cur.obs["view"].cpu().numpy(), fobs["view"])


def test_many_levels_vs_c_oracle():
    """100k DR levels and mutants vs the C restatement (pinned to the reference)."""
    p = amz.StaticParams()
    n = 100_000
    got = amz.sample_levels(amz.RngStream(77, (0,)), n, p)
    want = corc.sample_levels(77, (0,), 0, n)
    assert np.array_equal(tensor_rows(got), records_to_rows(want))
    mut = amz.mutate_levels(amz.RngStream(77, (9,)), got, 20, p)
    wmut = corc.mutate_levels(77, (9,), 0, want, 20)
    assert np.array_equal(tensor_rows(mut), records_to_rows(wmut))
    amz.check_levels(mut, p)


def test_check_levels_rejects_bad():
    p = amz.StaticParams()
    lv = amz.sample_levels(amz.RngStream(1, (0,)), 4, p)
    bad = lv.clone()
    bad[2, 4] = (bad[2, 4] & ~0xFF) | 0  # agent row 0 (border)
    with pytest.raises(amz.LevelError):
        amz.check_levels(bad, p)


def test_reset_lanes_and_levels():
    p = amz.StaticParams()
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 2, 3))
    res = benv.reset(amz.RngStream(8, (0,)), p)
    fresh = amz.sample_levels(amz.RngStream(9, (0,)), 2, p)
    st, obs = benv.reset_lanes(res.state, [1, 4], fresh, p)
    lv = benv.lane_levels_tensor(st)
    assert torch.equal(lv[1], fresh[0]) and torch.equal(lv[4], fresh[1])
    assert obs["view"].shape == (2, 5, 5)
    host = benv.lane_levels(st)
    assert len(host) == 6 and host[1] == amz.amaze.to_host_levels(fresh, p)[0]
