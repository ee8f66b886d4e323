"""numpy oracle (oracle/amaze_np.py) pinned against fixtures produced by the reference."""

import numpy as np
import pytest

from oracle import amaze_np as onp


def _levels_from_rows(rows, p):
    rec = np.zeros(len(rows), dtype=onp.LEVEL_DTYPE)
    rec["walls"] = rows[:, :4].astype(np.uint32)
    rec["agent_r"], rec["agent_c"], rec["agent_dir"] = rows[:, 4], rows[:, 5], rows[:, 6]
    rec["goal_r"], rec["goal_c"] = rows[:, 7], rows[:, 8]
    return onp.unpack_levels(rec, p)


@pytest.mark.parametrize("name", ["cfg1", "hier", "occl", "home"])
def test_rollout_matches_reference(golden, name):
    z = golden("rollouts")
    na, ne, nv, T, seed, aseed, home, st = (int(x) for x in z[f"{name}_meta"])
    B = na * ne * nv
    p = onp.Params(see_through_walls=bool(st))
    env = onp.AutoReset(B, p, "home" if home else "resample")
    if name == "home":
        asset = _levels_from_rows(golden("views")["asset_levels"], p)
        inner = [asset[i % nv] for i in range(ne * nv)]
        obs = env.reset_to_levels(seed, (0,), inner * na)
    else:
        obs = env.reset(seed)
    assert np.array_equal(obs["view"], z[f"{name}_view0"])
    acts = z[f"{name}_actions"]
    assert np.array_equal(acts, onp.random_actions(aseed, T, B))
    for t in range(T):
        obs, rew, done, info = env.step(acts[t])
        assert np.array_equal(obs["view"], z[f"{name}_view"][t]), t
        assert np.array_equal(obs["dir"], z[f"{name}_dir"][t]), t
        assert np.array_equal(rew, z[f"{name}_reward"][t]), t
        assert np.array_equal(done, z[f"{name}_done"][t]), t
        assert np.array_equal(info["solved"], z[f"{name}_solved"][t])
        assert np.array_equal(info["time"], z[f"{name}_time"][t])


def test_views_match_reference(golden):
    z = golden("views")
    for st in (0, 1):
        p = onp.Params(see_through_walls=bool(st))
        levels = _levels_from_rows(z["st_levels"], p)
        lanes = onp.Lanes(levels)
        lanes.pos = z["st_poses"][:, :2].copy()
        lanes.dir = z["st_poses"][:, 2].copy()
        assert np.array_equal(onp.observe(lanes, p)["view"], z[f"st_view_st{st}"])
        al = _levels_from_rows(z["asset_levels"], p)
        assert np.array_equal(onp.observe(onp.Lanes(al), p)["view"], z[f"asset_view_st{st}"])


def test_labyrinth_start_view(golden):
    """Labyrinth start view, dir N."""
    z = golden("views")
    names = list(z["asset_names"])
    v = z["asset_view_st1"][names.index("Labyrinth")]
    assert v.tolist() == [[3, 1, 0, 1, 0], [3, 1, 0, 1, 0], [3, 1, 0, 1, 0], [3, 1, 0, 1, 1], [3, 1, 0, 0, 0]]


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_gae_scores_match_reference(golden, tag):
    z = golden("scores")
    g, lam = z[f"sc_{tag}_gl"]
    adv, ret = onp.gae(z["sc_r"], z["sc_v"], z["sc_d"], z["sc_last"], g, lam)
    assert np.array_equal(adv, z[f"sc_{tag}_adv"])
    assert np.array_equal(ret, z[f"sc_{tag}_ret"])
    for fn in ("maxmc", "pvl"):
        for disc in (0, 1):
            s, m, _ = onp.lane_scores(z["sc_v"], adv, z["sc_r"], z["sc_d"], z["sc_prior"], fn, g, bool(disc))
            assert np.array_equal(s, z[f"sc_{tag}_{fn}_{disc}_score"])
            assert np.array_equal(m, z[f"sc_{tag}_{fn}_{disc}_maxret"])
    st = onp.episode_stats(z["sc_r"], z["sc_d"], g)
    for k in ("episodes", "mean_return", "max_return", "solved_rate"):
        assert np.array_equal(st[k], z[f"sc_{tag}_stats_{k}"])


def test_known_answers(golden):
    z = golden("scores")
    assert z["ka_pvl"][0] == 0.26666666666666666
    assert z["ka_maxmc"][0] == pytest.approx(0.8)
    adv, _ = onp.gae(np.ones((3, 1)), np.zeros((3, 1)), np.zeros((3, 1)), np.zeros(1), 1.0, 1.0)
    assert adv[:, 0].tolist() == [3.0, 2.0, 1.0]


@pytest.mark.parametrize("name", ["default", "dense", "small9", "wide", "assets"])
def test_env_metrics_match_reference(golden, name):
    """oracle env_metrics == the reference's amaze/metrics.py:21 on fixtures it produced."""
    z = golden("metrics")
    H, W = (int(x) for x in z[f"m_{name}_meta"])
    p = onp.Params(height=H, width=W)
    levels = _levels_from_rows(z[f"m_{name}_levels"], p)
    got = np.array([onp.env_metrics(lv) for lv in levels], dtype=object)
    assert np.array_equal(got[:, 0].astype(np.int64), z[f"m_{name}_nwalls"])
    assert np.array_equal(got[:, 1].astype(np.int64), z[f"m_{name}_spl"])
    assert np.array_equal(got[:, 2].astype(bool), z[f"m_{name}_solvable"])
    assert np.array_equal(got[:, 3].astype(np.float64), z[f"m_{name}_passable"])


@pytest.mark.parametrize("tag", ["a3f32", "a3", "a5", "a8", "a11", "wide"])
def test_sample_actions_oracle_matches_reference(golden, tag):
    z = golden("policy")
    lg = z[f"pa_{tag}_logits"]
    for t in range(lg.shape[0]):
        g = onp.generator(31, (t,))
        assert np.array_equal(onp.sample_actions(lg[t], g), z[f"pa_{tag}_actions"][t])
        assert np.array_equal(onp.log_softmax(lg[t]), z[f"pa_{tag}_logp"][t])


@pytest.mark.parametrize("tag", ["t13", "t9"])
def test_teacher_oracle_matches_reference(golden, tag):
    z = golden("teacher")
    H, W, budget, seed, B = (int(x) for x in z[f"{tag}_meta"])
    p = onp.Params(height=H, width=W, wall_budget=budget)
    lanes = [onp.Teacher(p) for _ in range(B)]
    acts = z[f"{tag}_actions"].reshape(z[f"{tag}_actions"].shape[0], -1)
    for t in range(acts.shape[0] + 1):
        obs = [ln.observe() for ln in lanes]
        assert np.array_equal(np.stack([o[0] for o in obs]), z[f"{tag}_grid"][t].reshape(B, H, W))
        assert np.array_equal(np.stack([o[1] for o in obs]), z[f"{tag}_phase"][t].reshape(B, 4))
        assert np.array_equal(np.array([o[2] for o in obs]), z[f"{tag}_n_placed"][t].reshape(B))
        if t < acts.shape[0]:
            for ln, a in zip(lanes, acts[t]):
                ln.step(a)
    assert np.array_equal(onp_rows([ln.level() for ln in lanes], p), z[f"{tag}_levels"])


def onp_rows(levels, p):
    rec = onp.pack_levels(levels, p)
    return np.stack([rec["walls"][:, 0], rec["walls"][:, 1], rec["walls"][:, 2], rec["walls"][:, 3],
                     rec["agent_r"], rec["agent_c"], rec["agent_dir"], rec["goal_r"], rec["goal_c"]],
                    axis=1).astype(np.int64)
