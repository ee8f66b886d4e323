"""PAIRED level designer on the GPU vs fixtures made by the reference
(amaze/teacher.py through batch_lift) and the numpy oracle on larger random batches."""

import numpy as np
import pytest

from oracle import amaze_np as onp

from .helpers import tensor_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["t13", "t9"])
def test_teacher_matches_reference(golden, tag):
    import torch

    import paper_2311_12716_b200 as amz

    z = golden(
        "teacher")
    H, W, budget, seed, B = (int(x) for x in z[f"{tag}_meta"])
    P = amz.StaticParams(height=H, width=W, wall_budget=budget)
    env = amz.batch_lift(amz.TeacherEnv(), amz.BatchShape(2, 1, B // 2))
    res = env.reset(amz.RngStream.from_seed(seed), P)
    c = lambda x: x.cpu().numpy()  # noqa: E731
    assert np.array_equal(c(res.observation["grid"]), z[f"{tag}_grid"][0])
    assert np.array_equal(c(res.observation["phase"]), z[f"{tag}_phase"][0])
    assert np.array_equal(c(res.observation["n_placed"]), z[f"{tag}_n_placed"][0])
    state = res.state
    for t in range(z[f"{tag}_actions"].shape[0]):
        r = env.step(None, state, torch.from_numpy(z[f"{tag}_actions"][t]).cuda(), P)
        state = r.state
        assert np.array_equal(c(r.observation["grid"]), z[f"{tag}_grid"][t + 1])
        assert np.array_equal(c(r.observation["phase"]), z[f"{tag}_phase"][t + 1])
        assert np.array_equal(c(r.observation["n_placed"]), z[f"{tag}_n_placed"][t + 1])
        assert np.array_equal(c(r.done), z[f"{tag}_done"][t])
        assert np.array_equal(c(r.info["time"]), z[f"{tag}_time"][t])
        assert not c(r.reward).any()
    assert np.array_equal(tensor_rows(env.designed_levels(state)), z[f"{tag}_levels"])
    # finished designs raise like TeacherEnv.step
    with pytest.raises(amz.ContractViolation):
        env.step(None, state, torch.zeros((2, B // 2), dtype=torch.int64), P)


def test_teacher_contract_errors():
    import torch

    import paper_2311_12716_b200 as amz

    P = amz.StaticParams()
    env = amz.batch_lift(amz.TeacherEnv(), amz.BatchShape(1, 1, 8))
    res = env.reset(amz.RngStream.from_seed(0), P)
    with pytest.raises(amz.ContractViolation):
        env.step(None, res.state, torch.full((1, 8), P.n_interior, dtype=torch.int64), P)
    res = env.reset(amz.RngStream.from_seed(0), P)
    env.step(None, res.state, torch.zeros((1, 8), dtype=torch.int64), P)
    with pytest.raises(amz.ContractViolation):  # unfinished designs do not decode
        env.designed_levels(res.state)


@pytest.mark.parametrize("hw,budget", [((13, 13), 60), ((11, 14), 40), ((6, 6), 14)])
def test_teacher_random_vs_oracle_and_paired_handoff(hw, budget):
    import torch

    import paper_2311_12716_b200 as amz

    H, W = hw
    P = amz.StaticParams(height=H, width=W, wall_budget=budget)
    B = 512
    env = amz.batch_lift(amz.TeacherEnv(), amz.BatchShape(1, 1, B))
    res = env.reset(amz.RngStream.from_seed(1), P)
    p = onp.Params(height=H, width=W, wall_budget=budget)
    lanes = [onp.Teacher(p) for _ in range(B)]
    g = np.random.default_rng(5)
    state = res.state
    for t in range(amz.TeacherEnv().episode_length(P)):
        a = g.integers(0, P.n_interior if t % 2 else 6, size=(1, B))
        r = env.step(None, state, torch.from_numpy(a).cuda(), P)
        state = r.state
        for ln, x in zip(lanes, a[0]):
            ln.step(x)
        grids = np.stack([ln.observe()[0] for ln in lanes])
        assert np.array_equal(r.observation["grid"].cpu().numpy()[0], grids)
    lv = env.designed_levels(state)
    rec = onp.pack_levels([ln.level() for ln in lanes], p)
    want = np.stack([rec["walls"][:, k] for k in range(4)] + [rec[f] for f in ("agent_r", "agent_c", "agent_dir",
                                                                               "goal_r", "goal_c")], axis=1)
    assert np.array_equal(tensor_rows(lv), want.astype(np.int64))
    # PAIRED hand-off: the designed levels go straight into the student env
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B))
    amz.check_levels(lv, P)
    out = benv.reset_to_levels(None, lv, P)
    assert out.observation["view"].shape[-1] == P.agent_view_size
