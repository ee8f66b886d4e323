"""Policy hand-off: the fused sample/log-prob kernel and the GPU
rollout() loop vs fixtures made by the reference (agents/rollout.py:87-152,
agents/ppo.py:82-96,136-138)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# exp/log are CUDA's: log-probabilities may differ from numpy's in the last ulp
LOGP_RTOL = 1e-14


@pytest.mark.parametrize("tag", ["a3f32", "a3", "a5", "a8", "a11", "wide"])
def test_policy_head_matches_reference(golden, tag):
    import torch

    import paper_2311_12716_b200 as amz

    z = golden("policy")
    lg = z[f"pa_{tag}_logits"]
    root = amz.RngStream.from_seed(31)
    for t in range(lg.shape[0]):
        x = torch.from_numpy(lg[t]).cuda()
        if tag == "a3f32":
            x = x.float()  # the model's float32 logits, cast to double inside the kernel
        a, lp = amz.policy_head(x, root.fold_in(t))
        want = z[f"pa_{tag}_actions"][t]
        assert np.array_equal(a.cpu().numpy(), want)
        ref = z[f"pa_{tag}_logp"][t][np.arange(len(want)), want]
        np.testing.assert_allclose(lp.cpu().numpy(), ref, rtol=LOGP_RTOL, atol=0)
        assert np.array_equal(amz.sample_actions(x, root.fold_in(t)).cpu().numpy(), want)


def test_policy_head_greedy_and_lane_offset(golden):
    import torch

    import paper_2311_12716_b200 as amz

    z = golden("policy")
    lg = z["pa_a5_logits"][0]
    a, _ = amz.policy_head(torch.from_numpy(lg).cuda(), greedy=True)
    assert np.array_equal(a.cpu().numpy(), lg.argmax(axis=-1))
    # a lane-sharded rank draws the global lanes' uniforms (lane0 offset)
    g = amz.RngStream.from_seed(31).fold_in(0)
    full, _ = amz.policy_head(torch.from_numpy(lg).cuda(), g)
    part, _ = amz.policy_head(torch.from_numpy(lg[150:]).cuda(), g, lane0=150)
    assert np.array_equal(part.cpu().numpy(), full.cpu().numpy()[150:])


class TorchExactActor:
    """The torch twin of make_golden._ExactActor (same exact integer arithmetic)."""

    def initial_hidden(self, n):
        import torch

        return torch.zeros((n, 2), dtype=torch.float64, device="cuda")

    def act(self, obs, hidden, g=None, greedy=False):
        import torch

        import paper_2311_12716_b200 as amz

        B = obs["dir"].shape[0]
        view = obs["view"].long().reshape(B, -1)
        d = obs["dir"].long()
        idx = torch.arange(view.shape[1], device=view.device)
        cols = [(((view + 1) * (a + 2 + idx % 3)) % 5).sum(dim=1).double() * 0.25 - 0.5 * ((d + a) % 4).double()
                for a in range(3)]
        logits = torch.stack(cols, dim=1)
        actions, logp = amz.policy_head(logits, g, greedy)
        values = 0.125 * (view.sum(dim=1) % 11).double() + 0.5 * d.double()
        hidden = hidden + torch.stack([torch.ones(B, dtype=torch.float64, device=view.device), d.double()], dim=1)
        return actions, logp, values, hidden


@pytest.mark.parametrize("tag,greedy", [("pr", False), ("prg", True)])
def test_policy_rollout_matches_reference(golden, tag, greedy):
    import paper_2311_12716_b200 as amz

    z = golden("policy")
    P = amz.StaticParams()
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 64)), amz.RESAMPLE)
    start = env.reset(amz.RngStream.from_seed(9), P)
    traj, cur = amz.rollout(amz.RngStream.from_seed(5), TorchExactActor(), env, start, 40, P, greedy=greedy)
    c = lambda x: x.cpu().numpy()  # noqa: E731
    assert np.array_equal(c(traj.obs["view"]), z[f"{tag}_view"])
    assert np.array_equal(c(traj.obs["dir"]), z[f"{tag}_dir"])
    assert np.array_equal(c(traj.actions), z[f"{tag}_actions"])
    assert np.array_equal(c(traj.values), z[f"{tag}_values"])
    assert np.array_equal(c(traj.rewards), z[f"{tag}_rewards"])
    assert np.array_equal(c(traj.dones), z[f"{tag}_dones"])
    assert np.array_equal(c(traj.pre_hidden), z[f"{tag}_pre_hidden"])
    np.testing.assert_allclose(c(traj.log_probs), z[f"{tag}_log_probs"], rtol=LOGP_RTOL, atol=0)
    assert np.array_equal(c(cur.obs["view"]), z[f"{tag}_cur_view"])
    assert np.array_equal(c(cur.obs["dir"]), z[f"{tag}_cur_dir"])
    assert np.array_equal(c(cur.hidden), z[f"{tag}_cur_hidden"])
    # continuing from the cursor equals one longer rollout
    env2 = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 64)), amz.RESAMPLE)
    s2 = env2.reset(amz.RngStream.from_seed(9), P)
    t1, c1 = amz.rollout(amz.RngStream.from_seed(5), TorchExactActor(), env2, s2, 25, P, greedy=greedy)
    assert np.array_equal(c(t1.actions), z[f"{tag}_actions"][:25])


@pytest.mark.parametrize("tag,greedy", [("pr", False), ("prg", True)])
def test_graph_rollout_matches_reference(golden, tag, greedy):
    """The CUDA-graph replayed rollout equals the reference; a second call (graph
    already captured) on the continued env equals the eager rollout's continuation."""
    import paper_2311_12716_b200 as amz

    z = golden("policy")
    P = amz.StaticParams()
    c = lambda x: x.cpu().numpy()  # noqa: E731
    env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 64)), amz.RESAMPLE)
    start = env.reset(amz.RngStream.from_seed(9), P)
    gr = amz.GraphRollout(TorchExactActor(), env, 40, greedy=greedy)
    traj, cur = gr(amz.RngStream.from_seed(5), start)
    assert np.array_equal(c(traj.obs["view"]), z[f"{tag}_view"])
    assert np.array_equal(c(traj.obs["dir"]), z[f"{tag}_dir"])
    assert np.array_equal(c(traj.actions), z[f"{tag}_actions"])
    assert np.array_equal(c(traj.values), z[f"{tag}_values"])
    assert np.array_equal(c(traj.rewards), z[f"{tag}_rewards"])
    assert np.array_equal(c(traj.dones), z[f"{tag}_dones"])
    assert np.array_equal(c(traj.pre_hidden), z[f"{tag}_pre_hidden"])
    np.testing.assert_allclose(c(traj.log_probs), z[f"{tag}_log_probs"], rtol=LOGP_RTOL, atol=0)
    assert np.array_equal(c(cur.obs["view"]), z[f"{tag}_cur_view"])
    assert np.array_equal(c(cur.hidden), z[f"{tag}_cur_hidden"])
    # replay path: continue both the graph env and an eager twin for another 40 steps
    env2 = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 64)), amz.RESAMPLE)
    s2 = env2.reset(amz.RngStream.from_seed(9), P)
    _, e_cur = amz.rollout(amz.RngStream.from_seed(5), TorchExactActor(), env2, s2, 40, P, greedy=greedy)
    e_traj, _ = amz.rollout(amz.RngStream.from_seed(6), TorchExactActor(), env2, e_cur, 40, P, greedy=greedy)
    g_traj, _ = gr(amz.RngStream.from_seed(6), cur)
    assert gr.graph is not None
    for name in ("actions", "rewards", "dones", "values", "pre_hidden"):
        assert np.array_equal(c(getattr(g_traj, name)), c(getattr(e_traj, name))), name
    assert np.array_equal(c(g_traj.obs["view"]), c(e_traj.obs["view"]))
    np.testing.assert_allclose(c(g_traj.log_probs), c(e_traj.log_probs), rtol=LOGP_RTOL, atol=0)
