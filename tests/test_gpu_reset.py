"""Fused DR reset (amz_env_reset_dr) vs the two-launch path it replaces.

VectorBatchEnv.reset = sample_levels + reset_to_levels (env/batch.py:86-95 over
amaze/generator.py:36-52); under AutoResetWrapper(RESAMPLE) the same launch also prepares
the timeout levels the first rollout would otherwise generate in k_spec_levels.  Every
output must be bit-identical to the unfused path, which test_gpu_parity pins to the oracle.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_2311_12716_b200 as amz  # noqa: E402

pytestmark = pytest.mark.gpu


def _pair(p, B, seed, mode=amz.RESAMPLE):
    rng = amz.RngStream.from_seed(seed)
    e1 = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
    e2 = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B)), mode)
    r1 = e1.reset(rng, p)
    rng_env, _ = rng.split(2)
    levels = amz.sample_levels(rng_env, B, p)
    r2 = e2.reset_to_levels(rng, levels, p)
    return e1, r1, e2, r2


def _same_traj(a, b):
    for k in ("view", "dir"):
        assert torch.equal(a.obs[k], b.obs[k]), k
    assert torch.equal(a.rewards, b.rewards)
    assert torch.equal(a.dones, b.dones)


def _same_cursor(a, b):
    for k in ("view", "dir"):
        assert torch.equal(a.obs[k], b.obs[k]), k
    assert torch.equal(a.state.state_table(), b.state.state_table())


# B >= 16384 runs the thread-per-level reset kernel (k_env_reset_dr_t), smaller B the
# warp-per-level one; both must equal sample_levels + reset_to_levels
@pytest.mark.parametrize("view,B", [(3, 777), (5, 777), (9, 777), (3, 16500), (5, 20000), (9, 16384)])
def test_reset_matches_sample_then_reset(view, B):
    p = amz.StaticParams(agent_view_size=view)
    e1, r1, e2, r2 = _pair(p, B, 31)
    assert torch.equal(r1.observation["view"], r2.observation["view"])
    assert torch.equal(r1.observation["dir"], r2.observation["dir"])
    assert torch.equal(r1.state.state_table(), r2.state.state_table())
    assert torch.equal(e1.benv.lane_levels_tensor(r1.state), e2.benv.lane_levels_tensor(r2.state))


@pytest.mark.parametrize("tep,T,B", [(20, 64, 1500), (9, 9, 1500), (5, 200, 1500), (20, 32, 16400)])
def test_prepared_timeout_levels_match(tep, T, B):
    """First RESAMPLE rollout after the fused reset (timeout levels prepared by the reset)
    equals the rollout after reset_to_levels (timeout levels from k_spec_levels)."""
    p = amz.StaticParams(max_episode_steps=tep)
    e1, r1, e2, r2 = _pair(p, B, 5)
    acts = torch.from_numpy(np.random.default_rng(2).integers(0, 3, (T, B)).astype(np.uint8)).cuda()
    t1, c1 = amz.rollout_actions(e1, r1, acts, p)
    t2, c2 = amz.rollout_actions(e2, r2, acts, p)
    _same_traj(t1, t2)
    _same_cursor(c1, c2)
    assert int(t1.dones.sum()) > 0
    # and the next chunk (no prepared levels any more) stays identical
    t1, _ = amz.rollout_actions(e1, c1, acts, p)
    t2, _ = amz.rollout_actions(e2, c2, acts, p)
    _same_traj(t1, t2)


def test_prepared_levels_unused_when_rollout_starts_later():
    """A short first chunk (T < timeout) never reaches the prepared step; the second
    chunk must regenerate its own timeout levels."""
    p = amz.StaticParams(max_episode_steps=30)
    B = 640
    e1, r1, e2, r2 = _pair(p, B, 8)
    rs = np.random.default_rng(3)
    for T in (7, 50, 50):
        acts = torch.from_numpy(rs.integers(0, 3, (T, B)).astype(np.uint8)).cuda()
        t1, r1 = amz.rollout_actions(e1, r1, acts, p)
        t2, r2 = amz.rollout_actions(e2, r2, acts, p)
        _same_traj(t1, t2)


def test_prepared_levels_dropped_on_other_key_or_step():
    p = amz.StaticParams(max_episode_steps=12)
    B = 512
    e1, r1, e2, r2 = _pair(p, B, 9)
    other = amz.RngStream.from_seed(1234)
    for r in (r1, r2):
        r.extras = dict(r.extras)
        r.extras[amz.AutoResetWrapper.EXTRAS_KEY] = {**r.extras[amz.AutoResetWrapper.EXTRAS_KEY], "rng": other}
    acts = torch.from_numpy(np.random.default_rng(4).integers(0, 3, (40, B)).astype(np.uint8)).cuda()
    t1, _ = amz.rollout_actions(e1, r1, acts, p)
    t2, _ = amz.rollout_actions(e2, r2, acts, p)
    _same_traj(t1, t2)


def test_home_mode_reset_matches():
    p = amz.StaticParams(max_episode_steps=10)
    B = 300
    e1, r1, e2, r2 = _pair(p, B, 10, amz.HOME)
    acts = torch.from_numpy(np.random.default_rng(6).integers(0, 3, (33, B)).astype(np.uint8)).cuda()
    t1, _ = amz.rollout_actions(e1, r1, acts, p)
    t2, _ = amz.rollout_actions(e2, r2, acts, p)
    _same_traj(t1, t2)


def test_single_steps_after_fused_reset():
    """Per-step API after the fused reset (prepared levels are not used by env_step)."""
    p = amz.StaticParams(max_episode_steps=6)
    B = 200
    e1, r1, e2, r2 = _pair(p, B, 11)
    rs = np.random.default_rng(7)
    for _ in range(15):
        a = torch.from_numpy(rs.integers(0, 3, (1, B))).cuda()
        r1 = e1.step(None, r1.state, a, p, r1.extras)
        r2 = e2.step(None, r2.state, a, p, r2.extras)
        assert torch.equal(r1.observation["view"], r2.observation["view"])
        assert torch.equal(r1.reward, r2.reward)
        assert torch.equal(r1.done, r2.done)
