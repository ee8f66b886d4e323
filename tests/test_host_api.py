"""Host-side API pieces that need no GPU: TrajectoryBatch (agents/rollout.py:19-70),
reset_lanes index rules, the bench's --gpus launcher, the PLR-perp oracle's SPEC
examples."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2311_12716_b200.batch import _lane_indices
from paper_2311_12716_b200.rollout import TrajectoryBatch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"


def _traj(T=5, B=4, seed=0):
    g = torch.Generator().manual_seed(seed)
    return TrajectoryBatch({"view": torch.randint(0, 4, (T, B, 5, 5), generator=g, dtype=torch.uint8),
                            "dir": torch.randint(0, 4, (T, B), generator=g)},
                           torch.randint(0, 3, (T, B), generator=g), torch.rand((T, B), generator=g, dtype=torch.float64),
                           torch.rand((T, B), generator=g, dtype=torch.float64),
                           torch.rand((T, B), generator=g, dtype=torch.float64), torch.rand((T, B), generator=g) < 0.3,
                           torch.rand((T, B, 3), generator=g))


def test_trajectory_field_order_matches_reference():
    import dataclasses

    names = [f.name for f in dataclasses.fields(TrajectoryBatch)]
    assert names == ["obs", "actions", "log_probs", "values", "rewards", "dones", "pre_hidden"]


def test_trajectory_methods_match_reference_semantics():
    tb = _traj()
    m = tb.reset_masks()
    assert m.dtype == torch.bool and not m[0].any() and torch.equal(m[1:], tb.dones[:-1])
    sl = tb.lane_slice([3, 1])
    assert torch.equal(sl.rewards, tb.rewards[:, [3, 1]]) and torch.equal(sl.obs["view"], tb.obs["view"][:, [3, 1]])
    assert torch.equal(sl.pre_hidden, tb.pre_hidden[:, [3, 1]])
    cat = TrajectoryBatch.concat_lanes([tb.lane_slice([0, 1]), tb.lane_slice([2, 3])])
    for f in TrajectoryBatch.FIELDS:
        assert torch.equal(getattr(cat, f), getattr(tb, f)), f
    # the fused action-stream rollout leaves the policy fields empty: they stay None
    bare = TrajectoryBatch(tb.obs, tb.actions, None, None, tb.rewards, tb.dones)
    assert TrajectoryBatch.concat_lanes([bare.lane_slice([0]), bare.lane_slice([1])]).values is None


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_trajectory_methods_equal_reference_on_the_same_arrays():
    """Same arrays through the reference's own TrajectoryBatch (numpy) and ours (torch)."""
    sys.path.insert(0, REF_SRC)
    try:
        import importlib

        R = importlib.import_module("autocurricula.agents.rollout")
    finally:
        sys.path.remove(REF_SRC)
    tb = _traj(seed=3)
    rt = R.TrajectoryBatch({k: v.numpy() for k, v in tb.obs.items()},
                           *(getattr(tb, f).numpy() for f in TrajectoryBatch.FIELDS))
    assert np.array_equal(rt.reset_masks(), tb.reset_masks().numpy())
    lanes = np.array([2, 0])
    a, b = rt.lane_slice(lanes), tb.lane_slice(lanes)
    for f in TrajectoryBatch.FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f).numpy()), f
    c1 = R.TrajectoryBatch.concat_lanes([rt.lane_slice(np.array([1])), rt.lane_slice(np.array([3, 0]))])
    c2 = TrajectoryBatch.concat_lanes([tb.lane_slice([1]), tb.lane_slice([3, 0])])
    for f in TrajectoryBatch.FIELDS:
        assert np.array_equal(getattr(c1, f), getattr(c2, f).numpy()), f


def test_lane_indices_follow_numpy_indexing():
    assert _lane_indices([0, -1, 2], 4).tolist() == [0, 3, 2]
    assert _lane_indices(np.array([True, False, True, False]), 4).tolist() == [0, 2]
    assert _lane_indices(torch.tensor([1, 3]), 4).tolist() == [1, 3]
    for bad in ([4], [-5], np.array([True, False])):
        with pytest.raises(IndexError):
            _lane_indices(bad, 4)
    with pytest.raises(IndexError):
        _lane_indices([0.5], 4)


def test_bench_gpus_flag_starts_that_many_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself with a world of 2 (the
    launcher-only mode does no GPU work, so this runs on CPU)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line == {"launcher_check": True, "world": 2, "ranks_seen": 2}


def test_plr_perp_oracle_spec_examples():
    """SPEC.md:391-399 examples on the oracle: p=0 -> always NEW; an empty buffer -> NEW
    even at p=1; ACCEL -> exactly q mutants per replay iteration."""
    from oracle import amaze_np as onp
    from oracle import plr_np

    p = onp.Params()
    calls = []

    def fake_rollout(levels, prior, key, which):
        calls.append(which)
        n = len(levels)
        return np.linspace(0.1, 0.9, n), np.zeros(n)

    buf = plr_np.LevelBuffer(16)
    for it in range(3):
        out = plr_np.plr_perp_iteration(buf, 1, (), it, 8, p, plr_np.PlrConfig(buffer_size=16, replay_rate=0.0),
                                        fake_rollout)
        assert out["branch"] == "new"
    buf2 = plr_np.LevelBuffer(16)
    cfg = plr_np.PlrConfig(buffer_size=16, replay_rate=1.0)
    assert plr_np.plr_perp_iteration(buf2, 1, (), 0, 8, p, cfg, fake_rollout)["branch"] == "new"
    calls.clear()
    out = plr_np.plr_perp_iteration(buf2, 1, (), 1, 8, p, cfg, fake_rollout, accel=(4, 20))
    assert out["branch"] == "replay" and len(out["mutants"]) == 4 and calls == ["main", "mutants"]


def test_stream_uniform_matches_numpy():
    """amz_stream_uniform (host C) == numpy's first Generator.random() of the stream."""
    import ctypes

    import numpy as np

    from paper_2311_12716_b200 import RngStream, _lib

    for entropy, key in [(0, ()), (7, (3,)), (11, (5, 0)), (2 ** 40 + 3, (1, 2, 3)), (123456789, (2 ** 31 + 5, 9))]:
        s = RngStream(entropy, key)
        u = ctypes.c_double(0.0)
        _lib.call("amz_stream_uniform", ctypes.byref(s.seed_prefix()), ctypes.byref(u))
        want = np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy=entropy, spawn_key=key))).random()
        assert u.value == want, (entropy, key)
