"""The PLR buffer oracle (oracle/plr_np.py) against SPEC.md's known answers (CPU only)."""

import numpy as np
import pytest

from oracle import amaze_np as onp
from oracle import plr_np


def _recs(n, seed=0):
    p = onp.Params()
    return onp.pack_levels([onp.sample_level(seed, (0, i), p) for i in range(n)], p)


def test_rank_probabilities_spec_example():
    """scores [3,1,2], beta=1, rho=0 -> [6/11, 2/11, 3/11]."""
    buf = plr_np.LevelBuffer(3)
    buf.update(_recs(3), np.array([3.0, 1.0, 2.0]), np.zeros(3), it=0)
    cfg = plr_np.PlrConfig(temperature=1.0, staleness_coef=0.0)
    assert np.allclose(buf.probabilities(cfg, it=1), [6 / 11, 2 / 11, 3 / 11], rtol=0, atol=1e-15)


def test_staleness_only():
    """rho=1 -> proportional to staleness."""
    buf = plr_np.LevelBuffer(3)
    lv = _recs(3)
    buf.update(lv[:1], np.array([1.0]), np.zeros(1), it=0)
    buf.update(lv[1:2], np.array([2.0]), np.zeros(1), it=2)
    buf.update(lv[2:], np.array([3.0]), np.zeros(1), it=3)
    cfg = plr_np.PlrConfig(temperature=1.0, staleness_coef=1.0)
    assert np.allclose(buf.probabilities(cfg, it=4), np.array([4, 2, 1]) / 7)


def test_buffer_update_spec_example():
    """K=2, inserting [5,1,3] -> {5,3}; below-min unchanged; re-insert keeps size."""
    buf = plr_np.LevelBuffer(2)
    lv = _recs(4)
    buf.update(lv[:3], np.array([5.0, 1.0, 3.0]), np.zeros(3), it=0)
    assert sorted(buf.score[: buf.size].tolist()) == [3.0, 5.0]
    before = buf.snapshot()
    buf.update(lv[3:], np.array([2.0]), np.zeros(1), it=1)
    assert all(np.array_equal(a, b) for a, b in zip(before, buf.snapshot()))
    buf.update(lv[:1], np.array([7.0]), np.array([0.5]), it=2)  # identical level: in place
    assert buf.size == 2 and 7.0 in buf.score[:2].tolist()


def test_stale_first_eviction():
    """equal min scores -> the smaller last_sampled goes."""
    buf = plr_np.LevelBuffer(2)
    lv = _recs(3)
    buf.update(lv[:1], np.array([1.0]), np.zeros(1), it=5)
    buf.update(lv[1:2], np.array([1.0]), np.zeros(1), it=3)
    buf.update(lv[2:], np.array([2.0]), np.zeros(1), it=6)
    keys = {plr_np.LevelBuffer.key(r) for r in buf.levels[: buf.size]}
    assert plr_np.LevelBuffer.key(lv[0]) in keys and plr_np.LevelBuffer.key(lv[1]) not in keys


def test_choice_recipe_equals_numpy_choice():
    """Generator.choice(n, k, p) == searchsorted(cumsum(p)/cumsum(p)[-1], random(k), 'right')
    with a sequential cumsum: the recipe the CUDA sampler implements."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = int(rng.integers(1, 4001))
        p = rng.uniform(0, 1, n) ** 3
        p /= p.sum()
        a = onp.generator(9, (trial,)).choice(n, 500, p=p)
        cdf = np.cumsum(p)
        cdf /= cdf[-1]
        b = cdf.searchsorted(onp.generator(9, (trial,)).random(500), side="right")
        assert np.array_equal(a, b)


def test_empirical_distribution():
    """5 entries, beta=0.3, rho=0.3, 1e5 draws within 0.01 of closed form."""
    buf = plr_np.LevelBuffer(5)
    buf.update(_recs(5), np.array([0.5, 0.1, 0.9, 0.3, 0.7]), np.zeros(5), it=0)
    buf.last_sampled[:] = [0, 1, 2, 3, 4]
    cfg = plr_np.PlrConfig(temperature=0.3, staleness_coef=0.3)
    p = buf.probabilities(cfg, it=5)
    ranks = np.array([3, 5, 1, 4, 2])
    ps = (1.0 / ranks) ** (1 / 0.3)
    ps /= ps.sum()
    pc = np.array([5, 4, 3, 2, 1]) / 15
    assert np.allclose(p, 0.7 * ps + 0.3 * pc)
    draws = onp.generator(1, (2,)).choice(5, 100_000, p=p)
    emp = np.bincount(draws, minlength=5) / 1e5
    assert np.abs(emp - p).max() < 0.01


def test_capacity_and_min_invariants():
    rng = np.random.default_rng(0)
    buf = plr_np.LevelBuffer(50)
    lv = _recs(400, seed=4)
    for it in range(8):
        idx = rng.integers(0, 400, 100)
        sc = rng.choice([0.0, 0.0, 0.1, 0.2, 0.5], 100)
        full = buf.size == buf.K
        mn = buf.score[: buf.size].min() if buf.size else None
        buf.update(lv[idx], sc, np.zeros(100), it)
        assert buf.size <= buf.K
        keys = [plr_np.LevelBuffer.key(r) for r in buf.levels[: buf.size]]
        assert len(set(keys)) == len(keys)
        del full, mn
