"""The C restatement of numpy's random streams (oracle/amaze_oracle.c) against numpy
itself and against the golden levels generated from the reference."""

import numpy as np
import pytest

from oracle import amaze_np as onp
from oracle import corc

KEYS = [(0, ()), (0, (0,)), (0, (1, 5, 7)), (123456789, (0, 3)), (2**40 + 17, (1, 2, 3)),
        (2**130 + 5, (9,)), (7, (2**33 + 1, 4))]


@pytest.mark.parametrize("entropy,key", KEYS)
def test_seedseq_key(entropy, key):
    ss = np.random.SeedSequence(entropy=entropy, spawn_key=key)
    assert np.array_equal(corc.seedseq_key(entropy, key), ss.generate_state(2, np.uint64))


@pytest.mark.parametrize("entropy,key", KEYS)
def test_raw_streams(entropy, key):
    g = onp.generator(entropy, key)
    assert np.array_equal(corc.probe(entropy, key, "next64", 37), g.bit_generator.random_raw(37))
    for n in (1, 2, 3, 4, 61, 120, 121, 1000003, 2**31 + 11):
        g = onp.generator(entropy, key)
        want = np.array([int(g.integers(0, n)) for _ in range(300)], dtype=np.uint64)
        assert np.array_equal(corc.probe(entropy, key, "below", 300, n), want), n
    g = onp.generator(entropy, key)
    assert np.array_equal(corc.probe(entropy, key, "random", 50), g.random(50))


def test_interleaved_u32_and_random_share_nothing():
    """random() does not consume the pending upper half of a 64-bit draw."""
    e, k = 5, (1, 2)
    g = onp.generator(e, k)
    a = [int(g.integers(0, 10)), float(g.random()), int(g.integers(0, 10)), int(g.integers(0, 10))]
    lv = corc.probe(e, k, "next64", 3)
    lo, hi = int(lv[0]) & 0xFFFFFFFF, int(lv[0]) >> 32
    assert a[0] == (lo * 10) >> 32
    assert a[1] == (int(lv[1]) >> 11) * (1.0 / 9007199254740992.0)
    assert a[2] == (hi * 10) >> 32


@pytest.mark.parametrize("n", [2, 3, 7, 49, 121])
def test_permutation_is_masked_fisher_yates(n):
    """Generator.permutation(n) == Fisher-Yates over masked-rejection draws on next32."""
    for key in [(0,), (3, 4), (11, 12, 13)]:
        want = onp.generator(1, key).permutation(n)
        words = iter(corc.probe(1, key, "next32", 4 * n + 64).tolist())
        arr = list(range(n))
        for i in range(n - 1, 0, -1):
            mask = (1 << i.bit_length()) - 1
            j = next(words) & mask
            while j > i:
                j = next(words) & mask
            arr[i], arr[j] = arr[j], arr[i]
        assert arr == want.tolist()


def _golden_levels(golden, name):
    z = golden("levels")
    return z[f"lv_{name}"], z[f"lv_{name}_meta"]


def _rows(rec):
    return np.stack([rec["walls"][:, 0], rec["walls"][:, 1], rec["walls"][:, 2], rec["walls"][:, 3],
                     rec["agent_r"], rec["agent_c"], rec["agent_dir"], rec["goal_r"], rec["goal_c"]],
                    axis=1).astype(np.int64)


@pytest.mark.parametrize("name", ["default", "seed12345", "budget0", "budget1", "budget119", "small9", "bigseed"])
def test_c_sampler_matches_reference(golden, name):
    want, meta = _golden_levels(golden, name)
    H, W, budget, seed, n = (int(x) for x in meta)
    got = corc.sample_levels(seed, (0,), 0, n, H, W, budget)
    assert np.array_equal(_rows(got), want)


@pytest.mark.parametrize("name", ["default", "budget0", "budget119", "small9"])
@pytest.mark.parametrize("edits", [1, 20])
def test_c_mutator_matches_reference(golden, name, edits):
    want_parent, meta = _golden_levels(golden, name)
    H, W, budget, seed, n = (int(x) for x in meta)
    parents = corc.sample_levels(seed, (0,), 0, n, H, W, budget)
    got = corc.mutate_levels(seed, (7,), 0, parents, edits, H, W)
    assert np.array_equal(_rows(got), golden("levels")[f"mut{edits}_{name}"])


@pytest.mark.parametrize("name", ["default", "budget119", "small9"])
def test_numpy_oracle_matches_reference(golden, name):
    want, meta = _golden_levels(golden, name)
    H, W, budget, seed, n = (int(x) for x in meta)
    p = onp.Params(height=H, width=W, wall_budget=budget)
    levels = [onp.sample_level(seed, (0, i), p) for i in range(min(n, 150))]
    assert np.array_equal(_rows(onp.pack_levels(levels, p)), want[: len(levels)])
    muts = [onp.mutate_level(seed, (7, i), lv, 20, p) for i, lv in enumerate(levels)]
    assert np.array_equal(_rows(onp.pack_levels(muts, p)), golden("levels")[f"mut20_{name}"][: len(levels)])
    # pack/unpack round trip
    back = onp.unpack_levels(onp.pack_levels(levels, p), p)
    for a, b in zip(levels, back):
        assert onp.level_key(a) == onp.level_key(b)
