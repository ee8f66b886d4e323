"""CPU-side checks of the C ABI: the library loads (no GPU needed) and exports every
function include/amaze_b200.h declares; host-side key setup matches numpy."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "amaze_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amz_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2311_12716_b200 import _lib

    L = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert sorted(_lib._SIGS) == names


def test_abi_version_and_param_validation():
    from paper_2311_12716_b200 import _lib
    from paper_2311_12716_b200.core import StaticParams
    from paper_2311_12716_b200.errors import ConfigError

    assert _lib.lib().amz_abi_version() == 1
    _lib.call("amz_validate_params", ctypes.byref(StaticParams().c_struct()))
    for bad in (StaticParams(height=2), StaticParams(agent_view_size=4), StaticParams(wall_budget=120),
                StaticParams(max_episode_steps=0), StaticParams(height=20, width=20)):
        with pytest.raises(ConfigError):
            _lib.call("amz_validate_params", ctypes.byref(bad.c_struct()))
        with pytest.raises(ConfigError):
            bad.validate()


def _absorb(pool, hc, w):
    M = 0xFFFFFFFF
    for d in range(4):
        v = (w ^ hc) & M
        hc = (hc * 0x931E8875) & M
        v = (v * hc) & M
        v ^= v >> 16
        r = (0xCA01F9DD * pool[d] - 0x4973F715 * v) & M
        pool[d] = r ^ (r >> 16)
    return pool, hc


def _key(pool):
    M = 0xFFFFFFFF
    h, out = 0x8B51F9DD, []
    for i in range(4):
        v = (pool[i] ^ h) & M
        h = (h * 0x58F38DED) & M
        v = (v * h) & M
        out.append(v ^ (v >> 16))
    return [out[0] | (out[1] << 32), out[2] | (out[3] << 32)]


@pytest.mark.parametrize("entropy,prefix,suffix", [(0, (), (5,)), (0, (1,), (7, 9)), (2**40 + 3, (0,), (11,)),
                                                   (2**140 + 1, (4, 5), (6,)), (12345, (2**35,), (1, 2))])
def test_seed_prefix_plus_device_suffix_equals_numpy(entropy, prefix, suffix):
    """The prefix state (C host code) + per-lane suffix absorption == SeedSequence key."""
    from paper_2311_12716_b200.rng import RngStream

    s = RngStream(entropy, prefix).seed_prefix()
    pool, hc = list(s.pool), s.hash_const
    for w in suffix:
        pool, hc = _absorb(pool, hc, w)
    want = np.random.SeedSequence(entropy=entropy, spawn_key=prefix + suffix).generate_state(2, np.uint64)
    assert _key(pool) == [int(x) for x in want]
