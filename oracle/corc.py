"""ctypes front-end for oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Same import restriction as the rest of ``oracle/``: tests, smoke() and the bench's
CPU legs only.  Build with ``make -C oracle``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .amaze_np import LEVEL_DTYPE

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = ctypes.CDLL(path)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.orc_sample_levels_batch.argtypes = [u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_mutate_levels_batch.argtypes = [u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p]
        L.orc_probe_stream.argtypes = [u32p, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                       ctypes.c_int, ctypes.c_void_p]
        L.orc_seedseq_key.argtypes = [u32p, ctypes.c_int, ctypes.c_void_p]
        _lib = L
    return _lib


def int_words(x: int) -> list:
    """numpy's _int_to_uint32_array: little-endian u32 words, 0 -> [0]."""
    if x < 0:
        raise ValueError("negative entropy")
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return out


def entropy_words(entropy: int, key: tuple) -> np.ndarray:
    """SeedSequence assembled entropy: run words (+ zero pad to 4 if a key) + key words."""
    run = int_words(int(entropy))
    spawn = [w for k in key for w in int_words(int(k))]
    if spawn and len(run) < 4:
        run = run + [0] * (4 - len(run))
    return np.array(run + spawn, dtype=np.uint32)


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def seedseq_key(entropy: int, key: tuple) -> np.ndarray:
    w = entropy_words(entropy, key)
    out = np.zeros(2, dtype=np.uint64)
    lib().orc_seedseq_key(_p(w), len(w), out.ctypes.data)
    return out


def probe(entropy: int, key: tuple, kind: str, count: int, arg: int = 0) -> np.ndarray:
    kinds = {"next64": 0, "next32": 1, "below": 2, "random": 3, "interval": 4}
    w = entropy_words(entropy, key)
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_probe_stream(_p(w), len(w), kinds[kind], arg, count, out.ctypes.data)
    return out.view(np.float64) if kind == "random" else out


def sample_levels(entropy: int, prefix: tuple, lane0: int, count: int, H=13, W=13, budget=60) -> np.ndarray:
    """Levels for keys prefix+(lane0+i,), as amz_level_t records."""
    w = entropy_words(entropy, tuple(prefix) + (0,))[:-1].copy()
    out = np.zeros(count, dtype=LEVEL_DTYPE)
    lib().orc_sample_levels_batch(_p(w), len(w), lane0, count, H, W, budget, out.ctypes.data)
    return out


def mutate_levels(entropy: int, prefix: tuple, lane0: int, parents: np.ndarray, n_edits: int,
                  H=13, W=13) -> np.ndarray:
    w = entropy_words(entropy, tuple(prefix) + (0,))[:-1].copy()
    parents = np.ascontiguousarray(parents, dtype=LEVEL_DTYPE)
    out = np.zeros(len(parents), dtype=LEVEL_DTYPE)
    lib().orc_mutate_levels_batch(_p(w), len(w), lane0, len(parents), H, W, n_edits,
                                  parents.ctypes.data, out.ctypes.data)
    return out
