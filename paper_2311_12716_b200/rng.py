"""Splittable random streams keyed exactly like the reference's ``RngStream``
(``rng.py:20-71``): a stream is (entropy, key tuple); ``split``/``fold_in`` extend the
key; the numbers behind a key are numpy's SeedSequence(entropy, spawn_key=key) ->
Philox4x64-10 stream.

Here a stream never materialises a numpy Generator on the host: ``seed_prefix()``
hands the CUDA kernels the SeedSequence state after the key, and each lane appends
its own suffix words (lane index, or auto-reset step and lane) on the device
(paper_2311_12716_b200/csrc/amz_rng.cuh).
"""

from __future__ import annotations

import ctypes

from . import _lib


def _u32_words(x: int) -> list[int]:
    """numpy's _int_to_uint32_array: little-endian 32-bit words, 0 -> [0]."""
    x = int(x)
    if x < 0:
        raise ValueError("entropy and key words must be non-negative")
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return out


class RngStream:
    """Immutable key (entropy, key) naming one numpy-compatible random stream."""

    __slots__ = ("_entropy", "_key", "_prefix")

    def __init__(self, entropy, key: tuple = ()):
        self._entropy = entropy
        self._key = tuple(int(k) for k in key)
        self._prefix = None

    @classmethod
    def from_seed(cls, seed: int) -> "RngStream":
        return cls(int(seed))

    @property
    def entropy(self):
        return self._entropy

    @property
    def key(self) -> tuple:
        return self._key

    def split(self, n: int) -> list["RngStream"]:
        if n < 0:
            raise ValueError(f"cannot split into {n} streams")
        return [RngStream(self._entropy, self._key + (i,)) for i in range(n)]

    def fold_in(self, data: int) -> "RngStream":
        return RngStream(self._entropy, self._key + (int(data),))

    def seed_prefix(self) -> _lib.AmzSeed:
        """SeedSequence state after this stream's key; device lanes append suffix words.
        Streams are immutable values, so the prefix is computed once per stream (a reset
        and the rollout that follows it both absorb the same wrapper key)."""
        if self._prefix is not None:
            return self._prefix
        run = _u32_words(self._entropy)
        key = [w for k in self._key for w in _u32_words(k)]
        ra = (ctypes.c_uint32 * len(run))(*run)
        ka = (ctypes.c_uint32 * max(1, len(key)))(*key)
        out = _lib.AmzSeed()
        _lib.call("amz_seed_prefix", ctypes.cast(ra, ctypes.c_void_p), len(run),
                  ctypes.cast(ka, ctypes.c_void_p), len(key), ctypes.byref(out))
        self._prefix = out
        return out

    def __repr__(self) -> str:
        return f"RngStream(entropy={self._entropy}, key={self._key})"

    def __reduce__(self):
        return (RngStream, (self._entropy, self._key))  # the cached prefix is not part of the value

    def __eq__(self, other) -> bool:
        return isinstance(other, RngStream) and (self._entropy, self._key) == (other._entropy, other._key)

    def __hash__(self) -> int:
        return hash((self._entropy, self._key))

    def __getstate__(self):
        return {"entropy": self._entropy, "key": self._key}

    def __setstate__(self, state):
        self._entropy = state["entropy"]
        self._key = tuple(state["key"])


def as_stream(rng) -> RngStream:
    """Accept our RngStream or any object with the reference's (_entropy, _key) slots."""
    if isinstance(rng, RngStream):
        return rng
    if hasattr(rng, "_entropy") and hasattr(rng, "_key"):
        return RngStream(rng._entropy, rng._key)
    raise TypeError(f"not a random stream: {rng!r}")
