"""PLR level buffer resident on the GPU.

The reference imports ``runners/buffer.py`` (``runners/scoring.py:14``) but never
shipped it; ``SPEC.md:332-377,427-433`` describe it.  This is that buffer on the
device: ``update`` = SPEC's ``buffer_update``, ``sample`` = ``buffer_sample_levels``
(rank prioritisation + staleness), ``decision`` = ``buffer_sample_decision``.  The open
choices SPEC leaves are pinned identically in the oracle (oracle/plr_np.py docstring)
and in DESIGN.md.  Both kernels are single-CTA (csrc/amz_plr.cu) and exact: the
sampler reproduces numpy ``Generator.choice`` bit for bit, the update reproduces the
sequential per-candidate rule.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, ContractViolation
from .rng import as_stream


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class PlrConfig:
    """SPEC.md:336-339 PlrConfig (+ the two fields runners/scoring.py reads)."""

    replay_rate: float = 0.5
    buffer_size: int = 4000
    score_fn: str = "maxmc"
    prioritization: str = "rank"
    temperature: float = 0.3
    staleness_coef: float = 0.3
    robust: bool = True
    maxmc_discounted: bool = False

    def validate(self) -> "PlrConfig":
        if not 0.0 <= self.replay_rate <= 1.0:
            raise ConfigError(f"replay_rate must be in [0, 1], got {self.replay_rate}")
        if not self.temperature > 0.0:
            raise ConfigError(f"temperature must be > 0, got {self.temperature}")
        if not 0.0 <= self.staleness_coef <= 1.0:
            raise ConfigError(f"staleness_coef must be in [0, 1], got {self.staleness_coef}")
        if self.score_fn not in ("maxmc", "pvl"):
            raise ConfigError(f"unknown score_fn {self.score_fn!r}")
        if self.prioritization not in ("rank", "proportional"):
            raise ConfigError(f"unknown prioritization {self.prioritization!r}: 'rank' or 'proportional'")
        if not 1 <= self.buffer_size <= 4096:
            raise ConfigError(f"buffer_size must be in [1, 4096], got {self.buffer_size}")
        return self


@dataclass(frozen=True)
class AccelConfig:
    """SPEC.md:340-343."""

    n_mutations: int = 20
    subsample_size: int = 4


def rank_weights(K: int, beta: float) -> np.ndarray:
    """(1/rank)^(1/beta), ranks 1..K, computed by numpy (host LUT)."""
    ranks = np.arange(1, K + 1, dtype=np.float64)
    return np.power(1.0 / ranks, 1.0 / beta)


class LevelBuffer:
    """Device PLR buffer of capacity K (slots 0..size-1 valid)."""

    def __init__(self, cfg: PlrConfig, device=None):
        torch = _torch()
        self.cfg = cfg.validate()
        self.K = cfg.buffer_size
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            h = ctypes.c_void_p()
            _lib.call("amz_plr_create", self.K, ctypes.byref(h))
        self.handle = h
        self.lut = torch.from_numpy(rank_weights(self.K, cfg.temperature)).to(self.device)
        self.nonempty = False  # host-side knowledge: the first update always inserts

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h is not None and h.value and _lib._lib is not None:
                _lib._lib.amz_plr_destroy(h)
        except (AttributeError, TypeError):  # interpreter shutdown: module globals already cleared
            pass
        self.handle = None

    def _stream(self):
        return _lib.stream_handle(self.device)

    def update(self, levels, scores, max_returns, it: int) -> None:
        torch = _torch()
        n = levels.shape[0]
        lv = levels.to(self.device).to(torch.int32).contiguous()
        sc = scores.to(self.device).to(torch.float64).contiguous()
        mx = max_returns.to(self.device).to(torch.float64).contiguous()
        _lib.call("amz_plr_update", self.handle, _lib.ptr(lv), _lib.ptr(sc), _lib.ptr(mx), n, int(it), self._stream())
        if n > 0:
            self.nonempty = True

    def prepare(self, levels, stream=None) -> None:
        """Build the next update's candidate twin table now (``amz_plr_prepare``), on
        ``stream`` (a torch stream; default the current one) -- e.g. on a side stream
        while the candidates are rolled out.  The update with the same ``levels`` tensor
        skips that work; the caller orders the streams (update after this, this after the
        previous update)."""
        torch = _torch()
        # the update recognises the prepared batch by its device pointer: a converted
        # temporary could be freed and its address reused by another batch
        if (levels.dtype != torch.int32 or not levels.is_contiguous() or levels.device != torch.device(self.device)
                or levels.dim() != 2 or levels.shape[1] != 8):
            raise ContractViolation("prepare() needs the update's own levels tensor: contiguous int32 [n, 8] "
                                    f"on {self.device}, got {levels.dtype} {tuple(levels.shape)} on {levels.device}")
        st = stream.cuda_stream if stream is not None else self._stream()
        _lib.call("amz_plr_prepare", self.handle, _lib.ptr(levels), levels.shape[0], st)

    def sample(self, rng, n: int, it: int, out: dict | None = None):
        """n replay draws -> dict(slots i32, levels [n, 8], max_returns f64, scores f64);
        ``out`` may supply any of those tensors (contiguous, on the buffer's device) to be
        written in place."""
        torch = _torch()
        if not self.nonempty:
            raise ContractViolation("cannot sample from an empty level buffer")
        want = {"slots": ((n,), torch.int32), "levels": ((n, 8), torch.int32),
                "max_returns": ((n,), torch.float64), "scores": ((n,), torch.float64)}
        given = dict(out or {})
        for k, (shape, dt) in want.items():
            t = given.get(k)
            if t is not None and (tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous()
                                  or t.device != self.device):
                raise ContractViolation(f"out[{k!r}] must be a contiguous {dt} {list(shape)} tensor on {self.device}")
        out = {k: (given[k] if given.get(k) is not None else torch.empty(shape, dtype=dt, device=self.device))
               for k, (shape, dt) in want.items()}
        seed = as_stream(rng).seed_prefix()
        if self.cfg.prioritization == "proportional":  # P_S ~ score^(1/beta)
            _lib.call("amz_plr_sample_proportional", self.handle, ctypes.byref(seed), n,
                      float(self.cfg.staleness_coef), float(self.cfg.temperature), int(it), _lib.ptr(out["slots"]),
                      _lib.ptr(out["levels"]), _lib.ptr(out["max_returns"]), _lib.ptr(out["scores"]), self._stream())
        else:
            _lib.call("amz_plr_sample", self.handle, ctypes.byref(seed), n, float(self.cfg.staleness_coef),
                      _lib.ptr(self.lut), int(it), _lib.ptr(out["slots"]), _lib.ptr(out["levels"]),
                      _lib.ptr(out["max_returns"]), _lib.ptr(out["scores"]), self._stream())
        return out

    def decision(self, rng) -> bool:
        """buffer_sample_decision: replay w.p. p iff non-empty.  The
        single uniform is numpy's Generator(Philox(SeedSequence(key))).random(), computed
        by the library on the host (amz_stream_uniform; ~100 us faster than numpy)."""
        if not self.nonempty:
            return False
        u = ctypes.c_double(0.0)  # numpy's first Generator.random() of the stream, computed in C
        _lib.call("amz_stream_uniform", ctypes.byref(as_stream(rng).seed_prefix()), ctypes.byref(u))
        return bool(u.value < self.cfg.replay_rate)

    def size(self) -> int:
        v = ctypes.c_int64(0)
        _lib.call("amz_plr_size", self.handle, ctypes.byref(v), self._stream())
        return int(v.value)

    def digest(self, out=None):
        """Device int64 [1] digest of the buffer state (amz_plr_digest): the replica drift
        check's input, computed without a host round trip."""
        torch = _torch()
        out = torch.empty(1, dtype=torch.int64, device=self.device) if out is None else out
        _lib.call("amz_plr_digest", self.handle, _lib.ptr(out), self._stream())
        return out

    def export(self) -> dict:
        torch = _torch()
        K, dev = self.K, self.device
        st = {"levels": torch.empty((K, 8), dtype=torch.int32, device=dev),
              "score": torch.empty(K, dtype=torch.float64, device=dev),
              "max_return": torch.empty(K, dtype=torch.float64, device=dev),
              "last_sampled": torch.empty(K, dtype=torch.int64, device=dev),
              "seq": torch.empty(K, dtype=torch.int64, device=dev),
              "meta": torch.empty(2, dtype=torch.int64, device=dev)}
        _lib.call("amz_plr_export", self.handle, *(_lib.ptr(st[k]) for k in
                                                   ("levels", "score", "max_return", "last_sampled", "seq", "meta")),
                  self._stream())
        return st

    def load(self, st: dict) -> None:
        """Import a state exported by ``export`` (checkpoint resume).  The state is checked
        first: 0 <= size <= K, next_seq >= 0, and the valid slots' seq values distinct and
        below next_seq (the update relies on new entries sorting after every stored one)."""
        torch = _torch()
        dtypes = {"levels": torch.int32, "score": torch.float64, "max_return": torch.float64,
                  "last_sampled": torch.int64, "seq": torch.int64, "meta": torch.int64}
        t = {}
        for k, dt in dtypes.items():
            if k not in st:
                raise ContractViolation(f"buffer state is missing {k!r}")
            v = torch.as_tensor(st[k])
            want = (self.K, 8) if k == "levels" else (2,) if k == "meta" else (self.K,)
            if tuple(v.shape) != want:
                raise ContractViolation(f"buffer state {k!r} has shape {tuple(v.shape)}, expected {want}")
            t[k] = v.to(self.device).to(dt).contiguous()
        size, next_seq = (int(x) for x in t["meta"].cpu())
        if not 0 <= size <= self.K:
            raise ContractViolation(f"buffer state size {size} outside [0, {self.K}]")
        seq = t["seq"][:size].cpu()
        if next_seq < 0 or (size and (int(seq.min()) < 0 or int(seq.max()) >= next_seq
                                      or seq.unique().numel() != size)):
            raise ContractViolation("buffer state seq values must be distinct and in [0, next_seq)")
        _lib.call("amz_plr_import", self.handle, *(_lib.ptr(t[k]) for k in
                                                   ("levels", "score", "max_return", "last_sampled", "seq", "meta")),
                  self._stream())
        self.nonempty = bool(int(t["meta"][0].item()) > 0)
        del torch


def top_q(scores, q: int):
    """Indices of the q highest scores (ties -> lower index), on device."""
    torch = _torch()
    out = torch.empty(q, dtype=torch.int32, device=scores.device)
    s = scores.to(torch.float64).contiguous()
    _lib.call("amz_plr_top_q", _lib.ptr(s), s.numel(), int(q), _lib.ptr(out), _lib.stream_handle(scores.device))
    return out
