"""Regret scores for level curation (runners/scoring.py:18-63) on the GPU.

All three functions run the fused score kernel (csrc/amz_score.cu) without its GAE
pass; the means use numpy's pairwise summation order, so results are bit-identical
to the reference.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .errors import ContractViolation
from .gae import _dev, _device_of, _stats_struct

NOCLAMP, PRIOR_FINAL = 0x100, 0x200


def _torch():
    import torch

    return torch


def _run(rewards, values, dones, adv, prior, fn: int, gamma: float, disc: bool, with_stats=False):
    torch = _torch()
    dev = values.device
    T, B = values.shape
    scores = torch.empty(B, dtype=torch.float64, device=dev)
    maxret = torch.empty(B, dtype=torch.float64, device=dev)
    stats, cst = _stats_struct(B, dev) if with_stats else (None, None)
    with torch.cuda.device(dev):
        _lib.call("amz_lane_scores", T, B, _lib.ptr(rewards), _lib.ptr(values), _lib.ptr(dones.view(torch.uint8)),
                  _lib.ptr(adv), float(gamma), _lib.ptr(prior), fn, int(bool(disc)), _lib.ptr(scores),
                  _lib.ptr(maxret), ctypes.byref(cst) if cst is not None else None, _lib.stream_handle(dev))
    return (scores, maxret, stats) if with_stats else (scores, maxret)


def _column(x):
    torch = _torch()
    t = _dev(x, torch.float64, _device_of(x)).reshape(-1, 1)
    if t.numel() == 0:
        raise ContractViolation("cannot score an empty trajectory slice")
    return t


def score_pvl(advantages) -> float:
    """Mean positive advantage over one slice (runners/scoring.py:18-23)."""
    torch = _torch()
    a = _column(advantages)
    z = torch.zeros_like(a)
    s, _ = _run(z, z, torch.zeros_like(a, dtype=torch.bool), a, None, _lib.AMZ_SCORE_PVL | NOCLAMP, 1.0, False)
    return float(s[0])


def score_maxmc(values, max_return: float) -> float:
    """Mean (max_return - V) over one slice (runners/scoring.py:26-31); not clamped."""
    torch = _torch()
    v = _column(values)
    prior = torch.full((1,), float(max_return), dtype=torch.float64, device=v.device)
    s, _ = _run(torch.zeros_like(v), v, torch.zeros_like(v, dtype=torch.bool), None, prior,
                _lib.AMZ_SCORE_MAXMC | NOCLAMP | PRIOR_FINAL, 1.0, False)
    return float(s[0])


def lane_scores(traj, advantages, prior_max_returns, cfg, gamma: float = 1.0, episode_stats=None):
    """runners/scoring.py:34-63 -> (scores clamped at 0 [B], running max returns [B]).

    ``traj`` needs ``rewards``, ``values``, ``dones`` ([T, B], time-major); ``cfg``
    needs ``score_fn`` ("maxmc" | "pvl") and ``maxmc_discounted``."""
    torch = _torch()
    dev = _device_of(traj.values, traj.rewards, advantages)
    r = _dev(traj.rewards, torch.float64, dev)
    v = _dev(traj.values, torch.float64, dev)
    d = _dev(traj.dones, torch.bool, dev)
    a = _dev(advantages, torch.float64, dev)
    prior = _dev(prior_max_returns, torch.float64, dev).reshape(-1)
    fn = _lib.AMZ_SCORE_PVL if cfg.score_fn == "pvl" else _lib.AMZ_SCORE_MAXMC
    if episode_stats is not None:
        smax = _dev(episode_stats["max_return"], torch.float64, dev).reshape(-1)
        # np.maximum(prior, max_return) with NaN propagation, then skip the episode pass
        prior = torch.where(torch.isnan(prior) | (prior >= smax), prior, smax)
        fn |= PRIOR_FINAL
    return _run(r, v, d, a, prior, fn, gamma, bool(getattr(cfg, "maxmc_discounted", False)))
