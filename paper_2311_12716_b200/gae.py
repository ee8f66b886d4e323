"""GAE, per-lane episode statistics and regret scores on the GPU.

Drop-ins for ``agents/gae.py:8-37`` (``compute_gae``), ``agents/rollout.py:155-189``
(``per_lane_episode_stats``) and ``runners/scoring.py:18-63`` (``score_pvl``,
``score_maxmc``, ``lane_scores``).  One fused kernel (csrc/amz_score.cu) reproduces the
reference's float64 arithmetic bit for bit, including numpy's pairwise summation inside
``.mean()``.  Inputs may be torch CUDA tensors (zero-copy) or numpy arrays (uploaded);
outputs are torch CUDA tensors.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .errors import ContractViolation, ShapeError


def _torch():
    import torch

    return torch


def _dev(x, dtype, device):
    torch = _torch()
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(x)
    return t.to(device=device, dtype=dtype).contiguous()


def _device_of(*xs):
    torch = _torch()
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return torch.device("cuda", torch.cuda.current_device())


def _stats_struct(B, device):
    torch = _torch()
    st = {"episodes": torch.empty(B, dtype=torch.int64, device=device),
          "mean_return": torch.empty(B, dtype=torch.float64, device=device),
          "max_return": torch.empty(B, dtype=torch.float64, device=device),
          "solved_rate": torch.empty(B, dtype=torch.float64, device=device)}
    c = _lib.AmzEpisodeStats(st["episodes"].data_ptr(), st["mean_return"].data_ptr(),
                             st["max_return"].data_ptr(), st["solved_rate"].data_ptr())
    return st, c


def gae_and_scores(rewards, values, dones, last_value, gamma: float, lam: float, prior_max_returns=None,
                   score_fn: str = "maxmc", maxmc_discounted: bool = False, with_stats: bool = False,
                   out: dict | None = None):
    """One launch: advantages, returns, per-lane scores, running max returns (+ stats).

    Equals ``compute_gae`` followed by ``lane_scores(traj, adv, prior, cfg, gamma)``.
    ``values`` and ``last_value`` may both be float32 tensors -- the policy's own output
    dtype, which the reference widens with ``value.double()`` (agents/ppo.py:96) -- and are
    then widened inside the kernel (bit-identical results, half the value bytes).
    ``out`` may supply the result tensors (keys advantages, returns [T, B] and scores,
    max_returns [B], float64, contiguous, on the device) to keep a loop allocation-free."""
    torch = _torch()
    dev = _device_of(rewards, values, dones, last_value)
    r = _dev(rewards, torch.float64, dev)
    v32 = (torch.is_tensor(values) and values.dtype == torch.float32 and torch.is_tensor(last_value)
           and last_value.dtype == torch.float32)
    v = _dev(values, torch.float32 if v32 else torch.float64, dev)
    if r.dim() != 2 or v.shape != r.shape:
        raise ShapeError(f"rewards {tuple(r.shape)} / values {tuple(v.shape)} must be equal [T, B]")
    T, B = r.shape
    d = _dev(dones, torch.bool, dev).view(torch.uint8)
    last = _dev(last_value, torch.float32 if v32 else torch.float64, dev).reshape(-1)
    if d.shape != r.shape or last.numel() != B:
        raise ShapeError("dones must be [T, B] and last_value [B]")
    prior = None if prior_max_returns is None else _dev(prior_max_returns, torch.float64, dev).reshape(-1)
    o = out or {}

    def _out(k, shape):
        t = o.get(k)
        if t is None:
            return torch.empty(shape, dtype=torch.float64, device=dev)
        if tuple(t.shape) != shape or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ShapeError(f"out[{k!r}] must be a contiguous float64 {shape} tensor on {dev}")
        return t

    adv = _out("advantages", (T, B))
    ret = _out("returns", (T, B))
    scores = _out("scores", (B,))
    maxret = _out("max_returns", (B,))
    stats, cst = _stats_struct(B, dev) if with_stats else (None, None)
    fn = {"maxmc": _lib.AMZ_SCORE_MAXMC, "pvl": _lib.AMZ_SCORE_PVL}[score_fn]
    with torch.cuda.device(dev):
        _lib.call("amz_gae_score_v32" if v32 else "amz_gae_score", T, B, _lib.ptr(r), _lib.ptr(v), _lib.ptr(d), _lib.ptr(last), float(gamma),
                  float(lam), _lib.ptr(prior), fn, int(bool(maxmc_discounted)), _lib.ptr(adv), _lib.ptr(ret),
                  _lib.ptr(scores), _lib.ptr(maxret), ctypes.byref(cst) if cst is not None else None,
                  _lib.stream_handle(dev))
    out = {"advantages": adv, "returns": ret, "scores": scores, "max_returns": maxret}
    if with_stats:
        out["stats"] = stats
    return out


def compute_gae(rewards, values, dones, last_value, gamma: float, lam: float):
    """agents/gae.py:8-37 -> (advantages, returns), float64 [T, B]."""
    o = gae_and_scores(rewards, values, dones, last_value, gamma, lam)
    return o["advantages"], o["returns"]


def per_lane_episode_stats(rewards, dones, gamma: float = 1.0) -> dict:
    """agents/rollout.py:155-189 (incl. its never-reset discount)."""
    torch = _torch()
    dev = _device_of(rewards, dones)
    r = _dev(rewards, torch.float64, dev)
    T, B = r.shape
    d = _dev(dones, torch.bool, dev).view(torch.uint8)
    v = torch.zeros_like(r)
    scores = torch.empty(B, dtype=torch.float64, device=dev)
    maxret = torch.empty(B, dtype=torch.float64, device=dev)
    stats, cst = _stats_struct(B, dev)
    with torch.cuda.device(dev):
        _lib.call("amz_lane_scores", T, B, _lib.ptr(r), _lib.ptr(v), _lib.ptr(d), None, float(gamma), None,
                  _lib.AMZ_SCORE_MAXMC, 1, _lib.ptr(scores), _lib.ptr(maxret), ctypes.byref(cst),
                  _lib.stream_handle(dev))
    return stats
