"""The policy side of the rollout loop on the GPU.

* ``sample_actions`` / ``policy_head`` -- agents/rollout.py:145-152 and the tail of
  ``PPOAgent.act`` (agents/ppo.py:82-96, log_softmax_np at :136-138) as ONE kernel:
  logits -> sampled (or greedy) action + its log-probability, numpy-exact draws.
* ``rollout`` -- agents/rollout.py:87-142 with torch CUDA tensors end to end: the actor
  runs on the GPU, the action hand-off is the fused kernel above, and the step kernel
  writes observations, rewards and dones straight into the trajectory store (no
  per-step host round trip).  ``GraphRollout`` replays the whole step as one CUDA graph.

The actor protocol mirrors the reference's: ``initial_hidden(n)`` and
``act(obs, hidden, g=None, greedy=False) -> (actions int64 [B], log_probs f64 [B],
values f64 [B], hidden)``, where ``obs`` holds CUDA tensors (view uint8 [B,V,V], dir
int64 [B]) and ``g`` names the step's random stream (``rng.fold_in(t)``), to be handed to
``policy_head``/``sample_actions``.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .errors import ContractViolation, ShapeError
from .rng import as_stream
from .rollout import RolloutCursor, TrajectoryBatch


def _torch():
    import torch

    return torch


def policy_head(logits, g=None, greedy: bool = False, lane0: int = 0, actions=None, log_probs=None, actions_u8=None,
                step_dev=None):
    """logits [B, A] (float32/float64 CUDA) -> (actions int64 [B], log_probs float64 [B]).

    ``g``: the step's stream (RngStream or the reference's; e.g. ``rng.fold_in(t)``);
    lane i draws the (lane0 + i)-th double of its generator, as ``g.random(B)[i]``.
    ``step_dev`` (uint32 CUDA scalar) switches to graph-replay keys: ``g`` is then the
    rollout stream and the device folds in the step it reads from ``step_dev``."""
    torch = _torch()
    if logits.dim() != 2:
        raise ShapeError(f"logits must be [B, A], got {tuple(logits.shape)}")
    if logits.dtype not in (torch.float32, torch.float64):
        logits = logits.double()
    lg = logits.contiguous()
    B, A = lg.shape
    dev = lg.device
    if actions is None:
        actions = torch.empty(B, dtype=torch.int64, device=dev)
    if log_probs is None:
        log_probs = torch.empty(B, dtype=torch.float64, device=dev)
    if not greedy and g is None:
        raise ContractViolation("sampling needs a generator stream g")
    key = as_stream(g).seed_prefix() if g is not None else None
    _lib.call("amz_policy_head", _lib.ptr(lg), 0 if lg.dtype == torch.float32 else 1, B, A,
              ctypes.byref(key) if key is not None else None, _lib.ptr(step_dev) if step_dev is not None else None,
              int(bool(greedy)), int(lane0), _lib.ptr(actions), _lib.ptr(actions_u8) if actions_u8 is not None else None,
              _lib.ptr(log_probs), _lib.stream_handle(dev))
    return actions, log_probs


def sample_actions(logits, g):
    """agents/rollout.py:145 drop-in: inverse-CDF categorical draw, one uniform per lane."""
    return policy_head(logits, g)[0]


class TorchPolicyActor:
    """PPOAgent.act (agents/ppo.py:82-96) over a torch policy module on the GPU:
    ``model(prepare(obs), hidden) -> (logits, value, hidden)`` (MazePolicy's forward),
    ``prepare`` = MazePolicy.prepare on tensors (agents/models.py:117-121)."""

    def __init__(self, model):
        self.model = model

    def initial_hidden(self, n: int):
        return self.model.initial_hidden(n)

    @staticmethod
    def prepare(obs: dict) -> dict:
        return {"view": obs["view"].long(), "dir": obs["dir"].long()}

    def act(self, obs: dict, hidden, g=None, greedy: bool = False):
        torch = _torch()
        with torch.no_grad():
            logits, value, h = self.model(self.prepare(obs), hidden)
        actions, log_probs = policy_head(logits, g, greedy)
        return actions, log_probs, value.double(), h


def _flat(obs: dict) -> dict:
    return {k: v.reshape(-1, *v.shape[2:]) for k, v in obs.items()}


def rollout(rng, actor, env, start, length: int, params, hidden=None, greedy: bool = False):
    """agents/rollout.py:87-142 on the GPU.  Returns (TrajectoryBatch, RolloutCursor) with
    time-major CUDA tensors: obs view u8 [T,B,V,V] / dir i64 [T,B], actions i64, log_probs,
    values, rewards f64, dones bool, pre_hidden [T, *hidden.shape]."""
    torch = _torch()
    if length < 1:
        raise ContractViolation(f"rollout length must be >= 1, got {length}")
    if isinstance(start, RolloutCursor):
        obs, state, extras = dict(start.obs), start.state, start.extras
        hidden = start.hidden if hidden is None else hidden
    else:
        obs = _flat(start.observation)
        state, extras = start.state, start.extras
    B = obs["view"].shape[0]
    if hidden is None:
        hidden = actor.initial_hidden(B)
    dev = obs["view"].device
    shape = env.shape
    v = obs["view"].shape[-1]
    view = torch.empty((length + 1, B, v, v), dtype=torch.uint8, device=dev)
    dirs = torch.empty((length + 1, B), dtype=torch.int64, device=dev)
    view[0].copy_(obs["view"])
    dirs[0].copy_(obs["dir"])
    actions = torch.empty((length, B), dtype=torch.int64, device=dev)
    log_probs = torch.empty((length, B), dtype=torch.float64, device=dev)
    values = torch.empty((length, B), dtype=torch.float64, device=dev)
    rewards = torch.empty((length, B), dtype=torch.float64, device=dev)
    dones = torch.empty((length, B), dtype=torch.bool, device=dev)
    pre_hidden = torch.empty((length, *hidden.shape), dtype=hidden.dtype, device=dev)
    rng = as_stream(rng)
    for t in range(length):
        pre_hidden[t].copy_(hidden)
        g = None if greedy else rng.fold_in(t)
        act, logp, val, hidden = actor.act({"view": view[t], "dir": dirs[t]}, hidden, g=g, greedy=greedy)
        res = env.step(None, state, act.reshape(shape.n_agents, shape.flat_size), params, extras,
                       out={"view": view[t + 1], "dir": dirs[t + 1], "reward": rewards[t], "done": dones[t]})
        actions[t].copy_(act)
        log_probs[t].copy_(logp)
        values[t].copy_(val)
        hidden = hidden * (~dones[t]).to(hidden.dtype).unsqueeze(-1)
        state, extras = res.state, res.extras
    traj = TrajectoryBatch({"view": view[:length], "dir": dirs[:length]}, actions, rewards, dones, values, log_probs,
                           pre_hidden)
    return traj, RolloutCursor({"view": view[length], "dir": dirs[length]}, state, extras, hidden)


__all__ = ["policy_head", "sample_actions", "TorchPolicyActor", "rollout"]
