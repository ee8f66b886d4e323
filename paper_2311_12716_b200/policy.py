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


class DeviceStepKey:
    """``rng.fold_in(t)`` with ``rng``'s SeedSequence prefix and ``t`` in device memory
    (CUDA-graph replay: the captured kernels read both at run time)."""

    def __init__(self, prefix, step):
        self.prefix = prefix  # uint8 CUDA tensor holding an amz_seed_t
        self.step = step      # int32 CUDA scalar tensor (u32 t)


def policy_head(logits, g=None, greedy: bool = False, lane0: int = 0, actions=None, log_probs=None, actions_u8=None):
    """logits [B, A] (float32/float64 CUDA) -> (actions int64 [B], log_probs float64 [B]).

    ``g``: the step's stream (RngStream or the reference's; e.g. ``rng.fold_in(t)``);
    lane i draws the (lane0 + i)-th double of its generator, as ``g.random(B)[i]``.
    ``g`` may be a ``DeviceStepKey`` (graph replay: key prefix and step read on device)."""
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
    a8 = _lib.ptr(actions_u8) if actions_u8 is not None else None
    dt = 0 if lg.dtype == torch.float32 else 1
    if isinstance(g, DeviceStepKey):
        _lib.call("amz_policy_head_dev", _lib.ptr(lg), dt, B, A, _lib.ptr(g.prefix), _lib.ptr(g.step),
                  int(bool(greedy)), int(lane0), _lib.ptr(actions), a8, _lib.ptr(log_probs), _lib.stream_handle(dev))
        return actions, log_probs
    key = as_stream(g).seed_prefix() if g is not None else None
    _lib.call("amz_policy_head", _lib.ptr(lg), dt, B, A, ctypes.byref(key) if key is not None else None,
              int(bool(greedy)), int(lane0), _lib.ptr(actions), a8, _lib.ptr(log_probs), _lib.stream_handle(dev))
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
    traj = TrajectoryBatch({"view": view[:length], "dir": dirs[:length]}, actions, log_probs, values, rewards, dones,
                           pre_hidden)
    return traj, RolloutCursor({"view": view[length], "dir": dirs[length]}, state, extras, hidden)


def _seed_bytes(stream, device):
    torch = _torch()
    raw = bytes(as_stream(stream).seed_prefix())
    return torch.tensor(list(raw), dtype=torch.uint8, device=device)


class GraphRollout:
    """``rollout`` with every step one replay of a captured CUDA graph (SURVEY §8f row
    1: "CUDA-Graph the rollout() loop").  One step = trajectory slot writes at the device
    step index, ``actor.act`` (torch, must be capturable: device work only, static
    shapes), the fused policy head, the device-counter env step, the carry reset.  Keys
    (the rollout stream's and the auto-reset wrapper's SeedSequence prefixes) and the
    step counters live in device memory, so the graph captured on the first call serves
    every later call on the same env (same lanes, same actor).  Results equal
    ``rollout``'s; the trajectory tensors are cloned unless ``copy=False`` (then they are
    the graph's buffers, overwritten by the next call)."""

    def __init__(self, actor, env, length: int, greedy: bool = False):
        if length < 1:
            raise ContractViolation(f"rollout length must be >= 1, got {length}")
        self.actor, self.env, self.T, self.greedy = actor, env, length, greedy
        self.graph = None
        self.buf = None

    def _alloc(self, obs, hidden, state):
        torch = _torch()
        B, v = obs["view"].shape[0], obs["view"].shape[-1]
        dev = obs["view"].device
        T = self.T
        self.buf = {
            "view": torch.empty((T, B, v, v), dtype=torch.uint8, device=dev),
            "dir": torch.empty((T, B), dtype=torch.int64, device=dev),
            "actions": torch.empty((T, B), dtype=torch.int64, device=dev),
            "log_probs": torch.empty((T, B), dtype=torch.float64, device=dev),
            "values": torch.empty((T, B), dtype=torch.float64, device=dev),
            "rewards": torch.empty((T, B), dtype=torch.float64, device=dev),
            "dones": torch.empty((T, B), dtype=torch.bool, device=dev),
            "pre_hidden": torch.empty((T, *hidden.shape), dtype=hidden.dtype, device=dev),
            "cur_view": torch.empty((B, v, v), dtype=torch.uint8, device=dev),
            "cur_dir": torch.empty((B,), dtype=torch.int64, device=dev),
            "cur_hidden": torch.empty_like(hidden),
            "cur_rew": torch.empty((B,), dtype=torch.float64, device=dev),
            "cur_done": torch.empty((B,), dtype=torch.bool, device=dev),
            "t32": torch.zeros(1, dtype=torch.int32, device=dev),
            "s32": torch.zeros(1, dtype=torch.int32, device=dev),
            "t64": torch.zeros(1, dtype=torch.int64, device=dev),
            "key": torch.zeros(24, dtype=torch.uint8, device=dev),
            "wrap": torch.zeros(24, dtype=torch.uint8, device=dev),
        }
        self.state = state

    def _body(self):
        from .batch import RESAMPLE

        b = self.buf
        t = b["t64"]
        b["view"].index_copy_(0, t, b["cur_view"].unsqueeze(0))
        b["dir"].index_copy_(0, t, b["cur_dir"].unsqueeze(0))
        b["pre_hidden"].index_copy_(0, t, b["cur_hidden"].unsqueeze(0))
        g = None if self.greedy else DeviceStepKey(b["key"], b["t32"])
        act, logp, val, h = self.actor.act({"view": b["cur_view"], "dir": b["cur_dir"]}, b["cur_hidden"], g=g,
                                           greedy=self.greedy)
        a = act.reshape(-1).to(_torch().int64).contiguous()
        mode = _lib.AMZ_RESET_RESAMPLE if self.env.mode == RESAMPLE else _lib.AMZ_RESET_HOME
        _lib.call("amz_env_step_dev", self.state.handle, _lib.ptr(a), 2, mode, _lib.ptr(b["wrap"]), _lib.ptr(b["s32"]),
                  _lib.ptr(b["cur_view"]), _lib.ptr(b["cur_dir"]), _lib.ptr(b["cur_rew"]), _lib.ptr(b["cur_done"]),
                  None, None, self.state.stream())
        b["actions"].index_copy_(0, t, a.unsqueeze(0))
        b["log_probs"].index_copy_(0, t, logp.reshape(1, -1).double())
        b["values"].index_copy_(0, t, val.reshape(1, -1).double())
        b["rewards"].index_copy_(0, t, b["cur_rew"].unsqueeze(0))
        b["dones"].index_copy_(0, t, b["cur_done"].unsqueeze(0))
        b["cur_hidden"].copy_(h * (~b["cur_done"]).to(h.dtype).unsqueeze(-1))
        b["t32"].add_(1)
        b["s32"].add_(1)
        b["t64"].add_(1)

    def __call__(self, rng, start, hidden=None, copy: bool = True):
        torch = _torch()
        from .batch import AutoResetWrapper

        if isinstance(start, RolloutCursor):
            obs, state, extras = dict(start.obs), start.state, start.extras
            hidden = start.hidden if hidden is None else hidden
        else:
            obs = _flat(start.observation)
            state, extras = start.state, start.extras
        if hidden is None:
            hidden = self.actor.initial_hidden(obs["view"].shape[0])
        wrap = extras[AutoResetWrapper.EXTRAS_KEY]
        if self.buf is None:
            self._alloc(obs, hidden, state)
        elif state is not self.state:
            raise ContractViolation("a GraphRollout is bound to the env state it was captured on")
        b = self.buf
        b["cur_view"].copy_(obs["view"])
        b["cur_dir"].copy_(obs["dir"].to(torch.int64))
        b["cur_hidden"].copy_(hidden)
        b["t32"].zero_()
        b["t64"].zero_()
        b["s32"].fill_(int(wrap["step"]))
        b["key"].copy_(_seed_bytes(rng, b["key"].device))
        if wrap.get("rng") is not None:
            b["wrap"].copy_(_seed_bytes(wrap["rng"], b["wrap"].device))
        steps = self.T
        if self.graph is None:
            self._body()  # step 0 runs eagerly (also warms up the actor's kernels)
            steps -= 1
            if steps > 0:
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph):
                    self._body()
        for _ in range(steps):
            self.graph.replay()
        c = (lambda x: x.clone()) if copy else (lambda x: x)
        traj = TrajectoryBatch({"view": c(b["view"]), "dir": c(b["dir"])}, c(b["actions"]), c(b["log_probs"]),
                               c(b["values"]), c(b["rewards"]), c(b["dones"]), c(b["pre_hidden"]))
        ext = dict(extras)
        ext[AutoResetWrapper.EXTRAS_KEY] = {**wrap, "step": wrap["step"] + self.T}
        cur = RolloutCursor({"view": b["cur_view"].clone(), "dir": b["cur_dir"].clone()}, state, ext,
                            b["cur_hidden"].clone())
        return traj, cur


__all__ = ["policy_head", "sample_actions", "TorchPolicyActor", "rollout", "GraphRollout", "DeviceStepKey"]
