"""Fused multi-step rollouts with a given action stream (the env side of
``agents/rollout.py:120-179``).

``rollout_actions`` advances every lane of an auto-resetting env ``T`` steps inside
one kernel launch (lane state in registers, level boards in shared memory) and
stores the trajectory time-major exactly as ``rollout()`` does: ``obs[t]`` is the
observation *before* step t, ``rewards``/``dones`` describe step t, and the cursor
holds the observation after the last step.  With ``actions[t]`` from a policy this is
the reference's rollout loop minus the per-step Python round trips; with random
actions it is SPEC's ``bench-sps`` workload.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .batch import HOME, RESAMPLE, AutoResetWrapper, DeviceLanes
from .errors import ContractViolation, ShapeError
from .rng import as_stream


def _torch():
    import torch

    return torch


@dataclass
class TrajectoryBatch:
    """Time-major rollout storage on the GPU ([T, B, ...] over flat lanes), field for
    field the reference's ``agents/rollout.py:19-70`` (same positional order, so code
    that builds one positionally keeps working).  The fused action-stream rollout has no
    policy outputs: its ``log_probs``/``values``/``pre_hidden`` are None."""

    obs: dict          # view uint8 [T, B, V, V], dir uint8 [T, B] (int64 from the policy rollout)
    actions: object    # uint8 [T, B] (int64 from the policy rollout)
    log_probs: object  # float64 [T, B] or None
    values: object     # float64 [T, B] or None
    rewards: object    # float64 [T, B]
    dones: object      # bool [T, B]
    pre_hidden: object = None  # [T, B, H]: carry fed to the policy at step t

    FIELDS = ("actions", "log_probs", "values", "rewards", "dones", "pre_hidden")

    @property
    def length(self) -> int:
        return self.actions.shape[0]

    @property
    def n_lanes(self) -> int:
        return self.actions.shape[1]

    def reset_masks(self):
        """True where the recurrent carry restarts before step t (agents/rollout.py:44-48)."""
        torch = _torch()
        masks = torch.zeros_like(self.dones)
        masks[1:] = self.dones[:-1]
        return masks

    def lane_slice(self, lanes) -> "TrajectoryBatch":
        """Lanes ``lanes`` (index array / tensor / slice) of every field (agents/rollout.py:50-60)."""
        torch = _torch()
        if not isinstance(lanes, slice):
            lanes = torch.as_tensor(lanes, device=self.actions.device)
            if lanes.dtype != torch.bool:
                lanes = lanes.to(torch.int64)

        def pick(v):
            return None if v is None else v[:, lanes]

        return TrajectoryBatch({k: v[:, lanes] for k, v in self.obs.items()},
                               *(pick(getattr(self, f)) for f in self.FIELDS))

    @staticmethod
    def concat_lanes(parts: list) -> "TrajectoryBatch":
        """Concatenate along the lane axis (agents/rollout.py:62-70); a field that is None
        in every part stays None."""
        torch = _torch()
        keys = parts[0].obs.keys()

        def cat(f):
            vs = [getattr(p, f) for p in parts]
            if all(v is None for v in vs):
                return None
            if any(v is None for v in vs):
                raise ShapeError(f"field {f!r} is missing in some of the concatenated trajectories")
            return torch.cat(vs, dim=1)

        return TrajectoryBatch({k: torch.cat([p.obs[k] for p in parts], dim=1) for k in keys},
                               *(cat(f) for f in TrajectoryBatch.FIELDS))


@dataclass
class RolloutCursor:
    obs: dict
    state: object
    extras: dict
    hidden: object = None


def random_actions(rng, T: int, B: int, device=None):
    """Uniform actions in {0,1,2} drawn on the GPU with a counter-based generator
    (torch's Philox): throughput workloads only.  Parity tests upload the reference's
    numpy action stream instead."""
    torch = _torch()
    g = torch.Generator(device=device or "cuda")
    s = as_stream(rng)
    g.manual_seed(hash((s.entropy, s.key)) & 0x7FFFFFFFFFFFFFFF)
    return torch.randint(0, 3, (T, B), generator=g, device=device or "cuda", dtype=torch.uint8)


def rollout_actions(env: AutoResetWrapper, start, actions, params, out: dict | None = None):
    """T fused steps of every lane with ``actions`` uint8 [T, B] (time-major).

    ``start`` is the StepResult of reset/reset_to_levels or a previous RolloutCursor.
    ``out`` may pre-allocate the trajectory tensors (keys view, dir, rewards, dones,
    final_view, final_dir) to keep a benchmark loop allocation-free.
    Returns (TrajectoryBatch, RolloutCursor)."""
    torch = _torch()
    if not isinstance(env, AutoResetWrapper):
        raise ContractViolation("rollout needs an AutoResetWrapper env")
    state, extras = start.state, start.extras
    if not isinstance(state, DeviceLanes):
        raise ContractViolation("start state is not a device env state")
    wrap = extras[AutoResetWrapper.EXTRAS_KEY]
    T, B = actions.shape
    if B != state.n:
        raise ShapeError(f"actions have {B} lanes, env has {state.n}")
    if T < 1:
        raise ContractViolation(f"rollout length must be >= 1, got {T}")
    dev = state.device
    a = actions.to(dev).to(torch.uint8).contiguous()
    v = state.params.agent_view_size
    o = out or {}
    view = o.get("view") if o.get("view") is not None else torch.empty((T, B, v, v), dtype=torch.uint8, device=dev)
    dirs = o.get("dir") if o.get("dir") is not None else torch.empty((T, B), dtype=torch.uint8, device=dev)
    rew = o.get("rewards") if o.get("rewards") is not None else torch.empty((T, B), dtype=torch.float64, device=dev)
    done = o.get("dones") if o.get("dones") is not None else torch.empty((T, B), dtype=torch.bool, device=dev)
    fview = o.get("final_view") if o.get("final_view") is not None else torch.empty((B, v, v), dtype=torch.uint8,
                                                                                    device=dev)
    fdir = o.get("final_dir") if o.get("final_dir") is not None else torch.empty((B,), dtype=torch.uint8, device=dev)
    mode = _lib.AMZ_RESET_RESAMPLE if env.mode == RESAMPLE else _lib.AMZ_RESET_HOME
    seed = wrap["rng"].seed_prefix() if env.mode == RESAMPLE else None
    _lib.call("amz_env_rollout", state.handle, T, _lib.ptr(a), mode, ctypes.byref(seed) if seed else None,
              ctypes.c_uint32(int(wrap["step"])), _lib.ptr(view), _lib.ptr(dirs), _lib.ptr(rew), _lib.ptr(done),
              _lib.ptr(fview), _lib.ptr(fdir), state.stream())
    traj = TrajectoryBatch({"view": view, "dir": dirs}, a, None, None, rew, done)
    ext = dict(extras)
    ext[AutoResetWrapper.EXTRAS_KEY] = {**wrap, "step": wrap["step"] + T}
    return traj, RolloutCursor({"view": fview, "dir": fdir}, state, ext)


__all__ = ["TrajectoryBatch", "RolloutCursor", "rollout_actions", "random_actions", "HOME", "RESAMPLE"]
