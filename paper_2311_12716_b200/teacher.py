"""The PAIRED level designer on the GPU (amaze/teacher.py:36-159).

``TeacherEnv`` is the single-environment facade (``action_count``, ``episode_length``,
``step_uses_rng``); ``batch_lift(TeacherEnv(), shape)`` gives ``TeacherBatchEnv``, the
batched design process with the reference's GenericBatchEnv results (obs ``grid`` u8
[A, F, H, W], ``phase`` f32 [A, F, 4], ``n_placed`` i64 [A, F]; reward 0.0; done;
``info["time"]``), every lane advanced by one kernel launch.  Finished designs decode to
level records (``designed_levels``) that feed straight into the maze env's
``reset_to_levels`` -- the PAIRED hand-off without a host round trip.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .core import BatchShape, StaticParams, StepResult, as_params
from .errors import ShapeError
from .level import tensor_to_records, unpack_levels


def _torch():
    import torch

    return torch


class TeacherEnv:
    """amaze/teacher.py:123-147 (the per-episode env; batch it with ``batch_lift``)."""

    step_uses_rng = False

    def action_count(self, params: StaticParams) -> int:
        return as_params(params).n_interior

    def episode_length(self, params: StaticParams) -> int:
        return as_params(params).wall_budget + 2


class TeacherLanes:
    """Owner of one amz_teacher_t (design lanes in HBM)."""

    def __init__(self, params: StaticParams, n: int, device):
        self.params, self.n, self.device = params, n, device
        h = ctypes.c_void_p()
        with _torch().cuda.device(device):
            _lib.call("amz_teacher_create", ctypes.byref(params.c_struct()), n, ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h is not None and h.value and _lib._lib is not None:
                _lib._lib.amz_teacher_destroy(h)
        except (AttributeError, TypeError):  # interpreter shutdown
            pass
        self.handle = None

    def stream(self) -> int:
        return _lib.stream_handle(self.device)


class TeacherBatchEnv:
    """batch_lift(TeacherEnv(), shape): GenericBatchEnv semantics (env/batch.py:118-167)."""

    def __init__(self, env: TeacherEnv, shape: BatchShape, device=None):
        torch = _torch()
        self.env = env
        self.shape = shape
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lanes = None

    @property
    def n_lanes(self) -> int:
        return self.shape.n_agents * self.shape.flat_size

    def action_count(self, params) -> int:
        return self.env.action_count(params)

    def _reshape(self, x):
        return x.reshape(self.shape.n_agents, self.shape.flat_size, *x.shape[1:])

    def _outputs(self, p):
        torch = _torch()
        n = self.n_lanes
        return (torch.empty((n, p.height, p.width), dtype=torch.uint8, device=self.device),
                torch.empty((n, 4), dtype=torch.float32, device=self.device),
                torch.empty((n,), dtype=torch.int64, device=self.device))

    def reset(self, rng, params) -> StepResult:
        torch = _torch()
        p = as_params(params).validate()
        if self.lanes is None or self.lanes.params != p:
            self.lanes = TeacherLanes(p, self.n_lanes, self.device)
        grid, phase, n_placed = self._outputs(p)
        _lib.call("amz_teacher_reset", self.lanes.handle, _lib.ptr(grid), _lib.ptr(phase), _lib.ptr(n_placed),
                  self.lanes.stream())
        n = self.n_lanes
        obs = {"grid": self._reshape(grid), "phase": self._reshape(phase), "n_placed": self._reshape(n_placed)}
        return StepResult(obs, self.lanes, self._reshape(torch.zeros(n, dtype=torch.float64, device=self.device)),
                          self._reshape(torch.zeros(n, dtype=torch.bool, device=self.device)),
                          {"time": self._reshape(torch.zeros(n, dtype=torch.int64, device=self.device))})

    def step(self, rng, state, actions, params) -> StepResult:
        """One design decision per lane; raises ContractViolation (synchronously) on a
        finished lane or an action outside the interior, as TeacherEnv.step does."""
        torch = _torch()
        lanes = state if isinstance(state, TeacherLanes) else self.lanes
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(actions)
        if tuple(a.shape) != (self.shape.n_agents, self.shape.flat_size):
            raise ShapeError(f"actions shape {tuple(a.shape)} != {(self.shape.n_agents, self.shape.flat_size)}")
        a = a.to(self.device).reshape(-1).to(torch.int64).contiguous()
        grid, phase, n_placed = self._outputs(lanes.params)
        n = self.n_lanes
        done = torch.empty(n, dtype=torch.bool, device=self.device)
        times = torch.empty(n, dtype=torch.int64, device=self.device)
        _lib.call("amz_teacher_step", lanes.handle, _lib.ptr(a), _lib.ptr(grid), _lib.ptr(phase), _lib.ptr(n_placed),
                  _lib.ptr(done), _lib.ptr(times), lanes.stream())
        _lib.call("amz_teacher_check", lanes.handle, lanes.stream())
        obs = {"grid": self._reshape(grid), "phase": self._reshape(phase), "n_placed": self._reshape(n_placed)}
        return StepResult(obs, lanes, self._reshape(torch.zeros(n, dtype=torch.float64, device=self.device)),
                          self._reshape(done), {"time": self._reshape(times)})

    def designed_levels(self, state=None):
        """decode_teacher_level for every lane -> int32 [n, 8] level records on the GPU
        (agent faces north); ContractViolation if a design is unfinished."""
        torch = _torch()
        lanes = state if isinstance(state, TeacherLanes) else self.lanes
        out = torch.empty((self.n_lanes, 8), dtype=torch.int32, device=self.device)
        _lib.call("amz_teacher_levels", lanes.handle, _lib.ptr(out), lanes.stream())
        return out

    def lane_levels(self, state=None) -> list:
        p = (state if isinstance(state, TeacherLanes) else self.lanes).params
        return unpack_levels(tensor_to_records(self.designed_levels(state)), p.height, p.width)


__all__ = ["TeacherEnv", "TeacherBatchEnv"]
