"""Batched AMaze environment and auto-reset wrapper on the GPU.

Drop-in for ``env/batch.py:24-115`` (``batch_lift``, ``VectorBatchEnv``) and
``env/wrappers.py:16-78`` (``AutoResetWrapper``, ``RESAMPLE``, ``HOME``).  Lane state
lives in HBM behind an ``amz_env_t`` handle; observations, rewards and dones come back
as torch CUDA tensors with the reference's shapes and dtypes
([n_agents, n_evals*n_envs, ...]; view uint8, dir int64, reward float64, done bool,
info solved float64 / time int64).

Ownership differs from the reference in one visible way: ``StepResult.state`` is the
environment's device state itself (the handle), advanced in place by ``step``.  The
reference's wrapper also updates state in place (``env/wrappers.py:72-75``); only a
caller holding on to an *old* ``MazeStateBatch`` would notice.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .amaze import MazeEnv, sample_levels, to_device_levels, to_host_levels
from .core import BatchShape, StaticParams, StepResult, as_params
from .errors import ContractViolation, ShapeError
from .rng import RngStream, as_stream

RESAMPLE = "resample"
HOME = "home"
_MODES = {None: _lib.AMZ_RESET_NONE, RESAMPLE: _lib.AMZ_RESET_RESAMPLE, HOME: _lib.AMZ_RESET_HOME}


def _torch():
    import torch

    return torch


def batch_lift(env, shape: BatchShape):
    """env/batch.py:24-28: any maze env with the vector lane protocol -> VectorBatchEnv;
    the PAIRED designer (teacher.TeacherEnv) -> teacher.TeacherBatchEnv."""
    if hasattr(env, "make_batch") and hasattr(env, "step_batch"):
        return VectorBatchEnv(env, shape)
    from .teacher import TeacherBatchEnv, TeacherEnv

    if isinstance(env, TeacherEnv):
        return TeacherBatchEnv(env, shape)
    raise ShapeError("only the AMaze env and the PAIRED designer are implemented on the GPU")


class DeviceLanes:
    """Owner of one amz_env_t (lane SoA in HBM)."""

    def __init__(self, params: StaticParams, n_lanes: int, device, lane_offset: int = 0):
        torch = _torch()
        self.params = params
        self.n = n_lanes
        self.device = torch.device(device)
        with torch.cuda.device(self.device):
            h = ctypes.c_void_p()
            _lib.call("amz_env_create", ctypes.byref(params.c_struct()), n_lanes, ctypes.byref(h))
        self.handle = h
        if lane_offset:
            _lib.call("amz_env_set_lane_offset", self.handle, ctypes.c_uint32(lane_offset))

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h is not None and h.value and _lib._lib is not None:
                _lib._lib.amz_env_destroy(h)
        except (AttributeError, TypeError):  # interpreter shutdown: module globals already cleared
            pass
        self.handle = None

    def __len__(self):
        return self.n

    def stream(self) -> int:
        return _lib.stream_handle(self.device)

    def levels(self):
        torch = _torch()
        out = torch.empty((self.n, 8), dtype=torch.int32, device=self.device)
        _lib.call("amz_env_levels", self.handle, _lib.ptr(out), self.stream())
        return out

    def state_table(self):
        """[B, 5] int32: row, col, dir, time, terminal."""
        torch = _torch()
        out = torch.empty((self.n, 5), dtype=torch.int32, device=self.device)
        _lib.call("amz_env_state", self.handle, _lib.ptr(out), self.stream())
        return out

    def set_state_table(self, table) -> None:
        t = table.to(self.device).to(_torch().int32).contiguous()
        _lib.call("amz_env_set_state", self.handle, _lib.ptr(t), self.stream())

    def observe(self):
        torch = _torch()
        v = self.params.agent_view_size
        view = torch.empty((self.n, v, v), dtype=torch.uint8, device=self.device)
        dirs = torch.empty((self.n,), dtype=torch.int64, device=self.device)
        _lib.call("amz_env_observe", self.handle, _lib.ptr(view), _lib.ptr(dirs), self.stream())
        return {"view": view, "dir": dirs}

    # reference-style accessors
    def level_at(self, i: int):
        return to_host_levels(self.levels()[i: i + 1], self.params)[0]

    def lane_levels(self) -> list:
        return to_host_levels(self.levels(), self.params)


class VectorBatchEnv:
    """env/batch.py:78-115 on device lanes."""

    def __init__(self, env=None, shape: BatchShape = BatchShape(), device=None, lane_offset: int = 0):
        torch = _torch()
        self.env = env if env is not None else MazeEnv()
        if getattr(self.env, "step_uses_rng", False):
            raise ShapeError("vector batching requires an env with deterministic stepping")
        self.shape = shape
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lane_offset = lane_offset
        self.lanes: DeviceLanes | None = None

    @property
    def n_lanes(self) -> int:
        return self.shape.n_agents * self.shape.flat_size

    def action_count(self, params=None) -> int:
        return 3

    # -- helpers ---------------------------------------------------------------
    def _ensure(self, params: StaticParams) -> DeviceLanes:
        if self.lanes is None or self.lanes.params != params:
            self.lanes = DeviceLanes(params, self.n_lanes, self.device, self.lane_offset)
        return self.lanes

    def _reshape(self, t):
        return t.reshape(self.shape.n_agents, self.shape.flat_size, *t.shape[1:])

    def _expand(self, levels):
        """env/batch.py:56-66: n_envs levels are replicated over evals and agents."""
        torch = _torch()
        n = levels.shape[0]
        if n == self.n_lanes:
            return levels
        if n != self.shape.n_envs:
            raise ShapeError(f"expected {self.shape.n_envs} levels (or {self.n_lanes} pre-flattened), got {n}")
        idx = torch.arange(self.shape.flat_size, device=levels.device) % self.shape.n_envs
        return levels[idx.repeat(self.shape.n_agents)].contiguous()

    def _flat_actions(self, actions):
        torch = _torch()
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(actions)
        expect = (self.shape.n_agents, self.shape.flat_size)
        if tuple(a.shape) != expect:
            raise ShapeError(f"actions shape {tuple(a.shape)} != {expect}")
        a = a.to(self.device).reshape(-1)
        if a.dtype == torch.uint8:
            return a.contiguous(), 0
        if a.dtype == torch.int32:
            return a.contiguous(), 1
        return a.to(torch.int64).contiguous(), 2

    def _zeros_result(self, obs, state):
        """reset results carry zero reward/done/info (env/batch.py:91-96); the zero
        tensors are allocated once per env and shared read-only across resets."""
        torch = _torch()
        if getattr(self, "_zeros", None) is None or self._zeros[0].numel() != self.n_lanes:
            n = self.n_lanes
            self._zeros = (torch.zeros(n, dtype=torch.float64, device=self.device),
                           torch.zeros(n, dtype=torch.bool, device=self.device),
                           torch.zeros(n, dtype=torch.int64, device=self.device))
        zf, zb, zi = self._zeros
        info = {"solved": self._reshape(zf), "time": self._reshape(zi)}
        return StepResult({k: self._reshape(v) for k, v in obs.items()}, state, self._reshape(zf),
                          self._reshape(zb), info)

    # -- reference API ---------------------------------------------------------
    def reset(self, rng, params, _prepare_wrap: RngStream | None = None) -> StepResult:
        """Level generation and reset in one launch (lane l plays the level of key
        rng.key + (lane_offset + l,), as sample_levels + reset_to_levels would).
        ``_prepare_wrap`` (AutoResetWrapper, RESAMPLE) also prepares the lanes'
        timeout levels for the first rollout under that wrapper key."""
        torch = _torch()
        p = as_params(params).validate()
        lanes = self._ensure(p)
        v = p.agent_view_size
        view = torch.empty((self.n_lanes, v, v), dtype=torch.uint8, device=self.device)
        dirs = torch.empty((self.n_lanes,), dtype=torch.int64, device=self.device)
        seed = as_stream(rng).seed_prefix()
        wseed = _prepare_wrap.seed_prefix() if _prepare_wrap is not None else None
        _lib.call("amz_env_reset_dr", lanes.handle, ctypes.byref(seed),
                  ctypes.byref(wseed) if wseed is not None else None, _lib.ptr(view), _lib.ptr(dirs),
                  lanes.stream())
        return self._zeros_result({"view": view, "dir": dirs}, lanes)

    def reset_to_levels(self, rng, levels, params) -> StepResult:
        torch = _torch()
        p = as_params(params).validate()
        lanes = self._ensure(p)
        lv = self._expand(to_device_levels(levels, p, self.device))
        v = p.agent_view_size
        view = torch.empty((self.n_lanes, v, v), dtype=torch.uint8, device=self.device)
        dirs = torch.empty((self.n_lanes,), dtype=torch.int64, device=self.device)
        _lib.call("amz_env_reset_to_levels", lanes.handle, _lib.ptr(lv), None, self.n_lanes, _lib.ptr(view),
                  _lib.ptr(dirs), lanes.stream())
        return self._zeros_result({"view": view, "dir": dirs}, lanes)

    def _step(self, state, actions, params, mode: int, wrap: RngStream | None, step_idx: int,
              out: dict | None = None) -> StepResult:
        """``out`` may hold flat-lane destination tensors (``view`` u8 [n,V,V], ``dir``
        int64 [n], ``reward`` f64 [n], ``done`` bool [n]), e.g. slices of a trajectory
        store, which the step kernel then writes directly."""
        torch = _torch()
        p = as_params(params)
        lanes = state if isinstance(state, DeviceLanes) else self.lanes
        if lanes is None:
            raise ContractViolation("step before reset")
        a, code = self._flat_actions(actions)
        n, v = self.n_lanes, p.agent_view_size
        o = out or {}
        view = o["view"] if "view" in o else torch.empty((n, v, v), dtype=torch.uint8, device=self.device)
        dirs = o["dir"] if "dir" in o else torch.empty((n,), dtype=torch.int64, device=self.device)
        rew = o["reward"] if "reward" in o else torch.empty((n,), dtype=torch.float64, device=self.device)
        done = o["done"] if "done" in o else torch.empty((n,), dtype=torch.bool, device=self.device)
        for name, x, dt in (("view", view, torch.uint8), ("dir", dirs, torch.int64), ("reward", rew, torch.float64),
                            ("done", done, torch.bool)):
            if x.dtype != dt or not x.is_contiguous() or x.numel() != (n * v * v if name == "view" else n):
                raise ShapeError(f"step output {name!r} must be a contiguous {dt} tensor of the lane count")
        solved = torch.empty((n,), dtype=torch.float64, device=self.device)
        times = torch.empty((n,), dtype=torch.int64, device=self.device)
        seed = wrap.seed_prefix() if wrap is not None else None
        _lib.call("amz_env_step", lanes.handle, _lib.ptr(a), code, mode,
                  ctypes.byref(seed) if seed is not None else None, ctypes.c_uint32(step_idx),
                  _lib.ptr(view), _lib.ptr(dirs), _lib.ptr(rew), _lib.ptr(done), _lib.ptr(solved),
                  _lib.ptr(times), lanes.stream())
        if mode == _lib.AMZ_RESET_NONE:
            _lib.call("amz_env_check", lanes.handle, lanes.stream())
        obs = {"view": self._reshape(view), "dir": self._reshape(dirs)}
        info = {"solved": self._reshape(solved), "time": self._reshape(times)}
        return StepResult(obs, lanes, self._reshape(rew), self._reshape(done), info)

    def step(self, rng, state, actions, params) -> StepResult:
        """Bare step (no auto-reset): terminal lanes raise ContractViolation next step."""
        return self._step(state, actions, params, _lib.AMZ_RESET_NONE, None, 0)

    def lane_levels(self, state=None) -> list:
        return (state if isinstance(state, DeviceLanes) else self.lanes).lane_levels()

    def lane_levels_tensor(self, state=None):
        return (state if isinstance(state, DeviceLanes) else self.lanes).levels()

    def reset_lanes(self, state, lanes, levels, params):
        """env/batch.py:107-115: reset the given flat lanes to ``levels``; returns
        (state, flat observations of those lanes)."""
        torch = _torch()
        p = as_params(params)
        dl = state if isinstance(state, DeviceLanes) else self.lanes
        idx = _lane_indices(lanes, dl.n).to(self.device)
        lv = to_device_levels(levels, p, self.device)
        if lv.shape[0] != idx.numel():
            raise ShapeError(f"{idx.numel()} lanes vs {lv.shape[0]} levels")
        v = p.agent_view_size
        view = torch.empty((idx.numel(), v, v), dtype=torch.uint8, device=self.device)
        dirs = torch.empty((idx.numel(),), dtype=torch.int64, device=self.device)
        _lib.call("amz_env_reset_to_levels", dl.handle, _lib.ptr(lv), _lib.ptr(idx), idx.numel(), _lib.ptr(view),
                  _lib.ptr(dirs), dl.stream())
        return dl, {"view": view, "dir": dirs}


def _lane_indices(lanes, n: int):
    """numpy's indexing rules for ``state.replace_lanes(lanes, ...)`` (amaze/env.py:308-313):
    a bool mask of length n selects its True lanes, negative indices wrap once, anything
    outside [-n, n) raises IndexError.  Checked on the host (this path is not the fused
    hot path; a device tensor is read back) so the kernel never sees an invalid lane."""
    torch = _torch()
    t = torch.as_tensor(lanes).detach().cpu()
    if t.dtype == torch.bool:
        if t.dim() != 1 or t.numel() != n:
            raise IndexError(f"boolean lane mask of shape {tuple(t.shape)} does not match {n} lanes")
        return t.nonzero().reshape(-1).to(torch.int64).contiguous()
    if t.is_floating_point() or t.is_complex():
        raise IndexError("lane indices must be integers or a boolean mask")
    t = t.to(torch.int64).reshape(-1)
    if t.numel() and (int(t.min()) < -n or int(t.max()) >= n):
        bad = int(t.min()) if int(t.min()) < -n else int(t.max())
        raise IndexError(f"lane index {bad} is out of bounds for {n} lanes")
    return torch.where(t < 0, t + n, t).contiguous()


class AutoResetWrapper:
    """env/wrappers.py:20-78 with the reset fused into the step kernel."""

    EXTRAS_KEY = "autoreset"

    def __init__(self, batch_env: VectorBatchEnv, mode: str = RESAMPLE):
        if mode not in (RESAMPLE, HOME):
            raise ContractViolation(f"unknown auto-reset mode {mode!r}")
        self.benv = batch_env
        self.mode = mode

    @property
    def shape(self):
        return self.benv.shape

    def action_count(self, params=None):
        return self.benv.action_count(params)

    def reset(self, rng, params) -> StepResult:
        rng_env, rng_wrap = as_stream(rng).split(2)
        prep = rng_wrap if self.mode == RESAMPLE and isinstance(self.benv, VectorBatchEnv) else None
        res = self.benv.reset(rng_env, params, prep) if prep is not None else self.benv.reset(rng_env, params)
        return self._attach(res, rng_wrap)

    def reset_to_levels(self, rng, levels, params) -> StepResult:
        rng_env, rng_wrap = as_stream(rng).split(2)
        return self._attach(self.benv.reset_to_levels(rng_env, levels, params), rng_wrap)

    def _attach(self, result: StepResult, rng_wrap: RngStream) -> StepResult:
        home = self.benv.lane_levels_tensor(result.state) if self.mode == HOME else None
        result.extras = dict(result.extras)
        result.extras[self.EXTRAS_KEY] = {"rng": rng_wrap, "step": 0, "home": home}
        return result

    def step(self, rng, state, actions, params, extras: dict, out: dict | None = None) -> StepResult:
        wrap = extras[self.EXTRAS_KEY]
        res = self.benv._step(state, actions, params, _MODES[self.mode],
                              wrap["rng"] if self.mode == RESAMPLE else None, int(wrap["step"]), out=out)
        res.extras = dict(extras)
        res.extras[self.EXTRAS_KEY] = {**wrap, "step": wrap["step"] + 1}
        return res
