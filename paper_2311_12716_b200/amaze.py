"""DR level generation, ACCEL mutation and the maze-env marker object, on the GPU.

Drop-in for ``amaze/generator.py:36-84`` (``sample_random_level``, ``mutate_level``)
and the lane-protocol parts of ``amaze/env.py:163-234`` (``MazeEnv``).  Batched entry
points take a parent ``RngStream`` and give level i the key ``parent.key + (lane0 + i,)``
-- the same keys ``VectorBatchEnv.reset`` (``env/batch.py:43-44,86-89``) and the
auto-reset wrapper (``env/wrappers.py:64-67``) derive -- so every level is bit-identical
to the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import StaticParams, as_params
from .errors import ContractViolation, LevelError
from .level import MazeLevel, pack_levels, records_to_tensor, tensor_to_records, unpack_levels
from .rng import RngStream, as_stream

N_ACTIONS = 3  # TURN_LEFT, TURN_RIGHT, FORWARD (amaze/env.py:23-26)
TILE_EMPTY, TILE_WALL, TILE_GOAL, TILE_OOB = 0, 1, 2, 3


def _torch():
    import torch

    return torch


def _split_key(rng: RngStream):
    """A stream's own key as (prefix stream, last word) for single-level calls."""
    if not rng.key:
        raise ContractViolation("single-level generation needs a non-empty stream key "
                                "(use split/fold_in, as the batched env does)")
    return RngStream(rng.entropy, rng.key[:-1]), rng.key[-1]


def sample_levels(rng, n: int, params: StaticParams, lane0: int = 0, lane_ids=None, device=None, out=None):
    """Levels for keys rng.key + (lane0 + i,) (or + (lane_ids[i],)) -> int32 [n, 8] on device
    (into ``out``, a contiguous int32 [n, 8] device tensor, when given)."""
    torch = _torch()
    p = as_params(params).validate()
    rng = as_stream(rng)
    if out is not None:
        if out.shape != (n, 8) or out.dtype != torch.int32 or not out.is_contiguous() or not out.is_cuda:
            raise ContractViolation("out must be a contiguous int32 [n, 8] CUDA tensor")
        dev = out.device
    else:
        dev = device or torch.device("cuda", torch.cuda.current_device())
        out = torch.empty((n, 8), dtype=torch.int32, device=dev)
    ids = None
    if lane_ids is not None:
        ids = torch.as_tensor(lane_ids, device=dev).to(torch.int32).contiguous()
        if ids.numel() != n:
            raise ContractViolation("lane_ids must have n entries")
    seed = rng.seed_prefix()
    _lib.call("amz_sample_levels", ctypes.byref(p.c_struct()), ctypes.byref(seed), ctypes.c_uint32(lane0),
              _lib.ptr(ids), n, _lib.ptr(out), _lib.stream_handle(dev))
    return out


def mutate_levels(rng, parents, n_edits: int, params: StaticParams, lane0: int = 0, parent_idx=None, n=None,
                  out=None):
    """ACCEL edits: out[i] = mutate(parents[parent_idx[i]] or parents[i], key rng.key + (lane0+i,))
    (into ``out``, a contiguous int32 [n, 8] device tensor, when given)."""
    torch = _torch()
    p = as_params(params).validate()
    rng = as_stream(rng)
    if n_edits < 1:
        raise ContractViolation(f"n_mutations must be >= 1, got {n_edits}")
    idx = None
    if parent_idx is not None:
        idx = torch.as_tensor(parent_idx, device=parents.device).to(torch.int32).contiguous()
        n = idx.numel()
    elif n is None:
        n = parents.shape[0]
    if out is None:
        out = torch.empty((n, 8), dtype=torch.int32, device=parents.device)
    elif out.shape != (n, 8) or out.dtype != torch.int32 or not out.is_contiguous() or out.device != parents.device:
        raise ContractViolation("out must be a contiguous int32 [n, 8] tensor on the parents' device")
    seed = rng.seed_prefix()
    _lib.call("amz_mutate_levels", ctypes.byref(p.c_struct()), ctypes.byref(seed), ctypes.c_uint32(lane0), n,
              _lib.ptr(parents.contiguous()), _lib.ptr(idx), int(n_edits), _lib.ptr(out),
              _lib.stream_handle(parents.device))
    return out


def check_levels(levels, params: StaticParams) -> None:
    """Raise LevelError if any packed level breaks MazeLevel invariants (synchronous)."""
    p = as_params(params).validate()
    bad = ctypes.c_int64(-1)
    _lib.call("amz_check_levels", ctypes.byref(p.c_struct()), _lib.ptr(levels.contiguous()), levels.shape[0],
              ctypes.byref(bad), _lib.stream_handle(levels.device))
    if bad.value >= 0:
        raise LevelError(f"level {bad.value} violates the MazeLevel invariants")


@dataclass(frozen=True)
class EnvMetrics:
    """amaze/metrics.py:13-18."""

    n_walls: int  # interior walls only
    shortest_path_length: int  # agent -> goal, 0 if unsolvable
    solvable: bool
    passable_ratio: float  # fraction of interior cells that are non-wall


def level_metrics(levels, params: StaticParams) -> dict:
    """Batched env_metrics (amaze/metrics.py:21-31) of packed device levels (int32 [N, 8]
    tensor, or anything ``to_device_levels`` accepts): dict of CUDA tensors
    ``n_walls`` int32, ``shortest_path_length`` int32, ``solvable`` bool,
    ``passable_ratio`` float64, each [N]."""
    torch = _torch()
    p = as_params(params).validate()
    lv = to_device_levels(levels, p)
    n = lv.shape[0]
    dev = lv.device
    out = {"n_walls": torch.empty(n, dtype=torch.int32, device=dev),
           "shortest_path_length": torch.empty(n, dtype=torch.int32, device=dev),
           "solvable": torch.empty(n, dtype=torch.bool, device=dev),
           "passable_ratio": torch.empty(n, dtype=torch.float64, device=dev)}
    _lib.call("amz_level_metrics", ctypes.byref(p.c_struct()), _lib.ptr(lv), n, _lib.ptr(out["n_walls"]),
              _lib.ptr(out["shortest_path_length"]), _lib.ptr(out["solvable"]), _lib.ptr(out["passable_ratio"]),
              _lib.stream_handle(dev))
    return out


def env_metrics(level, params: StaticParams | None = None) -> EnvMetrics:
    """amaze/metrics.py:21 for one level (ours or the reference's MazeLevel); the grid
    shape comes from the level when ``params`` is omitted."""
    ml = MazeLevel.from_any(level)
    if params is None:
        h, w = np.asarray(ml.walls).shape
        params = StaticParams(height=int(h), width=int(w), wall_budget=min(60, (int(h) - 2) * (int(w) - 2) - 2))
    m = level_metrics([ml], params)
    return EnvMetrics(int(m["n_walls"][0]), int(m["shortest_path_length"][0]), bool(m["solvable"][0]),
                      float(m["passable_ratio"][0]))


def to_device_levels(levels, params: StaticParams, device=None):
    """MazeLevel-like list (ours or the reference's) or an int32 [N, 8] tensor -> device tensor."""
    torch = _torch()
    if isinstance(levels, torch.Tensor):
        return levels.to(device or levels.device).to(torch.int32).contiguous()
    ml = [MazeLevel.from_any(lv).validate() for lv in levels]
    p = as_params(params)
    return records_to_tensor(pack_levels(ml, p.height, p.width), device or "cuda")


def to_host_levels(levels, params: StaticParams) -> list:
    p = as_params(params)
    return unpack_levels(tensor_to_records(levels), p.height, p.width)


def sample_random_level(rng, params: StaticParams) -> MazeLevel:
    """Drop-in for amaze/generator.py:36-52 (one level; synchronous)."""
    parent, last = _split_key(as_stream(rng))
    return to_host_levels(sample_levels(parent, 1, params, lane0=last), params)[0]


def mutate_level(rng, level, n_mutations: int, params: StaticParams) -> MazeLevel:
    """Drop-in for amaze/generator.py:55-84 (one level; synchronous)."""
    if n_mutations < 1:
        raise ContractViolation(f"n_mutations must be >= 1, got {n_mutations}")
    parent, last = _split_key(as_stream(rng))
    par = to_device_levels([level], params)
    return to_host_levels(mutate_levels(parent, par, n_mutations, params, lane0=last), params)[0]


class MazeEnv:
    """The vector-lane maze environment (amaze/env.py:163-234).  Stepping happens in
    ``batch.VectorBatchEnv``; this object carries the static facts the batching layer
    and callers query."""

    step_uses_rng = False

    def action_count(self, params=None) -> int:
        return N_ACTIONS

    def observation_spec(self, params) -> dict:
        v = as_params(params).agent_view_size
        return {"view": ((v, v), 4), "dir": ((), 4)}

    def sample_level(self, rng, params) -> MazeLevel:
        return sample_random_level(rng, params)

    # make_batch/step_batch presence lets batch_lift pick the vector path
    def make_batch(self, levels):  # pragma: no cover - protocol marker
        raise NotImplementedError("use batch.VectorBatchEnv")

    def step_batch(self, *a, **k):  # pragma: no cover - protocol marker
        raise NotImplementedError("use batch.VectorBatchEnv")


def levels_equal(a, b) -> bool:
    """Exact equality of two packed level tensors (walls + pose bytes)."""
    ra, rb = tensor_to_records(a), tensor_to_records(b)
    fields = ("walls", "agent_r", "agent_c", "agent_dir", "goal_r", "goal_c")
    return all(np.array_equal(ra[f], rb[f]) for f in fields)
