"""ctypes binding of libamaze_b200.so (the C ABI in include/amaze_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, the calls that need one raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, ContractViolation, LevelError, RunnerFault, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMZ_LIB_PATH: a differently-built copy of the same library (tuning experiments only)
LIB_PATH = os.environ.get("AMZ_LIB_PATH") or os.path.join(_HERE, "libamaze_b200.so")

AMZ_RESET_NONE, AMZ_RESET_RESAMPLE, AMZ_RESET_HOME = 0, 1, 2
AMZ_SCORE_MAXMC, AMZ_SCORE_PVL = 0, 1

_ERRORS = {-1: ConfigError, -2: LevelError, -3: ContractViolation, -4: ShapeError, -5: RunnerFault, -6: RunnerFault}


class AmzParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("height", "width", "max_episode_steps", "agent_view_size", "wall_budget", "see_through_walls")]


class AmzSeed(ctypes.Structure):
    _fields_ = [("pool", ctypes.c_uint32 * 4), ("hash_const", ctypes.c_uint32), ("n_words", ctypes.c_uint32)]


class AmzEpisodeStats(ctypes.Structure):
    _fields_ = [("episodes", ctypes.c_void_p), ("mean_return", ctypes.c_void_p),
                ("max_return", ctypes.c_void_p), ("solved_rate", ctypes.c_void_p)]


P, I32, I64, U32, VP = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p
D = ctypes.c_double
_SIGS = {
    "amz_abi_version": ([], I32),
    "amz_last_error": ([], ctypes.c_char_p),
    "amz_validate_params": ([ctypes.POINTER(AmzParams)], I32),
    "amz_seed_prefix": ([P, I32, P, I32, ctypes.POINTER(AmzSeed)], I32),
    "amz_stream_uniform": ([ctypes.POINTER(AmzSeed), P], I32),
    "amz_sample_levels": ([ctypes.POINTER(AmzParams), ctypes.POINTER(AmzSeed), U32, P, I64, P, VP], I32),
    "amz_mutate_levels": ([ctypes.POINTER(AmzParams), ctypes.POINTER(AmzSeed), U32, I64, P, P, I32, P, VP], I32),
    "amz_check_levels": ([ctypes.POINTER(AmzParams), P, I64, ctypes.POINTER(ctypes.c_int64), VP], I32),
    "amz_level_metrics": ([ctypes.POINTER(AmzParams), P, I64, P, P, P, P, VP], I32),
    "amz_policy_head": ([P, I32, I64, I32, ctypes.POINTER(AmzSeed), I32, I64, P, P, P, VP], I32),
    "amz_teacher_create": ([ctypes.POINTER(AmzParams), I64, ctypes.POINTER(ctypes.c_void_p)], I32),
    "amz_teacher_destroy": ([P], I32),
    "amz_teacher_reset": ([P, P, P, P, VP], I32),
    "amz_teacher_step": ([P, P, P, P, P, P, P, VP], I32),
    "amz_teacher_check": ([P, VP], I32),
    "amz_teacher_levels": ([P, P, VP], I32),
    "amz_policy_head_dev": ([P, I32, I64, I32, P, P, I32, I64, P, P, P, VP], I32),
    "amz_env_step_dev": ([P, P, I32, I32, P, P, P, P, P, P, P, P, VP], I32),
    "amz_host_alloc": ([ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], I32),
    "amz_host_free": ([P], I32),
    "amz_env_reset_dr": ([P, ctypes.POINTER(AmzSeed), ctypes.POINTER(AmzSeed), P, P, VP], I32),
    "amz_env_create": ([ctypes.POINTER(AmzParams), I64, ctypes.POINTER(ctypes.c_void_p)], I32),
    "amz_env_destroy": ([P], I32),
    "amz_env_lanes": ([P], I64),
    "amz_env_set_lane_offset": ([P, U32], I32),
    "amz_env_reset_to_levels": ([P, P, P, I64, P, P, VP], I32),
    "amz_env_step": ([P, P, I32, I32, ctypes.POINTER(AmzSeed), U32, P, P, P, P, P, P, VP], I32),
    "amz_env_rollout": ([P, I32, P, I32, ctypes.POINTER(AmzSeed), U32, P, P, P, P, P, P, VP], I32),
    "amz_env_reset_dr_iter": ([P, ctypes.POINTER(AmzSeed), P, P, P, VP], I32),
    "amz_env_rollout_iter": ([P, I32, P, ctypes.POINTER(AmzSeed), P, P, P, P, P, P, P, VP], I32),
    "amz_iter_advance": ([P, U32, VP], I32),
    "amz_copy_h2d": ([P, P, ctypes.c_size_t, I32, VP], I32),
    "amz_copy_d2h": ([P, P, ctypes.c_size_t, I32, VP], I32),
    "amz_env_observe": ([P, P, P, VP], I32),
    "amz_env_levels": ([P, P, VP], I32),
    "amz_env_state": ([P, P, VP], I32),
    "amz_env_set_state": ([P, P, VP], I32),
    "amz_env_check": ([P, VP], I32),
    "amz_gae_score": ([I32, I64, P, P, P, P, D, D, P, I32, I32, P, P, P, P,
                       ctypes.POINTER(AmzEpisodeStats), VP], I32),
    "amz_gae_score_v32": ([I32, I64, P, P, P, P, D, D, P, I32, I32, P, P, P, P,
                           ctypes.POINTER(AmzEpisodeStats), VP], I32),
    "amz_plr_create": ([I64, ctypes.POINTER(ctypes.c_void_p)], I32),
    "amz_plr_destroy": ([P], I32),
    "amz_plr_update": ([P, P, P, P, I64, I64, VP], I32),
    "amz_plr_prepare": ([P, P, I64, VP], I32),
    "amz_plr_sample": ([P, ctypes.POINTER(AmzSeed), I64, D, P, I64, P, P, P, P, VP], I32),
    "amz_plr_sample_proportional": ([P, ctypes.POINTER(AmzSeed), I64, D, D, I64, P, P, P, P, VP], I32),
    "amz_plr_top_q": ([P, I64, I32, P, VP], I32),
    "amz_plr_size": ([P, ctypes.POINTER(ctypes.c_int64), VP], I32),
    "amz_plr_digest": ([P, P, VP], I32),
    "amz_plr_export": ([P, P, P, P, P, P, P, VP], I32),
    "amz_plr_import": ([P, P, P, P, P, P, P, VP], I32),
    "amz_lane_scores": ([I32, I64, P, P, P, P, D, P, I32, I32, P, P, ctypes.POINTER(AmzEpisodeStats), VP], I32),
}

_lib = None


def lib():
    """Load the library once; raise (never fall back) if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RunnerFault(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes, fn.restype = args, res
        if L.amz_abi_version() != 1:
            raise RunnerFault("libamaze_b200.so ABI mismatch")
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().amz_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RunnerFault)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes through as NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    """Raw cudaStream_t of torch's current stream on ``device`` (per call: the caller may
    have switched streams).  torch's raw-stream query skips the Stream object."""
    import torch

    if device is None:
        idx = torch.cuda.current_device()
    elif isinstance(device, int):
        idx = device
    else:
        device = torch.device(device)  # accepts "cuda:0" strings as well as torch.device
        idx = device.index if device.index is not None else torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(idx)
