"""The DR iteration (configs[1]) as ONE CUDA-graph replay per step.

One step of the hot path is: DR level generation + reset of every lane
(``AutoResetWrapper.reset(root.fold_in(it))``, env/wrappers.py:43-56), T fused
RESAMPLE-auto-reset env steps driven by the policy's action stream (the env side of
agents/rollout.py:120-152), and GAE + MaxMC/PVL scores (agents/gae.py:8-37,
runners/scoring.py:34-63).  Eagerly that is 4 kernels plus ~0.1-0.2 ms of Python/ctypes
enqueue per step -- more than the kernels take at 4096 lanes.  Here the whole step is
captured once: the iteration's key streams come from a device iteration counter
(``amz_env_reset_dr_iter`` / ``amz_env_rollout_iter``, advanced by the graph itself), so
a replay needs no host-side key work, and the host's cost per step is one
``cudaGraphLaunch``.

``host_io=True`` captures the end-to-end form: the step's inputs (actions u8 [T, B],
values [T, B] and last values [B] in ``value_dtype``) are copied host->device from
pinned staging at the start of the graph and scores | max returns (float64 [2, B]) are
copied device->host at the end.  With ``overlap=True`` two graphs alternate between two
device input buffers and each copies the NEXT step's inputs on a side stream while it
computes the current step (the copy engines and the SMs work at the same time).

Results equal the eager calls bit for bit (tests/test_gpu_graph.py).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .batch import RESAMPLE, AutoResetWrapper, VectorBatchEnv
from .core import as_params
from .errors import ContractViolation
from .gae import gae_and_scores
from .host import pinned_empty
from .rng import as_stream


def _torch():
    import torch

    return torch


class DRIterationGraph:
    """Captured DR iteration over ``benv`` (a VectorBatchEnv of B lanes) with T steps.

    ``step(it)`` replays iteration ``it`` (keys root.fold_in(it)); iterations normally
    run in order (the graph advances its device counter), a jump costs one small
    synchronous copy.  Outputs live in ``self.out`` (trajectory tensors), ``self.gae``
    (advantages / returns / scores / max_returns) and, with ``host_io``, ``self.host_result``
    (pinned float64 [2, B]: scores | max returns of the last completed step)."""

    def __init__(self, benv: VectorBatchEnv, root_rng, T: int, params, gamma: float, lam: float,
                 score_fn: str = "maxmc", value_dtype=None, host_io: bool = False, overlap: bool = True,
                 copy_streams: int = 1, copy_ctas: int = 64):
        torch = _torch()
        if not isinstance(benv, VectorBatchEnv):
            raise ContractViolation("DRIterationGraph needs a VectorBatchEnv")
        self.torch = torch
        self.benv = benv
        self.env = AutoResetWrapper(benv, RESAMPLE)
        self.p = as_params(params).validate()
        self.T, self.B = int(T), benv.n_lanes
        self.gamma, self.lam, self.score_fn = float(gamma), float(lam), score_fn
        self.dev = benv.device
        self.vdt = value_dtype or torch.float64
        self.root = as_stream(root_rng)
        self.root_pfx = self.root.seed_prefix()
        self.host_io = host_io
        self.overlap = overlap and host_io
        self.copy_streams = 1
        self.copy_ctas = int(copy_ctas)
        T, B, dev, v = self.T, self.B, self.dev, self.p.agent_view_size
        self.it_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.next_it = 0
        nbuf = 2 if self.overlap else 1
        # one contiguous byte buffer per input slot (values | last values | actions), so the
        # host->device copy is two large copies (one per DMA engine) instead of three
        es = torch.empty((), dtype=self.vdt).element_size()
        self._nv, self._nl, self._na = T * B * es, B * es, T * B
        self._nbytes = self._nv + self._nl + self._na
        self._raw = [torch.zeros(self._nbytes, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
        self.inputs = [self._views(r) for r in self._raw]
        self.out = {"view": torch.empty((T, B, v, v), dtype=torch.uint8, device=dev),
                    "dir": torch.empty((T, B), dtype=torch.uint8, device=dev),
                    "rewards": torch.empty((T, B), dtype=torch.float64, device=dev),
                    "dones": torch.empty((T, B), dtype=torch.bool, device=dev),
                    "final_view": torch.empty((B, v, v), dtype=torch.uint8, device=dev),
                    "final_dir": torch.empty((B,), dtype=torch.uint8, device=dev),
                    "reset_view": torch.empty((B, v, v), dtype=torch.uint8, device=dev),
                    "reset_dir": torch.empty((B,), dtype=torch.int64, device=dev)}
        self.res = torch.empty((2, B), dtype=torch.float64, device=dev)  # scores | max returns
        self.gae = {"advantages": torch.empty((T, B), dtype=torch.float64, device=dev),
                    "returns": torch.empty((T, B), dtype=torch.float64, device=dev),
                    "scores": self.res[0], "max_returns": self.res[1]}
        if host_io:
            self._host_raw = pinned_empty((self._nbytes,), torch.uint8)
            self.host_inputs = self._views(self._host_raw)
            self.host_result = pinned_empty((2, B), torch.float64)
        self.graphs = []
        self.launches_per_step = 5  # k_env_reset_dr, k_dyn, k_render, k_gae_score*, k_iter_advance
        self._step_count = 0
        self._pending_h2d = False

    # -- one step's kernels on the current stream ------------------------------------
    def _kernels(self, inp, after_reset=None):
        """The step's kernels on the current stream; ``after_reset()`` runs right after the
        reset kernel is enqueued (the overlapped input copy forks there: the reset fills
        every SM's register file, the dynamics kernel leaves room beside it)."""
        torch = self.torch
        lanes = self.benv._ensure(self.p)
        o = self.out
        st = lanes.stream()
        _lib.call("amz_env_reset_dr_iter", lanes.handle, ctypes.byref(self.root_pfx), _lib.ptr(self.it_dev),
                  _lib.ptr(o["reset_view"]), _lib.ptr(o["reset_dir"]), st)
        if after_reset is not None:
            after_reset()
        _lib.call("amz_env_rollout_iter", lanes.handle, self.T, _lib.ptr(inp["actions"]), ctypes.byref(self.root_pfx),
                  _lib.ptr(self.it_dev), _lib.ptr(o["view"]), _lib.ptr(o["dir"]), _lib.ptr(o["rewards"]),
                  _lib.ptr(o["dones"]), _lib.ptr(o["final_view"]), _lib.ptr(o["final_dir"]), st)
        gae_and_scores(o["rewards"], inp["values"], o["dones"], inp["last"], self.gamma, self.lam,
                       score_fn=self.score_fn, out=self.gae)
        _lib.call("amz_iter_advance", _lib.ptr(self.it_dev), 1, st)
        del torch

    def _views(self, raw):
        T, B, nv, nl = self.T, self.B, self._nv, self._nl
        return {"values": raw[:nv].view(self.vdt).view(T, B), "last": raw[nv:nv + nl].view(self.vdt),
                "actions": raw[nv + nl:].view(T, B)}

    def _h2d(self, k, streams=None):
        """Copy the pinned staging into input slot k with ``amz_copy_h2d`` (a kernel
        reading the pinned buffer through its unified address: measured 46 GB/s, where a
        graph memcpy node from the same host buffer ran at 19-50 GB/s from one box to the
        next), on the given side stream (or the current one)."""
        torch = self.torch
        st = streams[0] if streams else torch.cuda.current_stream(self.dev)
        _lib.call("amz_copy_h2d", self._raw[k].data_ptr(), self._host_raw.data_ptr(), self._nbytes, self.copy_ctas,
                  st.cuda_stream)

    def capture(self):
        """Warm up (allocates the rollout scratch) and capture the graph(s)."""
        torch = self.torch
        with torch.cuda.device(self.dev):
            s = torch.cuda.Stream(device=self.dev)
            s.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(s):
                self._kernels(self.inputs[0])  # warm-up: scratch allocation, attributes
            torch.cuda.current_stream(self.dev).wait_stream(s)
            torch.cuda.synchronize(self.dev)
            self.graphs = []
            for k in range(len(self.inputs)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    cur = torch.cuda.current_stream(self.dev)
                    if self.host_io and not self.overlap:
                        self._h2d(k)
                    sides = []
                    if self.overlap:
                        # the next step's inputs on a side branch forked after the reset,
                        # concurrent with the dynamics / render / GAE kernels
                        sides = [torch.cuda.Stream(device=self.dev, priority=-5)]

                        def fork(k=k, sides=sides, cur=cur):
                            sides[0].wait_stream(cur)
                            self._h2d(k ^ 1, sides)
                    self._kernels(self.inputs[k], fork if self.overlap else None)
                    if self.host_io:
                        self.host_result.copy_(self.res, non_blocking=True)
                    if self.overlap:
                        for sd in sides:
                            cur.wait_stream(sd)
                self.graphs.append(g)
            torch.cuda.synchronize(self.dev)
        self.set_iteration(0)
        return self

    def set_iteration(self, it: int) -> None:
        """Point the device counter at iteration ``it`` (synchronous)."""
        if not 0 <= it < 2 ** 32:
            raise ContractViolation(f"iteration {it} outside the u32 counter range")
        torch = self.torch
        torch.cuda.synchronize(self.dev)
        self.it_dev.fill_(int(it) if it < 2 ** 31 else int(it) - 2 ** 32)
        torch.cuda.synchronize(self.dev)
        self.next_it = int(it)
        self._pending_h2d = False

    def prefetch(self):
        """overlap mode: copy the first step's inputs (later steps' copies ride along in
        the previous replay)."""
        if self.overlap:
            with self.torch.cuda.device(self.dev):
                self._h2d(self._step_count & 1)
            self._pending_h2d = True

    def step(self, it: int | None = None):
        """Replay one iteration (``it`` defaults to the next in order)."""
        if not self.graphs:
            self.capture()
        if it is not None and it != self.next_it:
            self.set_iteration(it)
        if self.overlap and not self._pending_h2d:
            self.prefetch()
        self.graphs[self._step_count % len(self.graphs)].replay()
        self._step_count += 1
        self.next_it += 1
        return self.gae


__all__ = ["DRIterationGraph"]
