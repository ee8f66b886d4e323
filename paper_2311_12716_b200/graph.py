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
pinned staging and scores | max returns (float64 [2, B]) are copied device->host at the
end of the graph.  With ``overlap=True`` (the default) two graphs alternate between two
device input slots and the copy of the NEXT step's inputs runs on its own copy stream
while the current step computes: the copy into slot k waits (event) only for the graph
that last read slot k, and the graph waits only for its own slot's copy, so the PCIe
transfer and the kernels pipeline across steps instead of joining inside one replay
(measured: 5.3 MB takes ~100 us over PCIe, the step's kernels ~135 us).  Host-side
contract of that pipeline: ``step(k)`` starts copying ``host_inputs`` for step k+1, so
the staging must hold step k+1's inputs when ``step(k)`` is called (the first step's
inputs are copied by ``prefetch()``, which ``step`` calls if needed) and must not be
rewritten until ``step(k+1)`` has been enqueued and the copy finished (synchronize, or
keep two host stagings).  ``host_result`` holds step k's scores | max returns once the
stream has passed step k.  Without overlap the copy is the first node of the graph and
``host_inputs`` belong to the step being called.

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
    (pinned float64 [2, B]: scores | max returns of the last completed step).

    host_io options: ``overlap`` pipelines the feed one step ahead on its own stream;
    ``copy_mode`` picks the H2D path ("kernel": ``amz_copy_h2d`` with ``copy_ctas`` CTAs,
    "engine": copy-engine memcpy split over ``copy_streams`` streams, "auto": the kernel
    until ``calibrate()`` -- run once by itself after ``calibrate_after`` steps -- times
    both and keeps the faster)."""

    def __init__(self, benv: VectorBatchEnv, root_rng, T: int, params, gamma: float, lam: float,
                 score_fn: str = "maxmc", value_dtype=None, host_io: bool = False, overlap: bool = True,
                 copy_streams: int = 1, copy_ctas: int = 32, copy_mode: str = "auto"):
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
        self.copy_streams = max(1, int(copy_streams))
        self.copy_ctas = int(copy_ctas)
        if copy_mode not in ("auto", "kernel", "engine"):
            raise ContractViolation(f"copy_mode {copy_mode!r}: 'auto', 'kernel' or 'engine'")
        self.copy_mode = copy_mode
        self.copy_engine = copy_mode == "engine"  # auto: the kernel until calibrate() decides
        self.calibrate_after = 200  # auto: steps before the one-off calibration
        self.calibration_ms = None
        T, B, dev, v = self.T, self.B, self.dev, self.p.agent_view_size
        self.it_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.next_it = 0
        nbuf = 2 if self.overlap else 1
        # one contiguous byte buffer per input slot (values | last values | actions): the
        # host->device feed is one copy (or copy_streams pieces with the copy engine)
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
        self._iter_stream = torch.cuda.Stream(device=dev)  # the counter advance beside GAE
        self._step_count = 0
        self._pending_h2d = False
        if self.overlap:
            # the copy stream(s): one for the copy kernel; copy-engine memcpys split the
            # bytes over copy_streams streams (one DMA engine each)
            self._cs = [torch.cuda.Stream(device=dev, priority=-5) for _ in range(self.copy_streams)]
            self._copied = [torch.cuda.Event() for _ in range(nbuf)]  # slot k filled
            self._used = [torch.cuda.Event() for _ in range(nbuf)]    # slot k read by its graph

    # -- one step's kernels on the current stream ------------------------------------
    @property
    def launches_per_step(self) -> int:
        """Kernels per step: k_env_reset_dr, k_dyn, k_render, k_gae_score*, k_iter_advance,
        with host_io the result read-back kernel and (unless a copy-engine H2D) the input
        copy kernel."""
        return 5 + (0 if not self.host_io else 1 + (0 if self.copy_engine else 1))

    def _kernels(self, inp):
        """The step's kernels on the current stream; the iteration counter advances on a
        side branch beside GAE (only the reset and the dynamics read it, both done by then)."""
        torch = self.torch
        lanes = self.benv._ensure(self.p)
        o = self.out
        st = lanes.stream()
        cur = torch.cuda.current_stream(self.dev)
        _lib.call("amz_env_reset_dr_iter", lanes.handle, ctypes.byref(self.root_pfx), _lib.ptr(self.it_dev),
                  _lib.ptr(o["reset_view"]), _lib.ptr(o["reset_dir"]), st)
        _lib.call("amz_env_rollout_iter", lanes.handle, self.T, _lib.ptr(inp["actions"]), ctypes.byref(self.root_pfx),
                  _lib.ptr(self.it_dev), _lib.ptr(o["view"]), _lib.ptr(o["dir"]), _lib.ptr(o["rewards"]),
                  _lib.ptr(o["dones"]), _lib.ptr(o["final_view"]), _lib.ptr(o["final_dir"]), st)
        side = self._iter_stream
        side.wait_stream(cur)
        _lib.call("amz_iter_advance", _lib.ptr(self.it_dev), 1, side.cuda_stream)
        gae_and_scores(o["rewards"], inp["values"], o["dones"], inp["last"], self.gamma, self.lam,
                       score_fn=self.score_fn, out=self.gae)
        cur.wait_stream(side)
        del torch

    def _views(self, raw):
        T, B, nv, nl = self.T, self.B, self._nv, self._nl
        return {"values": raw[:nv].view(self.vdt).view(T, B), "last": raw[nv:nv + nl].view(self.vdt),
                "actions": raw[nv + nl:].view(T, B)}

    def _h2d(self, k, stream=None):
        """Copy the pinned staging into input slot k with ``amz_copy_h2d`` (a kernel
        reading the pinned buffer through its unified address: measured 49 GB/s, where a
        copy-engine memcpy from the same host buffer ran at 19-50 GB/s from one box to the
        next), on ``stream`` (or the current one)."""
        torch = self.torch
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
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
                    if self.host_io and not self.overlap:
                        self._h2d(k)
                    self._kernels(self.inputs[k])
                    if self.host_io:  # scores | max returns -> pinned host, by a kernel
                        _lib.call("amz_copy_d2h", self.host_result.data_ptr(), self.res.data_ptr(),
                                  self.res.numel() * 8, 8, torch.cuda.current_stream(self.dev).cuda_stream)
                self.graphs.append(g)
            torch.cuda.synchronize(self.dev)
        self.set_iteration(0)
        return self

    def calibrate(self, rounds: int = 3, steps: int = 8) -> bool:
        """Time pipelined steps with each H2D path (alternating, ``rounds`` x ``steps``
        each, median per path) and keep the faster; returns True for the copy engine.
        copy_mode "auto" runs this once by itself after ``calibrate_after`` steps.

        Which path wins depends on the host and on its state.  Measured on B200 boxes
        (tools/e2e_content.py, tools/pcie_interference.py): a copy-engine memcpy leaves the
        SMs to the step (90 -> 101 us per step beside it) where the copy kernel takes SM
        slots (90 -> 150 us), and in steady state the engine path wins (152 vs 165 us per
        step); but for ~100-300 steps after the host CPU writes the pinned feed, PCIe
        reads of it run 2-4x slower, the engine's worst (460 vs 250 us).  Hence the
        decision is taken after a warm-up, not at capture.  The timed steps are real
        iterations; the counter is restored afterwards (every iteration starts from a
        full DR reset, so re-running one is side-effect free)."""
        torch = self.torch
        if not self.overlap:
            return False
        if not self.graphs:
            self.capture()
        resume = self.next_it
        times = {False: [], True: []}
        for _ in range(rounds):
            for ce in (False, True):
                self.copy_engine = ce
                self._pending_h2d = False
                self.step()
                torch.cuda.synchronize(self.dev)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(torch.cuda.current_stream(self.dev))
                for _ in range(steps):
                    self.step()
                b.record(torch.cuda.current_stream(self.dev))
                torch.cuda.synchronize(self.dev)
                times[ce].append(a.elapsed_time(b) / steps)
        med = {ce: sorted(v)[len(v) // 2] for ce, v in times.items()}
        self.copy_engine = med[True] < med[False]
        self.calibration_ms = med
        self.set_iteration(resume)
        return self.copy_engine

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

    def _issue_copy(self, k):
        """overlap mode: fill slot k from the pinned staging on the copy stream, after the
        graph that last read slot k."""
        if not self.copy_engine:
            cs = self._cs[0]
            cs.wait_event(self._used[k])
            self._h2d(k, cs)
            self._copied[k].record(cs)
            return
        torch = self.torch
        n, m = self._nbytes, len(self._cs)
        part = ((n + m - 1) // m + 4095) & ~4095
        first = self._cs[0]
        first.wait_event(self._used[k])
        for j, cs in enumerate(self._cs):
            if j:
                cs.wait_stream(first)
            lo, hi = j * part, min(n, (j + 1) * part)
            if lo < hi:
                with torch.cuda.stream(cs):
                    self._raw[k][lo:hi].copy_(self._host_raw[lo:hi], non_blocking=True)
        for cs in self._cs[1:]:
            first.wait_stream(cs)
        self._copied[k].record(first)

    def prefetch(self):
        """overlap mode: copy the first step's inputs (every later step's copy is issued
        one step ahead, concurrent with the previous step's kernels)."""
        if self.overlap:
            with self.torch.cuda.device(self.dev):
                self._issue_copy(self._step_count % len(self.graphs))
            self._pending_h2d = True

    def step(self, it: int | None = None):
        """Replay one iteration (``it`` defaults to the next in order)."""
        if not self.graphs:
            self.capture()
        if it is not None and it != self.next_it:
            self.set_iteration(it)
        if (self.overlap and self.copy_mode == "auto" and self.calibration_ms is None
                and self._step_count >= self.calibrate_after):
            self.calibration_ms = {}  # (re-entry guard: calibrate() steps too)
            self.calibrate()
        k = self._step_count % len(self.graphs)
        if self.overlap:
            if not self._pending_h2d:
                self.prefetch()
            cur = self.torch.cuda.current_stream(self.dev)
            cur.wait_event(self._copied[k])
            with self.torch.cuda.device(self.dev):
                self._issue_copy(k ^ 1)  # the next step's inputs, beside this step's kernels
            self.graphs[k].replay()
            self._used[k].record(cur)
        else:
            self.graphs[k].replay()
        self._step_count += 1
        self.next_it += 1
        return self.gae


__all__ = ["DRIterationGraph"]
