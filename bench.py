"""Benchmark of the AMaze + PLR hot path (BASELINE.json configs[1] by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the hot path over one batch of synthetic input (config 2,
"AMaze 13x13 DR with PPO rollout batch 4096 envs x 256 steps and GAE on 1xB200"):
  1.+2. DR level generation for every lane (keys (seed, (0, lane))) fused with the reset
     of every lane (VectorBatchEnv.reset),
  3. 256 fused env steps with RESAMPLE auto-reset driven by a uint8 [T, B] action
     stream resident in HBM (the policy is out of scope; its values are a resident
     float64 [T, B] tensor),
  4. GAE (gamma 0.995, lambda 0.98: the paper's DR column) + MaxMC
     regret scores + running max returns.
metric = env-steps/s = lanes * T / step time (whole job, all ranks).

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (one per GPU, NCCL); it fails if fewer than N GPUs
are visible.  Each rank runs its own lane shard of the headline workload (global lane
ids rank*B + i, so the keys equal a 1-GPU run over N*B lanes): weak scaling, no
data-path collective.  The ``parallel_plr`` key is configs[4]: 32768 GLOBAL lanes of a
PLR|| iteration split over the N ranks with the NCCL candidate all-gather (strong).

--impl reference times the reference itself (the unmodified autocurricula package
installed into baseline/_ref, driven through its public API: AutoResetWrapper /
batch_lift / compute_gae / lane_scores) on the host cores, lane-sharded over worker
processes, rank 0 only; without baseline/_ref it falls back to the oracle port
(oracle/amaze_np.py, bit-exact with the reference) and says so (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
GAMMA, LAMBDA = 0.995, 0.98  # PAPER.md:334-335, DR column
ENV_BYTES_PER_STEP = 36  # action u8 + view 25 u8 + dir u8 + reward f64 + done u8
GAE_BYTES_PER_ELEM = 33  # r f64 + V f64 + done u8 in, A f64 + R f64 out


PROFILE_ROUND = "r2x"  # the committed capture (tools/profile_round.sh + tools/summarize_round.py)


def _traffic():
    """Per-launch DRAM bytes of the roofline kernels from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", f"{PROFILE_ROUND}_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def _write_peak():
    """Measured write-only HBM stream rate (tools/bw_probe.py, profiles/<round>_bw.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"{PROFILE_ROUND}_bw.json")) as f:
            return float(json.load(f)["write_fill_GBs"])
    except (OSError, ValueError, KeyError):
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------------------------------------
# CPU reference (oracle port), lane-sharded over processes
# ------------------------------------------------------------------------------------
def _cpu_shard(args):
    """One lane shard of the config-2 step with the numpy oracle port; returns the wall
    seconds of each phase (reset, rollout, gae, scores) and the total."""
    lane0, n, T, seed, act_seed, gamma, lam = args
    import numpy as np

    from oracle import amaze_np as onp

    p = onp.Params()
    env = onp.AutoReset(n, p, "resample", lane_offset=lane0)
    rng = np.random.default_rng(act_seed + lane0)
    acts = rng.integers(0, 3, (T, n)).astype(np.uint8)
    values = rng.uniform(0, 1, (T, n))
    t0 = time.perf_counter()
    obs = env.reset(seed)
    t1 = time.perf_counter()
    view, dirs, rew, dn, fobs = onp.rollout(env, obs, acts)
    t2 = time.perf_counter()
    adv, ret = onp.gae(rew, values, dn, values[-1], gamma, lam)
    t3 = time.perf_counter()
    sc, mx, _ = onp.lane_scores(values, adv, rew, dn, np.zeros(n))
    t4 = time.perf_counter()
    return {"reset": t1 - t0, "rollout": t2 - t1, "gae": t3 - t2, "scores": t4 - t3, "total": t4 - t0}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference():
    """The unmodified reference from baseline/_ref.  runners/scoring.py imports a
    runners/buffer.py the reference never shipped: a stub module carrying the
    two fields lane_scores reads (runners/scoring.py:52,59) stands in for it."""
    import importlib
    import types
    from dataclasses import dataclass

    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    if "autocurricula.runners.buffer" not in sys.modules:
        stub = types.ModuleType("autocurricula.runners.buffer")

        @dataclass
        class PlrConfig:
            score_fn: str = "maxmc"
            maxmc_discounted: bool = False

        stub.PlrConfig = PlrConfig
        sys.modules["autocurricula.runners.buffer"] = stub
    mods = {k: importlib.import_module("autocurricula." + k)
            for k in ("amaze", "env", "rng", "agents.gae", "agents.rollout", "runners.scoring")}
    return types.SimpleNamespace(amaze=mods["amaze"], env=mods["env"], rng=mods["rng"], gae=mods["agents.gae"],
                                 rollout=mods["agents.rollout"], scoring=mods["runners.scoring"],
                                 PlrConfig=sys.modules["autocurricula.runners.buffer"].PlrConfig)


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "autocurricula"))


def _ref_shard(args):
    """One lane shard of the config-2 step through the REFERENCE's public API: DR reset
    (AutoResetWrapper(batch_lift(MazeEnv)).reset), T RESAMPLE steps, compute_gae,
    lane_scores (MaxMC).  Shards use seed + lane0 (the reference has no lane offset);
    the work per lane is statistically the same.  Returns per-phase wall seconds."""
    lane0, n, T, seed, act_seed, gamma, lam = args
    import numpy as np

    R = _import_reference()
    P = R.env.StaticParams()
    wrap = R.env.AutoResetWrapper(R.env.batch_lift(R.amaze.MazeEnv(), R.env.BatchShape(1, 1, n)), "resample")
    rng = np.random.default_rng(act_seed + lane0)
    acts = rng.integers(0, 3, (T, 1, n))
    values = rng.uniform(0, 1, (T, n))
    t0 = time.perf_counter()
    res = wrap.reset(R.rng.RngStream.from_seed(seed + lane0), P)
    t1 = time.perf_counter()
    state, extras = res.state, res.extras
    rews, dones = np.empty((T, n)), np.empty((T, n), dtype=bool)
    for t in range(T):
        r = wrap.step(None, state, acts[t], P, extras)
        rews[t], dones[t] = r.reward.reshape(-1), r.done.reshape(-1)
        state, extras = r.state, r.extras
    t2 = time.perf_counter()
    adv, _ = R.gae.compute_gae(rews, values, dones, values[-1], gamma, lam)
    t3 = time.perf_counter()
    tb = R.rollout.TrajectoryBatch({}, np.zeros((T, n), np.int64), np.zeros((T, n)), values, rews, dones,
                                   np.zeros((T, n, 1)))
    R.scoring.lane_scores(tb, adv, np.zeros(n), R.PlrConfig(score_fn="maxmc"))
    t4 = time.perf_counter()
    return {"reset": t1 - t0, "rollout": t2 - t1, "gae": t3 - t2, "scores": t4 - t3, "total": t4 - t0}


def cpu_reference_step(B, T, seed, workers, pool, phases=None, kind="port"):
    """One full step of the workload on the host: returns wall seconds.  ``phases``
    (a list) receives the per-phase seconds of the slowest shard.  kind "reference" runs
    the reference package (baseline/_ref), "port" the numpy oracle port."""
    shards = []
    per = (B + workers - 1) // workers
    for w in range(workers):
        lo = w * per
        n = min(per, B - lo)
        if n > 0:
            shards.append((lo, n, T, seed, 17, GAMMA, LAMBDA))
    fn = _ref_shard if kind == "reference" else _cpu_shard
    t0 = time.perf_counter()
    if pool is None:
        res = [fn(s) for s in shards]
    else:
        res = pool.map(fn, shards)
    wall = time.perf_counter() - t0
    if phases is not None:
        phases.append(max(res, key=lambda r: r["total"]))
    return wall


def _oracle_levels(p, n, seed):
    from oracle import amaze_np as onp

    return onp.pack_levels([onp.sample_level(seed, (0, i), p) for i in range(n)], p)


def cpu_buffer_update_seconds(n_new=4096, K=4000, it=1):
    """Oracle PLR⊥ buffer update (runners SPEC.md:360-377): n_new DR candidates into a
    full K-entry buffer, single process (the update is sequential by definition)."""
    import numpy as np

    from oracle import amaze_np as onp
    from oracle import plr_np

    p = onp.Params()
    buf = plr_np.LevelBuffer(K)
    rs = np.random.default_rng(5)
    fill = _oracle_levels(p, K, 5)
    buf.update(fill, rs.uniform(0, 1, K), rs.uniform(0, 1, K), 0)
    cand = _oracle_levels(p, n_new, 6)
    sc, mr = rs.uniform(0, 1, n_new), rs.uniform(0, 1, n_new)
    t0 = time.perf_counter()
    buf.update(cand, sc, mr, it)
    return time.perf_counter() - t0


METRIC = "AMaze env steps/sec (DR reset + 256-step RESAMPLE rollout + GAE/MaxMC)"


def workload_config(args, world):
    """The `config` dict both arms print (identical keys and values)."""
    return {"workload": "configs[1]: AMaze 13x13 DR, 4096 envs x 256 steps, RESAMPLE auto-reset, GAE+MaxMC",
            "lanes_per_gpu": args.lanes, "T": args.T, "gamma": GAMMA, "lambda": LAMBDA,
            "l2": "flushed (256 MB write) before every timed step (GPU arm)",
            "parallelism": f"lane-sharded x{world}"}


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------
# clocks sampler
# ------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML while ``active`` is set."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device):
        self.samples = []
        self.active = False
        self.stop_flag = False
        self.thread = None
        self.handle = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(device)
            try:
                bus = f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0"
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(torch.device(device).index or 0)
            self.nvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report unknown clocks
            self.err = repr(e)

    def start(self):
        if self.handle is None:
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        n = self.nvml
        while not self.stop_flag:
            if self.active:
                try:
                    sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
                    try:
                        rs = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                    except AttributeError:
                        rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
            time.sleep(0.002)

    def stop(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------
# GPU workload
# ------------------------------------------------------------------------------------
class Workload:
    """Config 2 on one device: DR reset + fused T-step rollout + GAE/MaxMC."""

    def __init__(self, B, T, seed, lane_offset, device):
        import torch

        import paper_2311_12716_b200 as amz

        self.amz, self.torch = amz, torch
        self.B, self.T, self.seed, self.dev = B, T, seed, device
        self.p = amz.StaticParams()
        self.benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B), device=device,
                                       lane_offset=lane_offset)
        self.env = amz.AutoResetWrapper(self.benv, amz.RESAMPLE)
        self.lane_offset = lane_offset
        g = torch.Generator(device=device)
        g.manual_seed(1234 + lane_offset)
        self.actions = torch.randint(0, 3, (T, B), generator=g, device=device, dtype=torch.uint8)
        self.values = torch.rand((T, B), generator=g, device=device, dtype=torch.float64)
        self.last = torch.rand((B,), generator=g, device=device, dtype=torch.float64)
        v = self.p.agent_view_size
        self.out = {"view": torch.empty((T, B, v, v), dtype=torch.uint8, device=device),
                    "dir": torch.empty((T, B), dtype=torch.uint8, device=device),
                    "rewards": torch.empty((T, B), dtype=torch.float64, device=device),
                    "dones": torch.empty((T, B), dtype=torch.bool, device=device),
                    "final_view": torch.empty((B, v, v), dtype=torch.uint8, device=device),
                    "final_dir": torch.empty((B,), dtype=torch.uint8, device=device)}
        self.root = amz.RngStream.from_seed(seed)
        # GAE/score results reused every step; scores and max returns share one [2, B]
        # tensor so the end-to-end result read is a single device->host copy
        self.res = torch.empty((2, B), dtype=torch.float64, device=device)
        self.gout = {"advantages": torch.empty((T, B), dtype=torch.float64, device=device),
                     "returns": torch.empty((T, B), dtype=torch.float64, device=device),
                     "scores": self.res[0], "max_returns": self.res[1]}
        # our kernels per step: k_env_reset_dr, k_dyn, k_render, k_gae_score4
        self.launches_per_step = 4
        self.ev_roll = None

    def step(self, it, actions=None, values=None, last=None, timing=None):
        amz, torch = self.amz, self.torch
        rng = self.root.fold_in(it)
        # DR level generation + reset in one launch; it also prepares the timeout levels of
        # the rollout's first auto-resets (keys rng_wrap ++ [tep - 1, lane])
        res = self.env.reset(rng, self.p)
        if timing is not None:
            timing[0].record()
        traj, cur = amz.rollout_actions(self.env, res, self.actions if actions is None else actions, self.p,
                                        out=self.out)
        if timing is not None:
            timing[1].record()
        o = amz.gae_and_scores(traj.rewards, self.values if values is None else values, traj.dones,
                               self.last if last is None else last, GAMMA, LAMBDA, out=self.gout)
        if timing is not None:
            timing[2].record()
        return o


def _graph(dev, B, T, seed, lane_offset, vdt, host_io, torch):
    """The public API's captured DR iteration (paper_2311_12716_b200.graph)."""
    import paper_2311_12716_b200 as amz
    from paper_2311_12716_b200.graph import DRIterationGraph

    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B), device=dev, lane_offset=lane_offset)
    gr = DRIterationGraph(benv, amz.RngStream.from_seed(seed), T, amz.StaticParams(), GAMMA, LAMBDA,
                          value_dtype=vdt, host_io=host_io, overlap=True)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + lane_offset)
    acts = torch.randint(0, 3, (T, B), generator=g, device=dev, dtype=torch.uint8)
    vals = torch.rand((T, B), generator=g, device=dev, dtype=torch.float64).to(vdt)
    last = torch.rand((B,), generator=g, device=dev, dtype=torch.float64).to(vdt)
    if host_io:
        gr.host_inputs["actions"].copy_(acts.cpu())
        gr.host_inputs["values"].copy_(vals.cpu())
        gr.host_inputs["last"].copy_(last.cpu())
    else:
        gr.inputs[0]["actions"].copy_(acts)
        gr.inputs[0]["values"].copy_(vals)
        gr.inputs[0]["last"].copy_(last)
    return gr.capture()


def run_ours(args, rank, world, local_rank):
    import torch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, T = args.lanes, args.T
    # 256 MB (> 126 MB L2) written as int64 words: the 8-byte fill runs near HBM write speed
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.int64, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_ranks(*vals):
        t = torch.tensor(list(vals), dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    clocks = ClockSampler(dev)
    clocks.start()

    # ---- headline: one CUDA-graph replay per step (DR reset -> rollout -> GAE/MaxMC),
    # inputs resident in HBM, L2 flushed before every step, events around each replay ----
    gr = _graph(dev, B, T, args.seed, rank * B, torch.float64, False, torch)
    for i in range(args.warmup):
        gr.step()
    torch.cuda.synchronize()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks.active = True
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record()
        gr.step()
        ev[i][1].record()
    torch.cuda.synchronize()
    clocks.active = False
    barrier()
    (total_ms,) = max_ranks(sum(a.elapsed_time(b) for a, b in ev))
    del gr

    # ---- the same step through the eager per-call API, kernel by kernel: the GPU is
    # held by a spin before each step so the host has enqueued the whole step before it
    # starts (kernel times without host gaps) ----
    wl = Workload(B, T, args.seed, rank * B, dev)
    for i in range(args.warmup):
        wl.step(i)
    torch.cuda.synchronize()
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    host0 = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        torch.cuda._sleep(400_000)  # ~0.2 ms of GPU spin: the host runs ahead
        eev[i][0].record()
        wl.step(args.warmup + i, timing=kev[i])
        eev[i][1].record()
    eager_host_ms = (time.perf_counter() - host0) * 1e3 / args.steps
    torch.cuda.synchronize()
    eager_ms = statistics.mean(a.elapsed_time(b) for a, b in eev)
    roll_ms = [k[0].elapsed_time(k[1]) for k in kev]
    gae_ms = [k[1].elapsed_time(k[2]) for k in kev]
    # eager back to back (no spin): what a plain Python loop over the per-call API gets
    torch.cuda.synchronize()
    b2b0, b2b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b2b0.record()
    for i in range(args.steps):
        wl.step(1000 + i)
    b2b1.record()
    torch.cuda.synchronize()
    eager_b2b_ms = b2b0.elapsed_time(b2b1) / args.steps
    del wl

    # ---- e2e through the public API: pinned host inputs in, scores | max returns out,
    # one graph replay per step, the next step's H2D overlapped with this step's kernels;
    # one timed region over all K steps including every copy, L2 flush and result read ----
    def e2e(vdt, flush_l2):
        g2 = _graph(dev, B, T, args.seed, rank * B, vdt, True, torch)
        # On these hosts PCIe reads of pinned pages the CPU has just written run 2-4x slow
        # for ~0.5-2 s (tools/e2e_recover.py); the synthetic feed is written once, so let
        # it settle, then warm up past the graph's one-off H2D path calibration
        # (copy_mode "auto", after calibrate_after steps)
        time.sleep(2.0)
        for _ in range(max(args.warmup, g2.calibrate_after + 64)):
            g2.step()
        torch.cuda.synchronize()
        barrier()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.active = True
        p0.record()
        h0 = time.perf_counter()
        for i in range(args.steps):
            if flush_l2:
                flush.fill_(i & 0xFF)
            g2.step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        p1.record()
        torch.cuda.synchronize()
        clocks.active = False
        es = torch.empty((), dtype=vdt).element_size()
        h2d = T * B * (1 + es) + B * es
        ms = p0.elapsed_time(p1)
        how = "copy-engine memcpy" if g2.copy_engine else f"copy kernel ({g2.copy_ctas} CTAs)"
        cal = g2.calibration_ms or {}
        how += " (calibration us/step: kernel %s, engine %s)" % tuple(
            round(cal[k] * 1e3, 1) if k in cal else None for k in (False, True))
        del g2
        return ms, host_ms, h2d, how

    e32_ms, host32_ms, h2d32, how32 = e2e(torch.float32, False)
    e32f_ms, host32f_ms, _, how32f = e2e(torch.float32, True)
    e64_ms, host64_ms, h2d64, how64 = e2e(torch.float64, False)
    e32_ms, e32f_ms, e64_ms = max_ranks(e32_ms, e32f_ms, e64_ms)
    peaks, src = _peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    extra = {}
    if not args.no_extra:
        its = max(3, min(args.steps, 10))
        # configs[4]: 32768 GLOBAL lanes of PLR|| split over the ranks, NCCL all-gather (strong scaling)
        extra["parallel_plr"] = measure_plr_parallel(dev, 16384, T, False, its, flush, world, "plr_parallel",
                                                     "configs[4] Parallel PLR multi-device: 32768 global lanes "
                                                     "(16384 new | 16384 replay), K=4000")
        extra["parallel_plr"]["scaling"] = "strong"
        if world == 1:
            extra["plr_perp"] = measure_plr_perp(dev, 4096, T, False, 2 * its, flush, "plr_perp",
                                                 "configs[2] PLR-perp: 4096 lanes, K=4000, MaxMC, rank replay")
            extra["accel_perp"] = measure_plr_perp(dev, 4096, T, True, 2 * its, flush, "accel_perp",
                                                   "configs[3] ACCEL: PLR-perp + 4 mutants x 20 edits per replay")
            extra["plr_parallel"] = measure_plr_parallel(dev, 2048, T, False, its, flush, 1, "plr_parallel",
                                                         "PLR|| (paper variant of configs[2]): 2048 new | 2048 replay")
            extra["accel_parallel"] = measure_plr_parallel(dev, 2048, T, True, its, flush, 1, "accel_parallel",
                                                           "ACCEL|| (paper variant of configs[3]): 2048 x 3 lanes")
            extra["large_batch"] = measure_large_batch(dev, 65536, T, 3, flush, peak)
            extra["level_metrics"] = measure_level_metrics(dev, 65536, 5, flush)
            extra["policy_rollout"] = measure_policy_rollout(dev, 4096, 64)
    clocks.stop()
    csum = clocks.summary()

    if rank != 0:
        return None
    units = B * T * world
    roll = statistics.mean(roll_ms)
    gae = statistics.mean(gae_ms)
    roll_gbs = ENV_BYTES_PER_STEP * B * T / (roll * 1e-3) / 1e9
    gae_gbs = GAE_BYTES_PER_ELEM * B * T / (gae * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    line = {
        "metric": METRIC,
        "value": units / (total_ms * 1e-3 / args.steps),
        "unit": "env-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8/int32 env, f64 GAE",
        "data": "synthetic: DR levels from (seed, lane) keys, uniform random actions and values resident in HBM",
        "config": workload_config(args, world),
        "mode": "one CUDA-graph replay per step (paper_2311_12716_b200.graph.DRIterationGraph: k_env_reset_dr -> "
                "k_dyn -> k_render -> k_gae_score -> k_iter_advance), device-timed with CUDA events per step",
        "eager": {"value": units / (eager_b2b_ms * 1e-3), "ms_per_step": eager_b2b_ms,
                  "kernel_ms_per_step": eager_ms, "host_enqueue_ms_per_step": eager_host_ms,
                  "mode": "per-call API (VectorBatchEnv/AutoResetWrapper.reset, rollout_actions, gae_and_scores) back "
                          "to back; kernel_ms_per_step with the host run ahead (GPU spin before each step)"},
        "e2e": {"value": units / (e32_ms * 1e-3 / args.steps), "unit": "env-steps/s",
                "h2d_bytes_per_step": h2d32, "d2h_bytes_per_step": 2 * B * 8,
                "ms_per_step": e32_ms / args.steps, "host_enqueue_ms_per_step": host32_ms,
                "inputs": "actions u8 [T, B] + values f32 [T, B] + last values f32 [B] (the policy's output dtype, "
                          "widened to f64 in-kernel like the reference's value.double(), agents/ppo.py:96)",
                "mode": "DRIterationGraph(host_io=True): one graph replay per step, two input slots; the H2D of "
                        "the NEXT step's pinned inputs runs on a copy stream concurrent with this step's graph "
                        "(event-ordered: it waits only for the graph that last read its slot), by the path the "
                        "graph's capture-time calibration found faster on this box (copy-engine memcpy or the "
                        "amz_copy_h2d kernel); the graph ends with a kernel storing scores | max returns into "
                        "pinned host memory; one timed region over all K steps",
                "h2d_path": how32,
                "warmup": "2 s after the host writes the synthetic feed (PCIe reads of pinned pages the CPU has just "
                          "written run 2-4x slower for ~0.5-2 s on these hosts: tools/e2e_recover.py; a feed rewritten "
                          "every step would see ~250-400 us/step), then max(W, 264) steps past the one-off copy-path "
                          "calibration",
                "l2": "not flushed between e2e steps: every step's inputs are copied fresh from pinned host memory and "
                      "its 54 MB of outputs overwrite the previous step's (with_l2_flush: a 256 MB write before every "
                      "step, inside the timed region)",
                "with_l2_flush": {"value": units / (e32f_ms * 1e-3 / args.steps), "ms_per_step": e32f_ms / args.steps,
                                  "host_enqueue_ms_per_step": host32f_ms, "h2d_path": how32f},
                "values_f64": {"value": units / (e64_ms * 1e-3 / args.steps), "ms_per_step": e64_ms / args.steps,
                               "h2d_bytes_per_step": h2d64, "host_enqueue_ms_per_step": host64_ms,
                               "h2d_path": how64}},
        "gpu_launches": 5 * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_env_rollout", "achieved": roll_gbs, "peak": peak, "unit": "GB/s",
                     "frac": roll_gbs / peak,
                     "traffic": _traffic().get("k_env_rollout", {}).get("dram_bytes"),
                     "traffic_source": f"profiles/{PROFILE_ROUND}_traffic.json (ncu --set full, per launch)",
                     "peak_source": src,
                     "algorithmic_bytes": f"{ENV_BYTES_PER_STEP} B/env-step x {B * T} env-steps per launch",
                     "kernel_ms": roll,
                     "write_stream_GBs": _write_peak(),
                     "frac_of_write_stream": (roll_gbs / _write_peak()) if _write_peak() else None,
                     "note": "k_env_rollout = k_dyn + k_render (the timeout levels of the first auto-resets "
                             "come prepared from the fused reset launch, so no k_spec_levels); at 4096 lanes the "
                             "per-lane 256-step dynamics chain (latency) bounds it, not HBM; the HBM point is "
                             "large_batch (65536 lanes)"},
        "kernels": {"k_env_rollout_ms": roll, "k_gae_score_ms": gae, "k_gae_score_GBs": gae_gbs,
                    "k_gae_score_frac": gae_gbs / peak,
                    "levels_scored_per_s": B * world / (gae * 1e-3)},
        "clocks": {k: csum[k] for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")},
    }
    line.update(extra)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = measure_cpu_baseline(args)
    return line


def _timed(fn, iters, flush, torch):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for i in range(iters):
        flush.fill_(i & 0xFF)
        evs[i][0].record()
        fn(i)
        evs[i][1].record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


# paper Table 4: (gamma, lambda, staleness rho, replay rate p)
HP = {"plr_perp": (0.999, 0.98, 0.3, 0.5), "plr_parallel": (0.999, 0.95, 0.5, 0.5),
      "accel_perp": (0.999, 0.98, 0.5, 0.8), "accel_parallel": (0.999, 0.98, 0.5, 0.8)}


def _plr_cfg(name):
    from paper_2311_12716_b200.buffer import PlrConfig

    g, lam, rho, p = HP[name]
    return PlrConfig(buffer_size=4000, score_fn="maxmc", temperature=0.3, staleness_coef=rho, replay_rate=p), g, lam


def _policy_inputs(dev, T, L, seed, torch):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    acts = torch.randint(0, 3, (T, L), generator=g, device=dev, dtype=torch.uint8)
    vals = torch.rand((T, L), generator=g, device=dev, dtype=torch.float64) * 0.2
    last = torch.rand((L,), generator=g, device=dev, dtype=torch.float64) * 0.2
    return acts, vals, last


def _max_over_ranks(ms, dev, world, torch):
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def measure_plr_parallel(dev, n, T, accel, iters, flush, world, name, config_label):
    """PLR|| / ACCEL|| iteration, env side: compose lanes (DR + rank-
    prioritised replay [+ 20-edit mutants]), HOME rollout, GAE + MaxMC, NCCL candidate
    all-gather (N > 1), replicated buffer update.  n new lanes, L = 2n / 3n GLOBAL lanes
    split over the ranks; K = 4000.  Iteration time = max over ranks."""
    import torch

    import paper_2311_12716_b200 as amz
    from paper_2311_12716_b200.buffer import AccelConfig
    from paper_2311_12716_b200.plr import ParallelPLR

    cfg, gamma, lam = _plr_cfg(name)
    plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(7), AccelConfig(20, 4) if accel else None,
                      gamma=gamma, lam=lam, device=dev, check_every=0)
    acts, vals, last = _policy_inputs(dev, T, plr.hi - plr.lo, 99 + plr.rank, torch)
    for it in range(3):  # fills the 4000-level buffer (the first iteration inserts its new levels)
        plr.iteration(it, acts, vals, last)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = _timed(lambda i: plr.iteration(3 + i, acts, vals, last), iters, flush, torch)
    it_ms = _max_over_ranks(statistics.mean(ms), dev, world, torch)
    plr.check_replicas()  # the drift check once per measurement (digest on device + all-reduce)
    out = {"config": config_label, "lanes_global": plr.L, "lanes_per_rank": plr.hi - plr.lo, "T": T,
           "buffer_size": 4000, "gamma": gamma, "lambda": lam, "staleness_coef": cfg.staleness_coef,
           "replay_rate": cfg.replay_rate, "iteration_ms": it_ms,
           "levels_scored_per_s": plr.L / (it_ms * 1e-3), "env_steps_per_s": plr.L * T / (it_ms * 1e-3),
           "collective": (("NCCL all_gather_into_tensor of 48-byte candidate records"
                           if torch.distributed.get_backend() == "nccl" else
                           f"{torch.distributed.get_backend()} all_gather of 48-byte candidate records (host-staged)")
                          if world > 1 else "none (1 rank)")}
    if world == 1 and n <= 4096:
        # the two buffer kernels on their own: an update with 4096 distinct new levels
        # (scores U(0,1): most evict -- the worst case) and one with 4000 replays of
        # buffered levels (in-place updates); the replay draw
        new_lv = amz.sample_levels(amz.RngStream(99, (0,)), 4096, amz.StaticParams(), device=dev)
        sc = torch.rand(4096, device=dev, dtype=torch.float64)
        sc2 = torch.rand(4000, device=dev, dtype=torch.float64)
        t_upd = _timed(lambda i: plr.buffer.update(new_lv, sc, sc, 1000 + i), iters, flush, torch)
        old_lv = plr.buffer.export()["levels"][:4000]  # exported after t_upd: every level is buffered
        t_rep = _timed(lambda i: plr.buffer.update(old_lv, sc2, sc2, 1000 + i), iters, flush, torch)
        t_smp = _timed(lambda i: plr.buffer.sample(amz.RngStream(5, (i,)), n, 2000 + i), iters, flush, torch)
        out.update({"buffer_update_us_4096_new_levels": 1e3 * statistics.mean(t_upd),
                    "buffer_update_us_4000_replays": 1e3 * statistics.mean(t_rep),
                    "buffer_sample_us": 1e3 * statistics.mean(t_smp)})
    return out


def measure_plr_perp(dev, n, T, accel, iters, flush, name, config_label):
    """PLR-perp / ACCEL-perp iteration: decision; NEW = n fresh DR
    levels, HOME rollout, score, update; REPLAY = n draws, rollout, in-place re-score
    [+ q=4 mutants, 20 edits, rolled out and inserted].  K = 4000, one GPU."""
    import torch

    import paper_2311_12716_b200 as amz
    from paper_2311_12716_b200.buffer import AccelConfig
    from paper_2311_12716_b200.plr import SequentialPLR

    cfg, gamma, lam = _plr_cfg(name)
    plr = SequentialPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(11), AccelConfig(20, 4) if accel else None,
                        gamma=gamma, lam=lam, device=dev)
    acts, vals, last = _policy_inputs(dev, T, n, 123, torch)
    it = 0
    while plr.buffer.size() < 4000 and it < 8:  # NEW iterations fill the buffer
        plr.iteration(it, acts, vals, last)
        it += 1
    torch.cuda.synchronize()
    branch = {"new": [], "replay": []}
    evs = []
    for i in range(iters):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = plr.iteration(it + i, acts, vals, last)
        b.record()
        evs.append((r.branch, a, b))
    torch.cuda.synchronize()
    for br, a, b in evs:
        branch[br].append(a.elapsed_time(b))
    allms = [x for v in branch.values() for x in v]
    it_ms = statistics.mean(allms)
    out = {"config": config_label, "lanes": n, "T": T, "buffer_size": 4000, "gamma": gamma, "lambda": lam,
           "staleness_coef": cfg.staleness_coef, "replay_rate": cfg.replay_rate, "iterations": len(allms),
           "iteration_ms": it_ms, "levels_scored_per_s": n / (it_ms * 1e-3), "env_steps_per_s": n * T / (it_ms * 1e-3)}
    for br, v in branch.items():
        if v:
            out[f"{br}_iterations"] = len(v)
            out[f"{br}_iteration_ms"] = statistics.mean(v)
    return out


def measure_large_batch(dev, B, T, iters, flush, peak):
    """Rollout + GAE at a batch that is HBM-sized (trajectory >> L2): the roofline point."""
    import torch

    wl = Workload(B, T, 3, 0, dev)
    for i in range(2):
        wl.step(i)
    torch.cuda.synchronize()
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(iters)]
    for i in range(iters):
        flush.fill_(i & 0xFF)
        torch.cuda._sleep(400_000)  # the host runs ahead: kernel times without host gaps
        wl.step(10 + i, timing=kev[i])
    torch.cuda.synchronize()
    roll = statistics.mean(k[0].elapsed_time(k[1]) for k in kev)
    gae = statistics.mean(k[1].elapsed_time(k[2]) for k in kev)
    rg = ENV_BYTES_PER_STEP * B * T / (roll * 1e-3) / 1e9
    gg = GAE_BYTES_PER_ELEM * B * T / (gae * 1e-3) / 1e9
    tr = _traffic().get("large_batch_rollout", {})
    wpk = _write_peak()
    out = {"lanes": B, "T": T, "rollout_ms": roll, "rollout_GBs": rg, "rollout_frac": rg / peak,
           "rollout_traffic": tr.get("dram_bytes"), "traffic_source": f"profiles/{PROFILE_ROUND}_traffic.json",
           "rollout_frac_of_write_stream": (rg / wpk) if wpk else None,
           "write_stream_note": "the rollout's bytes are 97% writes (view, dir, reward, done out; 1 B of action in); "
                                "a write-only stream (torch fill_) reaches the write_stream_GBs figure on this B200 "
                                f"(profiles/{PROFILE_ROUND}_bw.json), the copy peak above counts reads and writes",
           "write_stream_GBs": wpk,
           "rollout_env_steps_per_s": B * T / (roll * 1e-3), "gae_score_ms": gae, "gae_score_GBs": gg,
           "gae_score_frac": gg / peak, "levels_scored_per_s": B / (gae * 1e-3)}
    del wl
    torch.cuda.empty_cache()
    # GAE + scores alone at 2^17 lanes (the HBM fraction at >= 2^17 lanes),
    # synthetic rewards / dones / values of the configs' shape, L2 flushed before each
    import paper_2311_12716_b200 as amz

    B2 = 1 << 17
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    r = torch.rand((T, B2), generator=g, device=dev, dtype=torch.float64)
    d = torch.rand((T, B2), generator=g, device=dev, dtype=torch.float64) < 1.0 / 250
    r = torch.where(d, r, torch.zeros_like(r))
    v = torch.rand((T, B2), generator=g, device=dev, dtype=torch.float64)
    last = torch.rand((B2,), generator=g, device=dev, dtype=torch.float64)
    gout = {"advantages": torch.empty_like(v), "returns": torch.empty_like(v),
            "scores": torch.empty(B2, dtype=torch.float64, device=dev),
            "max_returns": torch.empty(B2, dtype=torch.float64, device=dev)}
    amz.gae_and_scores(r, v, d, last, GAMMA, LAMBDA, out=gout)
    ms = _timed(lambda i: amz.gae_and_scores(r, v, d, last, GAMMA, LAMBDA, out=gout), iters + 2, flush, torch)
    g2 = statistics.mean(ms)
    gb2 = GAE_BYTES_PER_ELEM * B2 * T / (g2 * 1e-3) / 1e9
    out["gae_score_131072"] = {"lanes": B2, "ms": g2, "GBs": gb2, "frac": gb2 / peak,
                               "levels_scored_per_s": B2 / (g2 * 1e-3)}
    del r, d, v, last, gout
    torch.cuda.empty_cache()
    return out


def measure_level_metrics(dev, n, iters, flush):
    """Curriculum metrics: BFS shortest path + wall stats per level."""
    import torch

    import paper_2311_12716_b200 as amz

    P = amz.StaticParams()
    lv = amz.sample_levels(amz.RngStream.from_seed(5), n, P, device=dev)
    amz.level_metrics(lv, P)
    torch.cuda.synchronize()
    ms = _timed(lambda i: amz.level_metrics(lv, P), iters, flush, torch)
    t = statistics.mean(ms)
    return {"levels": n, "ms": t, "levels_per_s": n / (t * 1e-3)}


def measure_policy_rollout(dev, B, T):
    """rollout() with a torch student net of the reference's architecture
    in the loop (fused policy head + device step), eager vs one CUDA-graph replay per step."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from policy_rollout_bench import StudentNet

    import paper_2311_12716_b200 as amz

    torch.manual_seed(0)
    actor = amz.TorchPolicyActor(StudentNet().to(dev).eval())
    P = amz.StaticParams()
    out = {"lanes": B, "T": T, "policy": "tile/dir embed -> Linear 128 -> GRUCell 256 -> heads, fp32, random init"}
    for name in ("eager", "graph"):
        env = amz.AutoResetWrapper(amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, B), device=dev), amz.RESAMPLE)
        start = env.reset(amz.RngStream.from_seed(1), P)
        gr = amz.GraphRollout(actor, env, T) if name == "graph" else None
        run = (lambda r, s: gr(r, s, copy=False)) if gr else (lambda r, s: amz.rollout(r, actor, env, s, T, P))
        _, cur = run(amz.RngStream.from_seed(2), start)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(2):
            _, cur = run(amz.RngStream.from_seed(3 + i), cur)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 2
        out[f"{name}_ms"] = ms
        out[f"{name}_lane_steps_per_s"] = B * T / (ms * 1e-3)
    return out


def measure_cpu_baseline(args, steps=1):
    """One config-2 step on the host cores, bounded (~10-30 s): the reference package
    when baseline/_ref is present, else the oracle port."""
    import multiprocessing as mp

    cores = _cores()
    B, T = args.lanes, args.T
    kind = "reference" if reference_available() else "port"
    if kind == "reference":
        _import_reference()  # once in the parent: the forked workers inherit the modules
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        secs = [cpu_reference_step(B, T, args.seed, cores, pool, kind=kind) for _ in range(steps)]
    s = statistics.mean(secs)
    what = ("the reference package (baseline/_ref, unmodified) through its public API" if kind == "reference"
            else "the numpy oracle port of the reference")
    return {"value": B * T / s, "unit": "env-steps/s", "cores": cores, "kind": kind,
            "sample": f"one full step ({B} lanes x {T} steps DR reset + RESAMPLE rollout + GAE/MaxMC) with {what}, "
                      f"lanes sharded over {cores} processes; host: {_cpu_model()}"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import multiprocessing as mp

    cores = _cores()
    B, T = args.lanes, args.T
    kind = "reference" if reference_available() else "port"
    if kind == "reference":
        _import_reference()  # once in the parent: the forked workers inherit the modules
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_reference_step(B, T, args.seed, cores, pool, kind=kind)
        phases = []
        secs = [cpu_reference_step(B, T, args.seed, cores, pool, phases, kind=kind) for _ in range(args.steps)]
    s = statistics.mean(secs)
    val = B * T / s
    # the phases separately (slowest shard, mean over the timed steps), one
    # single-process step (no sharding), and the oracle buffer update (sequential; the
    # reference never shipped its buffer)
    phase_ms = {k: 1e3 * statistics.mean(ph[k] for ph in phases) for k in ("reset", "rollout", "gae", "scores")}
    one = cpu_reference_step(B, T, args.seed, 1, None, kind=kind)
    buf_s = cpu_buffer_update_seconds(4096, 4000)
    what = ("the unmodified reference package (baseline/_ref) through its public API (AutoResetWrapper/batch_lift, "
            "compute_gae, lane_scores)" if kind == "reference" else
            "the numpy oracle port of the reference (baseline/_ref absent)")
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": val, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64 env, f64 GAE", "data": "synthetic (same workload shape, numpy random actions/values)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": val, "unit": "env-steps/s", "cores": cores, "kind": kind,
                         "sample": f"one full config-2 step per timed step with {what}, lanes sharded over {cores} "
                                   f"processes (shard seeds seed+lane0); host: {_cpu_model()}"},
        "e2e": {"value": val, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_ms_per_step": phase_ms,
        "single_process": {"env_steps_per_s": B * T / one, "ms_per_step": one * 1e3, "cores": 1},
        "buffer_update_ms_4096_new_levels": buf_s * 1e3,
        "buffer_update_impl": "oracle/plr_np.py (SPEC.md:373-377 transcription; the reference has no buffer)",
    }


def _relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec this script under torch.distributed.run with
    N ranks on this node (127.0.0.1 rendezvous).  NCCL's INIT lines go to stderr so the
    communicator size (comm nranks) is on record without touching the JSON line."""
    import socket

    if not args.launcher_check:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus and not os.environ.get("AMZ_BENCH_ONE_DEVICE"):
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def launcher_check(rank, world):
    """--launcher-check: the rank world only (gloo, no GPU work) -- lets a CPU test see
    that --gpus N really starts N ranks."""
    import torch

    torch.distributed.init_process_group("gloo")
    t = torch.ones(1)
    torch.distributed.all_reduce(t)
    torch.distributed.destroy_process_group()
    if rank == 0:
        return {"launcher_check": True, "world": world, "ranks_seen": int(t.item())}
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--lanes", type=int, default=4096)
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the PLR/ACCEL and large-batch measurements")
    ap.add_argument("--launcher-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launcher_check:
        line = launcher_check(rank, world)
    elif args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        import torch

        # test hooks (the multi-rank code path on a 1-GPU box): AMZ_BENCH_ONE_DEVICE=1 puts
        # every rank on cuda:0, AMZ_BENCH_BACKEND=gloo replaces NCCL (which refuses two ranks
        # on one device); timings from such a run are not scaling numbers
        dev_index = 0 if os.environ.get("AMZ_BENCH_ONE_DEVICE") else local_rank
        backend = os.environ.get("AMZ_BENCH_BACKEND", "nccl")
        if world > 1:
            torch.cuda.set_device(dev_index)
            if backend == "nccl":
                torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
            else:
                torch.distributed.init_process_group(backend)
        line = run_ours(args, rank, world, dev_index)
        if world > 1:
            torch.distributed.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
