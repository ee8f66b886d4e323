"""Benchmark of the AMaze + PLR hot path (BASELINE.json configs[1] by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the hot path over one batch of synthetic input (config 2,
"AMaze 13x13 DR with PPO rollout batch 4096 envs x 256 steps and GAE on 1xB200"):
  1.+2. DR level generation for every lane (keys (seed, (0, lane))) fused with the reset
     of every lane (VectorBatchEnv.reset),
  3. 256 fused env steps with RESAMPLE auto-reset driven by a uint8 [T, B] action
     stream resident in HBM (the policy is out of scope; its values are a resident
     float64 [T, B] tensor),
  4. GAE (gamma 0.995, lambda 0.95) + MaxMC regret scores + running max returns.
metric = env-steps/s = lanes * T / step time (whole job, all ranks).

Under torchrun each rank runs its own lane shard (global lane ids rank*B + i, so the
keys equal a 1-GPU run over N*B lanes): weak scaling, no data-path collective.

--impl reference times the oracle port of the reference (oracle/amaze_np.py, numpy,
lane-sharded over all host cores; the reference itself is pure Python and cannot be
installed on the GPU box) on the same workload, rank 0 only.
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
ENV_BYTES_PER_STEP = 36  # action u8 + view 25 u8 + dir u8 + reward f64 + done u8
GAE_BYTES_PER_ELEM = 33  # r f64 + V f64 + done u8 in, A f64 + R f64 out


def _traffic():
    """Per-launch DRAM bytes of the roofline kernels from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1m_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


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


def cpu_reference_step(B, T, seed, workers, pool, phases=None):
    """One full step of the workload on the host: returns wall seconds.  ``phases``
    (a list) receives the per-phase seconds of the slowest shard."""
    shards = []
    per = (B + workers - 1) // workers
    for w in range(workers):
        lo = w * per
        n = min(per, B - lo)
        if n > 0:
            shards.append((lo, n, T, seed, 17, 0.995, 0.95))
    t0 = time.perf_counter()
    if pool is None:
        res = [_cpu_shard(s) for s in shards]
    else:
        res = pool.map(_cpu_shard, shards)
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
                               self.last if last is None else last, 0.995, 0.95, out=self.gout)
        if timing is not None:
            timing[2].record()
        return o


def run_ours(args, rank, world, local_rank):
    import torch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, T = args.lanes, args.T
    wl = Workload(B, T, args.seed, rank * B, dev)
    # 256 MB (> 126 MB L2) written as int64 words: the 8-byte fill runs near HBM write speed
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.int64, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for i in range(args.warmup):
        wl.step(i)
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    clocks.active = True
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record()
        wl.step(args.warmup + i, timing=kev[i])
        ev[i][1].record()
    torch.cuda.synchronize()
    barrier()
    clocks.active = False
    step_ms = [a.elapsed_time(b) for a, b in ev]
    roll_ms = [k[0].elapsed_time(k[1]) for k in kev]
    gae_ms = [k[1].elapsed_time(k[2]) for k in kev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t.item())

    # ---- e2e through the public API: pinned host inputs in, scores out ----
    from paper_2311_12716_b200 import pinned_empty as amz_pinned_empty
    h_act = amz_pinned_empty((T, B), torch.uint8)
    h_act.copy_(wl.actions.cpu())
    h_val = amz_pinned_empty((T, B), torch.float64)
    h_val.copy_(wl.values.cpu())
    h_last = amz_pinned_empty((B,), torch.float64)
    h_last.copy_(wl.last.cpu())
    h_res = amz_pinned_empty((2, B), torch.float64)
    d_act = torch.empty_like(wl.actions)
    d_val = torch.empty_like(wl.values)
    d_last = torch.empty_like(wl.last)
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        e2e_ev[i][0].record()
        d_act.copy_(h_act, non_blocking=True)
        d_val.copy_(h_val, non_blocking=True)
        d_last.copy_(h_last, non_blocking=True)
        wl.step(10_000 + i, actions=d_act, values=d_val, last=d_last)
        h_res.copy_(wl.res, non_blocking=True)  # scores | max returns
        e2e_ev[i][1].record()
    torch.cuda.synchronize()
    seq_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)

    # pipelined: step i+1's host->device copies run on a copy stream (double-buffered
    # device inputs) while step i computes; one timed region around all K steps, every
    # step's copies, L2 flush, step and result read inside it
    # two copy streams: the box's H2D path reaches ~45 GB/s only with two DMA engines busy
    css = [torch.cuda.Stream(device=dev) for _ in range(2)]
    main = torch.cuda.current_stream(dev)

    def pipelined(vdt, step0):
        """One timed region over K pipelined steps; values (and last values) staged as vdt."""
        # one pinned staging buffer per step's inputs (values | last values | actions), two
        # copies per step (one per copy stream) instead of one per tensor
        es = torch.empty((), dtype=vdt).element_size()
        nv, nl, na = T * B * es, B * es, T * B
        h_in = amz_pinned_empty(nv + nl + na, torch.uint8)
        h_in[:nv].view(vdt).copy_(wl.values.to(vdt).cpu().reshape(-1))
        h_in[nv:nv + nl].view(vdt).copy_(wl.last.to(vdt).cpu())
        h_in[nv + nl:].copy_(h_act.reshape(-1))
        d_in = [torch.empty_like(h_in, device=dev) for _ in range(2)]
        bufs = [(d[nv + nl:].view(T, B), d[:nv].view(vdt).view(T, B), d[nv:nv + nl].view(vdt)) for d in d_in]
        outs = [amz_pinned_empty((2, B), torch.float64) for _ in range(2)]
        copied = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        half = (h_in.numel() // 2) & ~15

        def h2d(k):
            for c, cs in enumerate(css):
                cs.wait_event(freed[k])
                with torch.cuda.stream(cs):
                    if c == 0:
                        d_in[k][:half].copy_(h_in[:half], non_blocking=True)
                    else:
                        d_in[k][half:].copy_(h_in[half:], non_blocking=True)
                    copied[k][c].record(cs)

        torch.cuda.synchronize()
        barrier()
        for k in range(2):
            freed[k].record(main)
        clocks.active = True
        p0.record(main)
        host0 = time.perf_counter()
        for cs in css:
            cs.wait_event(p0)
        h2d(0)
        for i in range(args.steps):
            k = i & 1
            if i + 1 < args.steps:
                h2d(k ^ 1)
            main.wait_event(copied[k][0])
            main.wait_event(copied[k][1])
            flush.fill_(i & 0xFF)
            a, v, l_ = bufs[k]
            wl.step(step0 + i, actions=a, values=v, last=l_)
            outs[k].copy_(wl.res, non_blocking=True)  # scores | max returns
            freed[k].record(main)
        p1.record(main)
        host_ms = (time.perf_counter() - host0) * 1e3 / args.steps
        torch.cuda.synchronize()
        clocks.active = False
        return p0.elapsed_time(p1), host_ms, nv + nl + na

    e2e_ms, host_ms, _ = pipelined(torch.float64, 20_000)
    # the same pipeline with the values as the policy's float32 (the reference's actor
    # returns value.double() of a float32 output, agents/ppo.py:96); the kernel widens
    # them, so a float32-valued stream scores identically with half the value bytes
    e32_ms, _, h2d32 = pipelined(torch.float32, 30_000)
    te = torch.tensor([e2e_ms, seq_ms, e32_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_ms, seq_ms, e32_ms = float(te[0].item()), float(te[1].item()), float(te[2].item())
    peaks, src = _peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    extra = {}
    if not args.no_extra:
        extra["plr"] = measure_plr(dev, 2048, T, False, max(3, min(args.steps, 10)), flush, world)
        extra["accel"] = measure_plr(dev, 2048, T, True, max(3, min(args.steps, 10)), flush, world)
        if world == 1:
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
        "metric": "AMaze env steps/sec (DR reset + 256-step RESAMPLE rollout + GAE/MaxMC)",
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
        "config": {"workload": "configs[1]: AMaze 13x13 DR, 4096 envs x 256 steps, RESAMPLE auto-reset, GAE+MaxMC",
                   "lanes_per_gpu": B, "T": T, "gamma": 0.995, "lambda": 0.95, "l2": "flushed (256 MB write) "
                   "before every timed step", "parallelism": f"lane-sharded x{world}"},
        "e2e": {"value": units / (e2e_ms * 1e-3 / args.steps), "unit": "env-steps/s",
                "h2d_bytes_per_step": T * B * (1 + 8) + B * 8, "d2h_bytes_per_step": 2 * B * 8,
                "ms_per_step": e2e_ms / args.steps, "host_enqueue_ms_per_step": host_ms,
                "mode": "pipelined: step i+1's pinned H2D copies (two copy streams, double-buffered) overlap step i; "
                        "one timed region over all K steps including every copy, the L2 flush and the result read",
                "sequential": {"value": units / (seq_ms * 1e-3 / args.steps), "ms_per_step": seq_ms / args.steps,
                               "mode": "copies, step and read back to back per step (flush outside the timing)"},
                "values_f32": {"value": units / (e32_ms * 1e-3 / args.steps), "ms_per_step": e32_ms / args.steps,
                               "h2d_bytes_per_step": h2d32,
                               "mode": "pipelined as above with values / last values staged as float32 (the "
                                       "policy's output dtype; gae_and_scores widens them in-kernel)"}},
        "gpu_launches": wl.launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_env_rollout", "achieved": roll_gbs, "peak": peak, "unit": "GB/s",
                     "frac": roll_gbs / peak,
                     "traffic": _traffic().get("k_env_rollout", {}).get("dram_bytes"),
                     "traffic_source": "profiles/r1m_traffic.json (ncu --set full, per launch)",
                     "peak_source": src,
                     "algorithmic_bytes": f"{ENV_BYTES_PER_STEP} B/env-step x {B * T} env-steps per launch",
                     "kernel_ms": roll,
                     "note": "k_env_rollout = k_dyn + k_render (the timeout levels of the first auto-resets "
                             "come prepared from the fused reset launch, so no k_spec_levels); at 4096 lanes the per-lane "
                             "256-step dynamics chain (latency) bounds it, not HBM; the HBM point is "
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


def measure_plr(dev, n_per_gpu, T, accel, iters, flush, world):
    """Parallel PLR (configs[2]) / ACCEL (configs[3]) iteration, env side: compose lanes
    (DR + rank-prioritised replay [+ 20-edit mutants]), HOME rollout, GAE + MaxMC,
    NCCL candidate all-gather (N > 1), buffer update.  Buffer K = 4000."""
    import torch

    import paper_2311_12716_b200 as amz
    from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig
    from paper_2311_12716_b200.plr import ParallelPLR

    cfg = PlrConfig(buffer_size=4000, score_fn="maxmc", temperature=0.3,
                    staleness_coef=0.5 if accel else 0.3, replay_rate=0.8 if accel else 0.5)
    plr = ParallelPLR(n_per_gpu * world, amz.StaticParams(), cfg, amz.RngStream.from_seed(7),
                      AccelConfig(20, 4) if accel else None, device=dev)
    L = plr.hi - plr.lo
    g = torch.Generator(device=dev)
    g.manual_seed(99 + plr.rank)
    acts = torch.randint(0, 3, (T, L), generator=g, device=dev, dtype=torch.uint8)
    vals = torch.rand((T, L), generator=g, device=dev, dtype=torch.float64) * 0.2
    last = torch.rand((L,), generator=g, device=dev, dtype=torch.float64) * 0.2
    for it in range(3):  # fills the 4000-level buffer (first iteration inserts 4000 of the new levels)
        plr.iteration(it, acts, vals, last)
    torch.cuda.synchronize()
    ms = _timed(lambda i: plr.iteration(3 + i, acts, vals, last), iters, flush, torch)
    # the two buffer kernels on their own (latency-bound single-CTA kernels): an update
    # with 4096 distinct new levels (scores U(0,1): most evict -- the worst case) and one
    # with 4096 replays of buffered levels (in-place updates)
    new_lv = amz.sample_levels(amz.RngStream(99, (0,)), 4096, amz.StaticParams(), device=dev)
    sc = torch.rand(4096, device=dev, dtype=torch.float64)
    sc2 = torch.rand(4000, device=dev, dtype=torch.float64)
    t_upd = _timed(lambda i: plr.buffer.update(new_lv, sc, sc, 1000 + i), iters, flush, torch)
    old_lv = plr.buffer.export()["levels"][:4000]  # exported after t_upd: every level is buffered
    t_rep = _timed(lambda i: plr.buffer.update(old_lv, sc2, sc2, 1000 + i), iters, flush, torch)
    t_smp = _timed(lambda i: plr.buffer.sample(amz.RngStream(5, (i,)), n_per_gpu * world, 2000 + i), iters, flush,
                   torch)
    t = torch.tensor([statistics.mean(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    it_ms = float(t.item())
    lanes = plr.L
    return {"config": "configs[3] ACCEL-parallel" if accel else "configs[2] PLR-parallel",
            "lanes_global": lanes, "T": T, "buffer_size": 4000, "iteration_ms": it_ms,
            "levels_scored_per_s": lanes / (it_ms * 1e-3), "env_steps_per_s": lanes * T / (it_ms * 1e-3),
            "buffer_update_us_4096_new_levels": 1e3 * statistics.mean(t_upd),
            "buffer_update_us_4000_replays": 1e3 * statistics.mean(t_rep),
            "buffer_sample_us": 1e3 * statistics.mean(t_smp)}


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
        wl.step(10 + i, timing=kev[i])
    torch.cuda.synchronize()
    roll = statistics.mean(k[0].elapsed_time(k[1]) for k in kev)
    gae = statistics.mean(k[1].elapsed_time(k[2]) for k in kev)
    rg = ENV_BYTES_PER_STEP * B * T / (roll * 1e-3) / 1e9
    gg = GAE_BYTES_PER_ELEM * B * T / (gae * 1e-3) / 1e9
    out = {"lanes": B, "T": T, "rollout_ms": roll, "rollout_GBs": rg, "rollout_frac": rg / peak,
           "rollout_env_steps_per_s": B * T / (roll * 1e-3), "gae_score_ms": gae, "gae_score_GBs": gg,
           "gae_score_frac": gg / peak, "levels_scored_per_s": B / (gae * 1e-3)}
    del wl
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
    import multiprocessing as mp

    cores = _cores()
    B, T = args.lanes, args.T
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        secs = [cpu_reference_step(B, T, args.seed, cores, pool) for _ in range(steps)]
    s = statistics.mean(secs)
    return {"value": B * T / s, "unit": "env-steps/s", "cores": cores, "kind": "port",
            "sample": f"one full step ({B} lanes x {T} steps DR reset + rollout + GAE/MaxMC) with the numpy oracle "
                      f"port, lanes sharded over {cores} processes; host: {_cpu_model()}"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import multiprocessing as mp

    cores = _cores()
    B, T = args.lanes, args.T
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_reference_step(B, T, args.seed, cores, pool)
        phases = []
        secs = [cpu_reference_step(B, T, args.seed, cores, pool, phases) for _ in range(args.steps)]
    s = statistics.mean(secs)
    val = B * T / s
    # the phases separately (slowest shard, mean over the timed steps), one
    # single-process step (no sharding), and the oracle buffer update (sequential)
    phase_ms = {k: 1e3 * statistics.mean(ph[k] for ph in phases) for k in ("reset", "rollout", "gae", "scores")}
    one = cpu_reference_step(B, T, args.seed, 1, None)
    buf_s = cpu_buffer_update_seconds(4096, 4000)
    return {
        "impl": "reference",
        "metric": "AMaze env steps/sec (DR reset + 256-step RESAMPLE rollout + GAE/MaxMC)",
        "value": val, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64 env, f64 GAE", "data": "synthetic (same workload, numpy random actions/values)",
        "config": {"workload": "configs[1]: AMaze 13x13 DR, 4096 envs x 256 steps, RESAMPLE auto-reset, GAE+MaxMC",
                   "lanes": B, "T": T},
        "cpu_baseline": {"value": val, "unit": "env-steps/s", "cores": cores, "kind": "port",
                         "sample": f"full config-2 step per timed step, numpy oracle port of the reference, "
                                   f"lanes sharded over {cores} processes; host: {_cpu_model()}"},
        "e2e": {"value": val, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_ms_per_step": phase_ms,
        "single_process": {"env_steps_per_s": B * T / one, "ms_per_step": one * 1e3, "cores": 1},
        "buffer_update_ms_4096_new_levels": buf_s * 1e3,
    }


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
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        import torch

        if world > 1:
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl")
        line = run_ours(args, rank, world, local_rank)
        if world > 1:
            torch.distributed.destroy_process_group()
    if line is not None:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
