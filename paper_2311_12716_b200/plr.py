"""Parallel PLR (PLR||) and parallel ACCEL (ACCEL||) iterations, env side, on the GPU.

SPEC.md:400-411: one rollout over a lane batch laid out as [new n | replay n] (PLR||)
or [new n | replay n | mutants n] (ACCEL||, mutants of the q top-scoring replay lanes,
cycled), all lanes scored, one buffer_update with the whole batch in lane order.  An
empty buffer runs all-new lanes.  The policy update is out of scope: the
caller supplies the action stream and value estimates (or a policy callback fills
them) -- this module is the curriculum hot path around it.

Keys (pinned identically in oracle/plr_np.py): it = root.fold_in(iteration); new-level
lane keys it.fold_in(1) + (global lane,), replay draw it.fold_in(2), mutation keys
it.fold_in(3) + (mutant index,).

PLR-perp / ACCEL-perp (SequentialPLR): one branch per iteration
(NEW or REPLAY, decided by the iteration key's uniform), same keys, buffer and kernels.

Multi-GPU: each rank owns a contiguous slice of the global lane layout (dist.shard),
composes only its slice (the replay draw and top-q are replicated, not exchanged),
rolls out and scores its slice, then all-gathers the 48-byte candidate records and
applies the identical buffer update (dist.gather_candidates).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import dist
from .amaze import MazeEnv, mutate_levels, sample_levels
from .batch import HOME, AutoResetWrapper, VectorBatchEnv
from .buffer import AccelConfig, LevelBuffer, PlrConfig, top_q
from .core import BatchShape, StaticParams, as_params
from .gae import gae_and_scores
from .rng import as_stream
from .rollout import rollout_actions


def _torch():
    import torch

    return torch


@dataclass
class IterationResult:
    levels: object         # [L_local, 8] lane levels
    scores: object         # [L_local] f64
    max_returns: object    # [L_local] f64
    n_replay: int          # global replay lanes this iteration (0 = bootstrap)
    trajectory: object     # TrajectoryBatch of the local lanes
    advantages: object


class ParallelPLR:
    """PLR|| / ACCEL|| over n new lanes per iteration (L = 2n or 3n
    lanes globally, sharded over the torch.distributed world).  ``check_every`` > 0 runs
    the replica drift check (on-device buffer digest + one all-reduce, RunnerFault on a
    mismatch) after every ``check_every``-th iteration when world > 1.  In a 1-rank
    world the lane levels of an ``IterationResult`` live in internal double-buffered
    arrays: valid until the iteration after next (clone to keep them longer)."""

    def __init__(self, n: int, params: StaticParams, cfg: PlrConfig, root_rng, accel: AccelConfig | None = None,
                 gamma: float = 0.995, lam: float = 0.95, device=None, check_every: int = 16):
        torch = _torch()
        self.n = n
        self.p = as_params(params).validate()
        self.cfg = cfg.validate()
        self.accel = accel
        self.root = as_stream(root_rng)
        self.gamma, self.lam = gamma, lam
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.thirds = 3 if accel is not None else 2
        self.L = self.thirds * n
        self.rank, self.world = dist.world()
        self.lo, self.hi = dist.shard(self.L, self.rank, self.world)
        self.benv = VectorBatchEnv(MazeEnv(), BatchShape(1, 1, self.hi - self.lo), device=self.device,
                                   lane_offset=self.lo)
        self.env = AutoResetWrapper(self.benv, HOME)
        self.buffer = LevelBuffer(cfg, self.device)
        self.check_every = int(check_every)
        self.iterations = 0

    # -- lane composition ---------------------------------------------------------------
    def compose(self, it: int):
        """Levels and prior max returns of this rank's lanes for iteration ``it``."""
        torch = _torch()
        itr = self.root.fold_in(it)
        lo, hi, n, dev = self.lo, self.hi, self.n, self.device
        if not self.buffer.nonempty:  # bootstrap: all lanes new
            ids = torch.arange(lo, hi, device=dev, dtype=torch.int32)
            levels = sample_levels(itr.fold_in(1), hi - lo, self.p, lane_ids=ids, device=dev)
            return levels, torch.zeros(hi - lo, dtype=torch.float64, device=dev), 0
        if self.world == 1:
            return self._compose_local(itr, it)
        parts, priors = [], []
        # new lanes [0, n)
        a, b = max(lo, 0), min(hi, n)
        if a < b:
            ids = torch.arange(a, b, device=dev, dtype=torch.int32)
            parts.append(sample_levels(itr.fold_in(1), b - a, self.p, lane_ids=ids, device=dev))
            priors.append(torch.zeros(b - a, dtype=torch.float64, device=dev))
        # replay lanes [n, 2n): replicated draw, local slice
        rep = self.buffer.sample(itr.fold_in(2), n, it)
        a, b = max(lo, n), min(hi, 2 * n)
        if a < b:
            parts.append(rep["levels"][a - n:b - n])
            priors.append(rep["max_returns"][a - n:b - n])
        # mutant lanes [2n, 3n): parents = q top replay lanes by buffer score, cycled
        if self.accel is not None:
            a, b = max(lo, 2 * n), min(hi, 3 * n)
            if a < b:
                q = self.accel.subsample_size
                top = top_q(rep["scores"], q)
                pidx = top[(torch.arange(a - 2 * n, b - 2 * n, device=dev) % q)]
                parts.append(mutate_levels(itr.fold_in(3), rep["levels"], self.accel.n_mutations, self.p,
                                           lane0=a - 2 * n, parent_idx=pidx))
                priors.append(torch.zeros(b - a, dtype=torch.float64, device=dev))
        return torch.cat(parts), torch.cat(priors), n

    def _compose_local(self, itr, it: int):
        """compose() for a 1-rank world without staging copies: the new levels, the replay
        draw (levels and prior max returns) and the mutants are written straight into
        preallocated lane arrays (alternating between two sets, so an iteration's
        ``IterationResult.levels`` stays valid through the next iteration); the prior of
        new and mutant lanes is a zero region nothing writes."""
        torch = _torch()
        n, dev = self.n, self.device
        if not hasattr(self, "_lane_bufs"):
            self._lane_bufs = [(torch.empty((self.L, 8), dtype=torch.int32, device=dev),
                                torch.zeros(self.L, dtype=torch.float64, device=dev)) for _ in range(2)]
            if self.accel is not None:  # mutant j takes parent j mod q of the top-q replay lanes
                self._pcycle = torch.arange(n, device=dev) % self.accel.subsample_size
        lv, pr = self._lane_bufs[self.iterations & 1]
        sample_levels(itr.fold_in(1), n, self.p, lane0=0, out=lv[:n])
        rep = self.buffer.sample(itr.fold_in(2), n, it, out={"levels": lv[n:2 * n], "max_returns": pr[n:2 * n]})
        if self.accel is not None:
            top = top_q(rep["scores"], self.accel.subsample_size)
            mutate_levels(itr.fold_in(3), lv[n:2 * n], self.accel.n_mutations, self.p, lane0=0,
                          parent_idx=top[self._pcycle], out=lv[2 * n:3 * n])
        return lv, pr, n

    # -- one iteration ---------------------------------------------------------------------
    def iteration(self, it: int, actions, values, last_values, out=None) -> IterationResult:
        """actions uint8 [T, L_local], values f64 [T, L_local], last_values f64 [L_local]
        (the policy side's outputs for this rank's lanes)."""
        torch = _torch()
        levels, prior, n_replay = self.compose(it)
        side = None
        if self.world == 1:
            # the update's candidate twin table depends on the levels only: build it on a
            # side stream beside the rollout (joined before the update)
            if not hasattr(self, "_prep_stream"):
                self._prep_stream = torch.cuda.Stream(device=self.device)
            side = self._prep_stream
            cur = torch.cuda.current_stream(self.device)
            side.wait_stream(cur)
            self.buffer.prepare(levels, stream=side)
        start = self.env.reset_to_levels(self.root.fold_in(it).fold_in(4), levels, self.p)
        tout, gout = self._iteration_outputs(actions.shape[0], out)
        traj, _ = rollout_actions(self.env, start, actions, self.p, out=tout)
        o = gae_and_scores(traj.rewards, values, traj.dones, last_values, self.gamma, self.lam, prior,
                           self.cfg.score_fn, self.cfg.maxmc_discounted, out=gout)
        g_levels, g_scores, g_max = dist.gather_candidates(levels, o["scores"], o["max_returns"])
        if side is not None:
            torch.cuda.current_stream(self.device).wait_stream(side)
            levels.record_stream(side)
        self.buffer.update(g_levels, g_scores, g_max, it)
        self.iterations += 1
        if self.world > 1 and self.check_every > 0 and self.iterations % self.check_every == 0:
            self.check_replicas()
        return IterationResult(levels, o["scores"], o["max_returns"], n_replay, traj, o["advantages"])

    def _iteration_outputs(self, T: int, out):
        """Trajectory and GAE result tensors of this iteration: two persistent sets used in
        turn (like the lane arrays of _compose_local, an IterationResult stays valid
        through the next iteration), so an iteration allocates nothing; a caller's
        ``out`` (rollout tensors) takes precedence."""
        torch = _torch()
        n, dev, v = self.hi - self.lo, self.device, self.p.agent_view_size
        if getattr(self, "_out_T", None) != T:
            self._out_T = T
            self._out_sets = [({"view": torch.empty((T, n, v, v), dtype=torch.uint8, device=dev),
                                "dir": torch.empty((T, n), dtype=torch.uint8, device=dev),
                                "rewards": torch.empty((T, n), dtype=torch.float64, device=dev),
                                "dones": torch.empty((T, n), dtype=torch.bool, device=dev),
                                "final_view": torch.empty((n, v, v), dtype=torch.uint8, device=dev),
                                "final_dir": torch.empty((n,), dtype=torch.uint8, device=dev)},
                               {"advantages": torch.empty((T, n), dtype=torch.float64, device=dev),
                                "returns": torch.empty((T, n), dtype=torch.float64, device=dev),
                                "scores": torch.empty((n,), dtype=torch.float64, device=dev),
                                "max_returns": torch.empty((n,), dtype=torch.float64, device=dev)})
                              for _ in range(2)]
        tout, gout = self._out_sets[self.iterations & 1]
        return (out if out is not None else tout), gout

    def check_replicas(self) -> None:
        """Drift check now: every rank's buffer digest must agree (RunnerFault if not)."""
        dist.check_replicas(self.buffer.digest())


@dataclass
class PerpResult:
    branch: str            # "new" | "replay"
    levels: object         # [n, 8] levels rolled out (fresh or drawn)
    scores: object
    max_returns: object
    slots: object          # drawn slots (replay) or None
    trajectory: object
    advantages: object
    mutants: object = None             # ACCEL-perp: [q, 8] mutant levels (replay branch)
    mutant_scores: object = None
    mutant_max_returns: object = None


class SequentialPLR:
    """PLR-perp / ACCEL-perp (`plr_iteration`): one branch per iteration.

    * decision (buffer_sample_decision, key it.fold_in(0)): replay w.p. p iff non-empty;
    * NEW: n fresh DR levels (keys it.fold_in(1) + (lane,)), HOME rollout, score from max
      return 0, buffer_update with the n candidates;
    * REPLAY: n rank-prioritised draws (key it.fold_in(2)), rollout from the entries' max
      returns, the drawn entries re-scored in place (buffer_update with the drawn levels);
      with ACCEL, the q drawn entries with the highest buffer score at sampling time are
      mutated (mutant j from parent j, keys it.fold_in(3) + (j,)), rolled out (HOME, reset
      key it.fold_in(5)) and scored from 0, then one buffer_update with the q mutants.

    The caller (the policy side) supplies actions / values for the n main lanes and,
    optionally, for the q mutant lanes (default: the first q columns of the main
    streams).  Same keys, buffer and kernels as ParallelPLR; the oracle is
    oracle/plr_np.plr_perp_iteration."""

    def __init__(self, n: int, params: StaticParams, cfg: PlrConfig, root_rng, accel: AccelConfig | None = None,
                 gamma: float = 0.995, lam: float = 0.95, device=None):
        torch = _torch()
        self.n = n
        self.p = as_params(params).validate()
        self.cfg = cfg.validate()
        self.accel = accel
        self.root = as_stream(root_rng)
        self.gamma, self.lam = gamma, lam
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.env = AutoResetWrapper(VectorBatchEnv(MazeEnv(), BatchShape(1, 1, n), device=self.device), HOME)
        self.menv = None
        if accel is not None:
            self.menv = AutoResetWrapper(VectorBatchEnv(MazeEnv(), BatchShape(1, 1, accel.subsample_size),
                                                        device=self.device), HOME)
        self.buffer = LevelBuffer(cfg, self.device)

    def decide(self, it: int) -> bool:
        """True = replay this iteration (host: one uniform of the iteration's key)."""
        return self.buffer.decision(self.root.fold_in(it).fold_in(0))

    def _roll_score(self, env, key, levels, prior, actions, values, last, out=None):
        start = env.reset_to_levels(key, levels, self.p)
        traj, _ = rollout_actions(env, start, actions, self.p, out=out)
        o = gae_and_scores(traj.rewards, values, traj.dones, last, self.gamma, self.lam, prior,
                           self.cfg.score_fn, self.cfg.maxmc_discounted)
        return traj, o

    def iteration(self, it: int, actions, values, last_values, mutant_inputs=None, out=None) -> PerpResult:
        """actions uint8 [T, n], values f64 [T, n], last_values f64 [n]; ``mutant_inputs``
        = (actions [T, q], values [T, q], last [q]) for the ACCEL mutant rollout."""
        torch = _torch()
        itr = self.root.fold_in(it)
        n, dev = self.n, self.device
        if not self.decide(it):
            levels = sample_levels(itr.fold_in(1), n, self.p, lane0=0, device=dev)
            if not hasattr(self, "_zero_prior"):
                self._zero_prior = torch.zeros(n, dtype=torch.float64, device=dev)  # read-only
            traj, o = self._roll_score(self.env, itr.fold_in(4), levels, self._zero_prior, actions, values,
                                       last_values, out)
            self.buffer.update(levels, o["scores"], o["max_returns"], it)
            return PerpResult("new", levels, o["scores"], o["max_returns"], None, traj, o["advantages"])
        rep = self.buffer.sample(itr.fold_in(2), n, it)
        traj, o = self._roll_score(self.env, itr.fold_in(4), rep["levels"], rep["max_returns"], actions, values,
                                   last_values, out)
        self.buffer.update(rep["levels"], o["scores"], o["max_returns"], it)
        res = PerpResult("replay", rep["levels"], o["scores"], o["max_returns"], rep["slots"], traj, o["advantages"])
        if self.accel is not None:
            q = self.accel.subsample_size
            top = top_q(rep["scores"], q)  # buffer scores at sampling time
            muts = mutate_levels(itr.fold_in(3), rep["levels"], self.accel.n_mutations, self.p, lane0=0,
                                 parent_idx=top)
            if mutant_inputs is None:
                mutant_inputs = (actions[:, :q], values[:, :q], last_values[:q])
            ma, mv, ml = (x.contiguous() for x in mutant_inputs)
            _, mo = self._roll_score(self.menv, itr.fold_in(5), muts, torch.zeros(q, dtype=torch.float64, device=dev),
                                     ma, mv, ml)
            self.buffer.update(muts, mo["scores"], mo["max_returns"], it)
            res.mutants, res.mutant_scores, res.mutant_max_returns = muts, mo["scores"], mo["max_returns"]
        return res
