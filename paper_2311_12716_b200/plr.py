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
        self.thirds = 3 if accel is not None else 2
        self.L = self.thirds * n
        self.rank, self.world = dist.world()
        self.lo, self.hi = dist.shard(self.L, self.rank, self.world)
        self.benv = VectorBatchEnv(MazeEnv(), BatchShape(1, 1, self.hi - self.lo), device=self.device,
                                   lane_offset=self.lo)
        self.env = AutoResetWrapper(self.benv, HOME)
        self.buffer = LevelBuffer(cfg, self.device)

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

    # -- one iteration ---------------------------------------------------------------------
    def iteration(self, it: int, actions, values, last_values, out=None) -> IterationResult:
        """actions uint8 [T, L_local], values f64 [T, L_local], last_values f64 [L_local]
        (the policy side's outputs for this rank's lanes)."""
        levels, prior, n_replay = self.compose(it)
        start = self.env.reset_to_levels(self.root.fold_in(it).fold_in(4), levels, self.p)
        traj, _ = rollout_actions(self.env, start, actions, self.p, out=out)
        o = gae_and_scores(traj.rewards, values, traj.dones, last_values, self.gamma, self.lam, prior,
                           self.cfg.score_fn, self.cfg.maxmc_discounted)
        g_levels, g_scores, g_max = dist.gather_candidates(levels, o["scores"], o["max_returns"])
        self.buffer.update(g_levels, g_scores, g_max, it)
        return IterationResult(levels, o["scores"], o["max_returns"], n_replay, traj, o["advantages"])
