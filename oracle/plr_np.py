"""Sequential PLR level buffer + parallel PLR/ACCEL lane composition -- TEST INFRASTRUCTURE ONLY.

The reference imports ``runners/buffer.py`` (runners/scoring.py:14) but never shipped
it; its behaviour exists only as prose in SPEC.md.  This module is a
literal transcription of that prose and is the parity oracle for the CUDA buffer
(paper_2311_12716_b200/csrc/amz_plr.cu):

  types       SPEC.md:332-343  LevelBufferEntry(level, score, max_return,
                               last_sampled_iter, insert_iter), PlrConfig, AccelConfig
  decision    SPEC.md:360-364  replay w.p. p iff the buffer is non-empty
  sample      SPEC.md:365-372  P = (1-rho) P_S + rho P_C, P_S ~ (1/rank)^(1/beta),
                               P_C ~ (iter - last_sampled); with replacement;
                               sampled entries get last_sampled = iter
  update      SPEC.md:373-377  per candidate, in order: identical level present ->
                               update score/max_return in place; else insert if not
                               full; else replace the min-score entry iff score > min
  decisions   SPEC.md:427-433  undiscounted MaxMC, all-new bootstrap, stale-first
                               eviction, dedupe by exact tile map incl. agent pose
  parallel    SPEC.md:400-411  PLR||: lanes [new n | replay n]; ACCEL||: [new | replay |
                               mutants of the q top-scoring replay lanes, cycled]

Choices SPEC leaves open, pinned here (and in DESIGN.md) so GPU and oracle agree:
  * rank ties: equal scores rank by insertion sequence number, older first;
  * eviction ties: (score, last_sampled, seq) lexicographic minimum -- the stale-first
    rule of SPEC.md:430, then the older insertion;
  * a new entry's last_sampled is its insertion iteration (staleness starts at 0);
  * in-place updates change score and max_return only;
  * if every staleness is 0, P = P_S (P_C is undefined);
  * sampling = numpy ``Generator.choice(size, n, p=P)`` on the stream's generator;
  * ACCEL parents: the q replay lanes with the highest buffer score at sampling time,
    ties to the lower lane index; mutant lane j uses parent j % q;
  * iteration keys: it = root.fold_in(iter); new-level lane keys it.fold_in(1)+(lane,),
    replay draw it.fold_in(2), mutation keys it.fold_in(3)+(j,), PLR-perp decision
    it.fold_in(0), HOME rollout reset it.fold_in(4) (PLR-perp mutant rollout: it.fold_in(5));
  * PLR-perp: NEW = n fresh levels, roll out, score, update; REPLAY =
    n draws, roll out from the entries' max returns, re-score the drawn entries in place
    (an update with the drawn levels); ACCEL-perp adds q mutants after a replay (parents
    = the q highest buffer scores among the drawn entries at sampling time, mutant j
    from parent j, keys it.fold_in(3)+(j,)), rolled out and scored from max return 0,
    then one update with them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import amaze_np as onp


@dataclass(frozen=True)
class PlrConfig:
    replay_rate: float = 0.5       # p
    buffer_size: int = 4000        # K
    score_fn: str = "maxmc"        # "maxmc" | "pvl"
    prioritization: str = "rank"   # "rank" | "proportional"
    temperature: float = 0.3       # beta
    staleness_coef: float = 0.3    # rho
    robust: bool = True
    maxmc_discounted: bool = False


def rank_weights(K: int, beta: float) -> np.ndarray:
    """(1/rank)^(1/beta) for ranks 1..K, float64 (the host LUT the GPU also uses)."""
    ranks = np.arange(1, K + 1, dtype=np.float64)
    return np.power(1.0 / ranks, 1.0 / beta)


class LevelBuffer:
    def __init__(self, capacity: int):
        self.K = capacity
        self.levels = np.zeros(capacity, dtype=onp.LEVEL_DTYPE)
        self.score = np.zeros(capacity)
        self.max_return = np.zeros(capacity)
        self.last_sampled = np.zeros(capacity, dtype=np.int64)
        self.seq = np.zeros(capacity, dtype=np.int64)
        self.size = 0
        self.next_seq = 0
        self._index = {}  # identity key -> slot

    @staticmethod
    def key(rec) -> bytes:
        """MazeLevel.key() equivalent on a packed record: wall bits + pose."""
        return rec["walls"].tobytes() + bytes([int(rec["agent_r"]), int(rec["agent_c"]), int(rec["agent_dir"]),
                                               int(rec["goal_r"]), int(rec["goal_c"])])

    # -- buffer_update -------------------------------------------
    def update(self, levels: np.ndarray, scores: np.ndarray, max_returns: np.ndarray, it: int) -> None:
        for rec, s, m in zip(levels, scores, max_returns):
            k = self.key(rec)
            slot = self._index.get(k)
            if slot is not None:
                self.score[slot] = s
                self.max_return[slot] = m
                continue
            if self.size < self.K:
                slot = self.size
                self.size += 1
            else:
                n = self.size
                order = np.lexsort((self.seq[:n], self.last_sampled[:n], self.score[:n]))
                slot = int(order[0])
                if not s > self.score[slot]:
                    continue
                del self._index[self.key(self.levels[slot])]
            self.levels[slot] = rec
            self.score[slot] = s
            self.max_return[slot] = m
            self.last_sampled[slot] = it
            self.seq[slot] = self.next_seq
            self.next_seq += 1
            self._index[k] = slot

    # -- buffer_sample_levels -------------------------------------
    def probabilities(self, cfg: PlrConfig, it: int) -> np.ndarray:
        n = self.size
        if n == 0:
            raise ValueError("cannot sample from an empty buffer")
        if cfg.prioritization == "rank":
            order = np.lexsort((self.seq[:n], -self.score[:n]))  # score desc, older first
            ranks = np.empty(n, dtype=np.int64)
            ranks[order] = np.arange(1, n + 1)
            w = rank_weights(self.K, cfg.temperature)[ranks - 1]
        else:
            w = np.power(self.score[:n], 1.0 / cfg.temperature)
        ps = w / w.sum()
        st = it - self.last_sampled[:n]
        tot = st.sum()
        if tot == 0:
            return ps
        pc = st / tot
        return (1 - cfg.staleness_coef) * ps + cfg.staleness_coef * pc

    def sample(self, entropy: int, key: tuple, n: int, cfg: PlrConfig, it: int) -> np.ndarray:
        p = self.probabilities(cfg, it)
        g = onp.generator(entropy, key)
        slots = g.choice(self.size, n, p=p)
        self.last_sampled[slots] = it
        return slots

    def decision(self, entropy: int, key: tuple, p: float) -> bool:
        """True = replay."""
        return self.size > 0 and onp.generator(entropy, key).random() < p

    def snapshot(self):
        n = self.size
        return (self.levels[:n].copy(), self.score[:n].copy(), self.max_return[:n].copy(),
                self.last_sampled[:n].copy(), self.seq[:n].copy())


def top_q(scores: np.ndarray, q: int) -> np.ndarray:
    """Indices of the q highest scores, ties to the lower index."""
    return np.argsort(-scores, kind="stable")[:q]


def compose_lanes(buf: LevelBuffer, entropy: int, root_key: tuple, it: int, n: int, p: onp.Params,
                  cfg: PlrConfig, accel=None):
    """Lane levels of one PLR||/ACCEL|| iteration.

    Returns (levels records [L], prior_max [L], n_replay, slots)."""
    itk = tuple(root_key) + (it,)
    thirds = 3 if accel is not None else 2
    if buf.size == 0:  # bootstrap: all-new
        L = thirds * n
        new = [onp.sample_level(entropy, itk + (1, i), p) for i in range(L)]
        return onp.pack_levels(new, p), np.zeros(L), 0, np.zeros(0, dtype=np.int64)
    new = onp.pack_levels([onp.sample_level(entropy, itk + (1, i), p) for i in range(n)], p)
    rep_scores_before = None
    slots = buf.sample(entropy, itk + (2,), n, cfg, it)
    rep = buf.levels[slots]
    rep_scores_before = buf.score[slots]
    parts = [new, rep]
    prior = [np.zeros(n), buf.max_return[slots].copy()]
    if accel is not None:
        q, n_edits = accel
        parents = top_q(rep_scores_before, q)
        par_levels = onp.unpack_levels(rep[parents], p)
        muts = [onp.mutate_level(entropy, itk + (3, j), par_levels[j % q], n_edits, p) for j in range(n)]
        parts.append(onp.pack_levels(muts, p))
        prior.append(np.zeros(n))
    return np.concatenate(parts), np.concatenate(prior), n, slots


def plr_perp_iteration(buf: LevelBuffer, entropy: int, root_key: tuple, it: int, n: int, p: onp.Params,
                       cfg: PlrConfig, rollout_score, accel=None):
    """One PLR-perp (or ACCEL-perp) iteration against this buffer.

    ``rollout_score(levels, prior, reset_key, which)`` rolls the packed levels out (HOME
    auto-reset from ``reset_key``) and returns (scores, max_returns); ``which`` is
    "main" or "mutants" so a harness can feed each rollout its own action stream.
    Returns dict(branch, levels, scores, max_returns, slots, mutants...)."""
    itk = tuple(root_key) + (it,)
    replay = buf.decision(entropy, itk + (0,), cfg.replay_rate)
    out = {"branch": "replay" if replay else "new"}
    if not replay:
        levels = onp.pack_levels([onp.sample_level(entropy, itk + (1, i), p) for i in range(n)], p)
        sc, mx = rollout_score(levels, np.zeros(n), itk + (4,), "main")
        buf.update(levels, sc, mx, it)
        out.update(levels=levels, scores=sc, max_returns=mx)
        return out
    slots = buf.sample(entropy, itk + (2,), n, cfg, it)
    levels = buf.levels[slots].copy()
    before = buf.score[slots].copy()
    sc, mx = rollout_score(levels, buf.max_return[slots].copy(), itk + (4,), "main")
    buf.update(levels, sc, mx, it)
    out.update(levels=levels, scores=sc, max_returns=mx, slots=slots)
    if accel is not None:
        q, n_edits = accel
        parents = top_q(before, q)
        par_levels = onp.unpack_levels(levels[parents], p)
        muts = onp.pack_levels([onp.mutate_level(entropy, itk + (3, j), par_levels[j], n_edits, p)
                                for j in range(q)], p)
        msc, mmx = rollout_score(muts, np.zeros(q), itk + (5,), "mutants")
        buf.update(muts, msc, mmx, it)
        out.update(mutants=muts, mutant_scores=msc, mutant_max_returns=mmx)
    return out
