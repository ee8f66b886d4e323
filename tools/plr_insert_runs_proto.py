"""Prototype (numpy, host) of the parallel "insert run" buffer update that k_plr_update
implements, checked against the sequential oracle (oracle/plr_np.py) on tie-heavy
random batches:  python tools/plr_insert_runs_proto.py [trials]

A run is a maximal stretch of consecutive candidates that are certainly new (no key
match in the buffer at kernel start, first occurrence of their key in the batch).  For
such a run the sequential rule (insert while not full, else replace the
(score, last_sampled, seq)-minimum iff score > its score) is a streaming top-K under the
order x < y  <=>  score(x) < score(y), or equal scores and x entered first (every stored
entry entered before every candidate of the run; free slots are virtual entries of
score -inf in slot order).  With that order:
  accept_i  <=>  #{j < i : s_j > s_i} < #{x in buffer : s_x <= s_i}
  the p accepted candidates evict the p smallest of (buffer U accepted), in order, and
  the k-th acceptance takes the slot of the k-th eviction (chained through earlier
  acceptances that are evicted again).
The order differs from the real rule only when a candidate's score EQUALS the score of
the minimum present at its arrival (the real rule rejects, the order would accept).
That minimum is exactly element q_i of the merged order (q_i = acceptances before i:
every later acceptance exceeds it), so the first such candidate f is found exactly; the
prefix before f is committed, f and every later candidate scoring <= s_f are rejected
(the minimum never drops), and the next pass runs over the rest.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import amaze_np as onp  # noqa: E402
from oracle import plr_np  # noqa: E402


def proto_update(buf: plr_np.LevelBuffer, levels, scores, maxrets, it, stats):
    K = buf.K
    init_keys = {buf.key(buf.levels[s]): s for s in range(buf.size)}
    seen = set()
    pure = []
    for rec in levels:
        k = buf.key(rec)
        pure.append(k not in init_keys and k not in seen)
        seen.add(k)
    n = len(levels)
    i = 0
    while i < n:
        if not pure[i] or (buf.size > 0 and buf.last_sampled[:buf.size].max() > it):
            buf.update(levels[i:i + 1], scores[i:i + 1], maxrets[i:i + 1], it)
            stats["seq"] += 1
            i += 1
            continue
        j = i
        while j < n and pure[j]:
            j += 1
        i = run(buf, levels, scores, maxrets, it, i, j, stats)


def run(buf, levels, scores, maxrets, it, r0, r1, stats):
    """Apply candidates [r0, r1) (all certainly new) in passes; returns r1."""
    live = list(range(r0, r1))
    while live:
        K, size = buf.K, buf.size
        s = np.array([scores[c] for c in live], dtype=np.float64) + 0.0  # -0.0 -> 0.0
        m = len(s)
        # buffer in eviction order (virtual free slots first, in slot order)
        ex_score = np.concatenate([np.full(K - size, -np.inf), buf.score[:size] + 0.0])
        ex_last = np.concatenate([np.zeros(K - size, np.int64), buf.last_sampled[:size]])
        ex_seq = np.concatenate([np.arange(K - size), buf.seq[:size]])
        ex_slot = np.concatenate([np.arange(size, K), np.arange(size)])
        ex_virtual = np.concatenate([np.ones(K - size, bool), np.zeros(size, bool)])
        order = np.lexsort((ex_seq, ex_last, ~ex_virtual, ex_score))
        below = np.searchsorted(ex_score[order], s, side="right")
        greater = np.array([(s[:i] > s[i]).sum() for i in range(m)], dtype=np.int64)
        acc = greater < below
        A = np.nonzero(acc)[0]
        p = len(A)
        q = np.concatenate([[0], np.cumsum(acc)])[:m]  # acceptances before each arrival
        items = [(ex_score[o], 0, k, ("b", o)) for k, o in enumerate(order)]
        items += [(s[a], 1, a, ("a", a)) for a in A]
        items.sort(key=lambda x: (x[0], x[1], x[2]))
        # exact ties: the minimum present at arrival i is merged element q_i
        flags = [i for i in range(m) if items[q[i]][0] == s[i]]
        f = flags[0] if flags else m
        stats["runs"] += 1
        stats["flagged"] += int(bool(flags))
        acc_before = [a for a in A if a < f]
        slot_of_new = {}
        size_new = size
        for jj, a in enumerate(acc_before):
            kind, ref = items[jj][3]
            if kind == "b":
                slot = int(ex_slot[ref])
                if ex_virtual[ref]:
                    size_new += 1
                else:
                    del buf._index[buf.key(buf.levels[slot])]
            else:
                slot = slot_of_new.pop(ref)
                del buf._index[buf.key(levels[live[ref]])]
            slot_of_new[a] = slot
            c = live[a]
            buf.levels[slot] = levels[c]
            buf.score[slot] = scores[c]
            buf.max_return[slot] = maxrets[c]
            buf.last_sampled[slot] = it
            buf.seq[slot] = buf.next_seq
            buf.next_seq += 1
            buf._index[buf.key(levels[c])] = slot
        buf.size = size_new
        stats["par"] += f
        if f < m:  # f and every later candidate scoring <= s_f are rejected
            live = [live[i] for i in range(f + 1, m) if s[i] > s[f]]
        else:
            live = []
    return r1


def same(a, b):
    return (a.size == b.size and a.next_seq == b.next_seq and np.array_equal(a.levels[:a.size], b.levels[:b.size])
            and np.array_equal(a.score[:a.size], b.score[:b.size])
            and np.array_equal(a.max_return[:a.size], b.max_return[:b.size])
            and np.array_equal(a.last_sampled[:a.size], b.last_sampled[:b.size])
            and np.array_equal(a.seq[:a.size], b.seq[:b.size]))


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    p = onp.Params()
    pool = onp.pack_levels([onp.sample_level(1, (0, i), p) for i in range(600)], p)
    stats = {"runs": 0, "flagged": 0, "par": 0, "seq": 0}
    for t in range(trials):
        rng = np.random.default_rng(t)
        K = int(rng.choice([4, 16, 60, 200]))
        a, b = plr_np.LevelBuffer(K), plr_np.LevelBuffer(K)
        for it in range(5):
            n = int(rng.integers(1, 3 * K))
            idx = rng.integers(0, len(pool), n)
            choices = [0.0, -0.0, 0.1, 0.2, 0.2, 0.3] if t % 3 == 0 else None
            sc = rng.choice(choices, n) if choices else np.round(rng.uniform(0, 1, n), int(rng.integers(1, 4)))
            mx = rng.uniform(0, 1, n)
            a.update(pool[idx], sc, mx, it)
            proto_update(b, pool[idx], sc, mx, it, stats)
            assert same(a, b), (t, it)
            if rng.uniform() < 0.3 and b.size:  # replay marks (last_sampled = it)
                sl = rng.integers(0, b.size, 5)
                a.last_sampled[sl] = it
                b.last_sampled[sl] = it
    print("ok", stats)


if __name__ == "__main__":
    main()
