"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference package is imported read-only from /root/reference/pkg/src.  Its
``runners/scoring.py`` imports a ``runners/buffer.py`` that the reference never
shipped; we inject a stub module carrying only the two fields
``lane_scores`` reads (``score_fn``, ``maxmc_discounted``, runners/scoring.py:52,59).

Nothing at test time reads /root/reference: the tests read only the .npz files
written here.
"""

from __future__ import annotations

import os
import sys
import types
from dataclasses import dataclass

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.path.insert(0, REF)
    stub = types.ModuleType("autocurricula.runners.buffer")

    @dataclass
    class PlrConfig:  # fields read by runners/scoring.py:52,59
        score_fn: str = "maxmc"
        maxmc_discounted: bool = False

    stub.PlrConfig = PlrConfig
    sys.modules["autocurricula.runners.buffer"] = stub
    import autocurricula  # noqa: F401
    from autocurricula import amaze, env, rng
    import importlib

    gae = importlib.import_module("autocurricula.agents.gae")
    rollout = importlib.import_module("autocurricula.agents.rollout")
    scoring = importlib.import_module("autocurricula.runners.scoring")

    return types.SimpleNamespace(amaze=amaze, env=env, rng=rng, gae=gae, rollout=rollout,
                                 scoring=scoring, PlrConfig=PlrConfig)


def pack(levels, H, W):
    """MazeLevel list -> [N, 9] int64 rows: 4 mask words, agent r, c, dir, goal r, c."""
    rows = []
    for lv in levels:
        inner = np.asarray(lv.walls)[1:-1, 1:-1].reshape(-1).astype(np.uint64)
        bits = np.zeros(128, dtype=np.uint64)
        bits[: inner.size] = inner
        words = [int((bits[32 * k: 32 * k + 32] << np.arange(32, dtype=np.uint64)).sum()) for k in range(4)]
        rows.append(words + [lv.agent_pos[0], lv.agent_pos[1], lv.agent_dir, lv.goal_pos[0], lv.goal_pos[1]])
    return np.array(rows, dtype=np.int64)


def gen_levels(R):
    out = {}
    cases = [  # (name, H, W, budget, seed, n)
        ("default", 13, 13, 60, 0, 600),
        ("seed12345", 13, 13, 60, 12345, 200),
        ("budget0", 13, 13, 0, 3, 100),
        ("budget1", 13, 13, 1, 4, 100),
        ("budget119", 13, 13, 119, 5, 200),
        ("small9", 9, 9, 25, 6, 200),
    ]
    for name, H, W, budget, seed, n in cases:
        P = R.env.StaticParams(height=H, width=W, wall_budget=budget)
        root = R.rng.RngStream.from_seed(seed)
        # lane keys (seed, (0, i)) -- the VectorBatchEnv.reset lane streams
        levels = [R.amaze.sample_random_level(k, P) for k in root.fold_in(0).split(n)]
        out[f"lv_{name}"] = pack(levels, H, W)
        out[f"lv_{name}_meta"] = np.array([H, W, budget, seed, n], dtype=np.int64)
        # mutation keys (seed, (7, i)); 20 edits and 1 edit
        for ne in (1, 20):
            muts = [R.amaze.mutate_level(root.fold_in(7).fold_in(i), lv, ne, P) for i, lv in enumerate(levels)]
            out[f"mut{ne}_{name}"] = pack(muts, H, W)
    # large seeds exercise the multi-word entropy path
    P = R.env.StaticParams()
    root = R.rng.RngStream.from_seed(2**40 + 17)
    levels = [R.amaze.sample_random_level(k, P) for k in root.fold_in(0).split(100)]
    out["lv_bigseed"] = pack(levels, 13, 13)
    out["lv_bigseed_meta"] = np.array([13, 13, 60, 2**40 + 17, 100], dtype=np.int64)
    return out


def gen_rollout(R, name, shape, mode, T, seed, act_seed, see_through=True, levels_from=None):
    P = R.env.StaticParams(see_through_walls=see_through)
    menv = R.amaze.MazeEnv()
    benv = R.env.batch_lift(menv, R.env.BatchShape(*shape))
    wrap = R.env.AutoResetWrapper(benv, mode)
    root = R.rng.RngStream.from_seed(seed)
    if levels_from is None:
        res = wrap.reset(root, P)
    else:
        res = wrap.reset_to_levels(root, levels_from, P)
    B = int(np.prod(shape))
    flat = R.rollout.flatten_obs
    acts = np.stack([R.rng.RngStream.from_seed(act_seed).fold_in(t).generator().integers(0, 3, size=B)
                     for t in range(T)])
    obs = flat(res.observation)
    o = {f"{name}_view0": obs["view"], f"{name}_dir0": obs["dir"]}
    views, dirs, rews, dones, solved, times = [], [], [], [], [], []
    state, extras = res.state, res.extras
    for t in range(T):
        r = wrap.step(None, state, acts[t].reshape(shape[0], -1), P, extras)
        ob = flat(r.observation)
        views.append(ob["view"]); dirs.append(ob["dir"])
        rews.append(r.reward.reshape(-1)); dones.append(r.done.reshape(-1))
        solved.append(r.info["solved"].reshape(-1)); times.append(r.info["time"].reshape(-1))
        state, extras = r.state, r.extras
    o.update({
        f"{name}_actions": acts.astype(np.uint8),
        f"{name}_view": np.stack(views), f"{name}_dir": np.stack(dirs).astype(np.uint8),
        f"{name}_reward": np.stack(rews), f"{name}_done": np.stack(dones),
        f"{name}_solved": np.stack(solved), f"{name}_time": np.stack(times).astype(np.int32),
        f"{name}_meta": np.array([shape[0], shape[1], shape[2], T, seed, act_seed,
                                  int(mode == "home"), int(see_through)], dtype=np.int64),
        f"{name}_final_levels": pack(benv.lane_levels(state), 13, 13),
    })
    return o


def gen_scores(R):
    rng = np.random.default_rng(0)
    T, B = 256, 96
    V = rng.uniform(0.0, 1.0, (T, B))
    d = rng.uniform(size=(T, B)) < 1.0 / 40
    r = np.where(d & (rng.uniform(size=(T, B)) < 0.5), 1.0 - 0.9 * rng.integers(1, 251, (T, B)) / 250, 0.0)
    # a few lanes with nonzero rewards off done steps (generic GAE inputs)
    r[:, :8] += rng.normal(0, 0.1, (T, 8))
    last = rng.uniform(0, 1, B)
    prior = np.where(rng.uniform(size=B) < 0.5, rng.uniform(0, 1, B), 0.0)
    out = {"sc_r": r, "sc_v": V, "sc_d": d, "sc_last": last, "sc_prior": prior}
    for tag, g, lam in (("a", 0.999, 0.98), ("b", 0.995, 0.95), ("c", 1.0, 1.0)):
        adv, ret = R.gae.compute_gae(r, V, d, last, g, lam)
        out[f"sc_{tag}_adv"], out[f"sc_{tag}_ret"] = adv, ret
        out[f"sc_{tag}_gl"] = np.array([g, lam])
        tb = R.rollout.TrajectoryBatch({}, np.zeros((T, B), np.int64), np.zeros((T, B)), V, r, d,
                                       np.zeros((T, B, 1)))
        for fn in ("maxmc", "pvl"):
            for disc in (False, True):
                cfg = R.PlrConfig(score_fn=fn, maxmc_discounted=disc)
                s, m = R.scoring.lane_scores(tb, adv, prior, cfg, gamma=g)
                out[f"sc_{tag}_{fn}_{int(disc)}_score"], out[f"sc_{tag}_{fn}_{int(disc)}_maxret"] = s, m
        st = R.rollout.per_lane_episode_stats(r, d, gamma=g)
        for k, v in st.items():
            out[f"sc_{tag}_stats_{k}"] = v
    # SPEC known answers (runners/scoring.py)
    out["ka_pvl"] = np.array([R.scoring.score_pvl(np.array([0.5, -0.2, 0.3]))])
    out["ka_maxmc"] = np.array([R.scoring.score_maxmc(np.full(7, 0.2), 1.0)])
    return out


def gen_assets(R):
    names = R.amaze.asset_names()
    levels = [R.amaze.load_asset(n) for n in names]
    out = {"asset_levels": pack(levels, 13, 13),
           "asset_names": np.array(names)}
    for st in (True, False):
        P = R.env.StaticParams(see_through_walls=st)
        obs = [R.amaze.observe(R.amaze.EnvState.from_level(lv), P) for lv in levels]
        out[f"asset_view_st{int(st)}"] = np.stack([o.view for o in obs])
    return out


def gen_states(R):
    """Random (level, pose) states observed with and without occlusion (scalar path)."""
    rng = np.random.default_rng(1)
    P = R.env.StaticParams()
    root = R.rng.RngStream.from_seed(99)
    levels = [R.amaze.sample_random_level(k, P) for k in root.split(400)]
    poses = []
    out = {}
    for st in (True, False):
        P2 = R.env.StaticParams(see_through_walls=st)
        views = []
        for i, lv in enumerate(levels):
            if st:
                free = np.argwhere(~lv.walls)
                rc = free[rng.integers(len(free))]
                poses.append([rc[0], rc[1], rng.integers(4)])
            pr, pc, pd = poses[i]
            s = R.amaze.EnvState(lv, (int(pr), int(pc)), int(pd), 0, False)
            views.append(R.amaze.observe(s, P2).view)
        out[f"st_view_st{int(st)}"] = np.stack(views)
    out["st_levels"] = pack(levels, 13, 13)
    out["st_poses"] = np.array(poses, dtype=np.int64)
    return out


def gen_metrics(R):
    """env_metrics (amaze/metrics.py:21-31: BFS agent -> goal, amaze/pathfinding.py:116-135)."""
    out = {}
    cases = [  # (name, H, W, budget, seed, n)
        ("default", 13, 13, 60, 21, 400),
        ("dense", 13, 13, 119, 22, 300),
        ("small9", 9, 9, 30, 23, 200),
        ("wide", 11, 15, 70, 24, 200),
    ]
    sets = []
    for name, H, W, budget, seed, n in cases:
        P = R.env.StaticParams(height=H, width=W, wall_budget=budget)
        root = R.rng.RngStream.from_seed(seed)
        sets.append((name, H, W, [R.amaze.sample_random_level(k, P) for k in root.fold_in(0).split(n)]))
    sets.append(("assets", 13, 13, [R.amaze.load_asset(nm) for nm in R.amaze.asset_names()]))
    from autocurricula.amaze.metrics import env_metrics
    for name, H, W, levels in sets:
        ms = [env_metrics(lv) for lv in levels]
        out[f"m_{name}_levels"] = pack(levels, H, W)
        out[f"m_{name}_meta"] = np.array([H, W], dtype=np.int64)
        out[f"m_{name}_nwalls"] = np.array([m.n_walls for m in ms], dtype=np.int64)
        out[f"m_{name}_spl"] = np.array([m.shortest_path_length for m in ms], dtype=np.int64)
        out[f"m_{name}_solvable"] = np.array([m.solvable for m in ms], dtype=bool)
        out[f"m_{name}_passable"] = np.array([m.passable_ratio for m in ms], dtype=np.float64)
    return out


class _ExactActor:
    """A policy whose arithmetic is exact in any evaluation order (small integer sums
    times powers of two), so a torch copy on the GPU reproduces it bit for bit; the
    action hand-off is the reference's own sample_actions / log_softmax_np."""

    def __init__(self, R):
        self.R = R

    def initial_hidden(self, n):
        return np.zeros((n, 2))

    def logits(self, obs):
        view = obs["view"].astype(np.int64).reshape(obs["dir"].shape[0], -1)
        d = obs["dir"].astype(np.int64)
        idx = np.arange(view.shape[1])
        cols = [(((view + 1) * (a + 2 + idx % 3)) % 5).sum(axis=1) * 0.25 - 0.5 * ((d + a) % 4) for a in range(3)]
        return np.stack(cols, axis=1).astype(np.float64)

    def act(self, obs, hidden, g=None, greedy=False):
        import importlib

        ppo = importlib.import_module("autocurricula.agents.ppo")
        logits = self.logits(obs)
        B = logits.shape[0]
        actions = logits.argmax(axis=-1).astype(np.int64) if greedy else self.R.rollout.sample_actions(logits, g)
        logp = ppo.log_softmax_np(logits)[np.arange(B), actions]
        view = obs["view"].astype(np.int64).reshape(B, -1)
        d = obs["dir"].astype(np.int64)
        values = 0.125 * (view.sum(axis=1) % 11) + 0.5 * d
        hidden = hidden + np.stack([np.ones(B), d.astype(np.float64)], axis=1)
        return actions, logp, values, hidden


def gen_policy(R):
    """agents/rollout.py:145-152 sample_actions, agents/ppo.py:136 log_softmax_np, and a
    full agents/rollout.py:87 rollout() with an exact actor (RESAMPLE, 64 lanes x 40)."""
    import importlib

    ppo = importlib.import_module("autocurricula.agents.ppo")
    rng = np.random.default_rng(7)
    out = {}
    for tag, A, scale, f32 in (("a3f32", 3, 2.0, True), ("a3", 3, 1.0, False), ("a5", 5, 3.0, False),
                               ("a8", 8, 2.0, False), ("a11", 11, 4.0, False), ("wide", 3, 300.0, False)):
        T, B = 4, 400
        lg = rng.normal(0, scale, (T, B, A))
        if f32:
            lg = lg.astype(np.float32).astype(np.float64)
        lg[:, :10] = np.round(lg[:, :10])  # ties
        acts = np.stack([R.rollout.sample_actions(lg[t], R.rng.RngStream.from_seed(31).fold_in(t).generator())
                         for t in range(T)])
        out[f"pa_{tag}_logits"] = lg
        out[f"pa_{tag}_actions"] = acts
        out[f"pa_{tag}_logp"] = np.stack([ppo.log_softmax_np(lg[t]) for t in range(T)])
    P = R.env.StaticParams()
    for tag, greedy in (("pr", False), ("prg", True)):
        benv = R.env.VectorBatchEnv(R.amaze.MazeEnv(), R.env.BatchShape(1, 1, 64))
        wrap = R.env.AutoResetWrapper(benv, R.env.RESAMPLE)
        start = wrap.reset(R.rng.RngStream.from_seed(9), P)
        traj, cur = R.rollout.rollout(R.rng.RngStream.from_seed(5), _ExactActor(R), wrap, start, 40, P, greedy=greedy)
        out.update({f"{tag}_view": traj.obs["view"], f"{tag}_dir": traj.obs["dir"], f"{tag}_actions": traj.actions,
                    f"{tag}_log_probs": traj.log_probs, f"{tag}_values": traj.values, f"{tag}_rewards": traj.rewards,
                    f"{tag}_dones": traj.dones, f"{tag}_pre_hidden": traj.pre_hidden,
                    f"{tag}_cur_view": cur.obs["view"], f"{tag}_cur_dir": cur.obs["dir"],
                    f"{tag}_cur_hidden": cur.hidden})
    return out


def gen_teacher(R):
    """amaze/teacher.py via batch_lift (GenericBatchEnv): random design episodes plus the
    decoded levels; cases 13x13 budget 60 and 9x9 budget 5 (dense aiming -> agent wraps)."""
    import importlib

    teacher = importlib.import_module("autocurricula.amaze.teacher")
    out = {}
    for tag, H, W, budget, seed, B in (("t13", 13, 13, 60, 41, 48), ("t9", 9, 9, 5, 42, 64)):
        P = R.env.StaticParams(height=H, width=W, wall_budget=budget)
        env = R.env.batch_lift(teacher.TeacherEnv(), R.env.BatchShape(2, 1, B // 2))
        res = env.reset(R.rng.RngStream.from_seed(seed), P)
        T = teacher.TeacherEnv().episode_length(P)
        g = np.random.default_rng(seed)
        ni = P.n_interior
        acts, grids, phases, nps, dones, times = [], [], [], [], [], []
        state = res.state
        grids.append(res.observation["grid"]); phases.append(res.observation["phase"])
        nps.append(res.observation["n_placed"])
        for t in range(T):
            # aim at few cells so the no-op / wall-clearing / agent-wrap rules all fire
            a = g.integers(0, ni if t % 3 else min(ni, 9), size=(2, B // 2))
            r = env.step(None, state, a, P)
            state = r.state
            acts.append(a); grids.append(r.observation["grid"]); phases.append(r.observation["phase"])
            nps.append(r.observation["n_placed"]); dones.append(r.done); times.append(r.info["time"])
        levels = [env.env.designed_level(s) for s in state]
        out.update({f"{tag}_meta": np.array([H, W, budget, seed, B], dtype=np.int64),
                    f"{tag}_actions": np.stack(acts), f"{tag}_grid": np.stack(grids), f"{tag}_phase": np.stack(phases),
                    f"{tag}_n_placed": np.stack(nps), f"{tag}_done": np.stack(dones), f"{tag}_time": np.stack(times),
                    f"{tag}_levels": pack(levels, H, W)})
    return out


def gen_codec(R):
    """amaze/level.py:83-145: encode_level texts of the shipped assets and DR levels, and
    the LevelParseError (message, line, col) the reference raises on malformed texts."""
    lv_mod = R.amaze.level if hasattr(R.amaze, "level") else __import__("autocurricula.amaze.level", fromlist=["x"])
    names = R.amaze.asset_names()
    levels = [R.amaze.load_asset(n) for n in names]
    P = R.env.StaticParams()
    root = R.rng.RngStream.from_seed(77)
    levels += [R.amaze.sample_random_level(k, P) for k in root.split(20)]
    texts = [lv_mod.encode_level(lv) for lv in levels]
    bad = ["", "\n\n", "#####\n#.G.#\n####\n", "#####\n#^G.#\n#####\n", "#####\n#^Gx#\n#####\n",
           "#####\n#^G^#\n#####\n", "#####\n#GG>#\n#####\n", "#####\n#...#\n#####\n", "#####\n#.^.#\n#####\n",
           "#####\n#.^.G\n#####\n", "#####\n\n#^.G#\n\n#####\n", "######\n#^..G#\n######\n"]
    errs = []
    for t in bad:
        try:
            lv_mod.decode_level(t, expected_shape=(3, 5) if t.startswith("######") else None)
            errs.append(("ok", 0, 0))
        except Exception as e:  # noqa: BLE001 - recorded verbatim
            errs.append((str(e), getattr(e, "line", 0), getattr(e, "col", 0)))
    return {"codec_levels": pack(levels, 13, 13), "codec_texts": np.array(texts), "codec_bad": np.array(bad),
            "codec_bad_msg": np.array([e[0] for e in errs]), "codec_bad_line": np.array([e[1] for e in errs]),
            "codec_bad_col": np.array([e[2] for e in errs])}


def main():
    if "--only-codec" in sys.argv:
        np.savez_compressed(os.path.join(OUT, "codec.npz"), **gen_codec(_import_reference()))
        return
    if "--only-teacher" in sys.argv:
        np.savez_compressed(os.path.join(OUT, "teacher.npz"), **gen_teacher(_import_reference()))
        return
    if "--only-policy" in sys.argv:
        np.savez_compressed(os.path.join(OUT, "policy.npz"), **gen_policy(_import_reference()))
        return
    if "--only-metrics" in sys.argv:
        np.savez_compressed(os.path.join(OUT, "metrics.npz"), **gen_metrics(_import_reference()))
        return
    R = _import_reference()
    fx = {}
    fx.update(gen_levels(R))
    np.savez_compressed(os.path.join(OUT, "levels.npz"), **fx)
    ro = {}
    ro.update(gen_rollout(R, "cfg1", (1, 1, 32), "resample", 256, 0, 1))
    ro.update(gen_rollout(R, "hier", (2, 3, 4), "resample", 300, 7, 8))
    ro.update(gen_rollout(R, "occl", (1, 1, 48), "resample", 260, 11, 12, see_through=False))
    assets = [R.amaze.load_asset(n) for n in R.amaze.asset_names()]
    ro.update(gen_rollout(R, "home", (1, 2, 10), "home", 300, 5, 6, levels_from=assets))
    np.savez_compressed(os.path.join(OUT, "rollouts.npz"), **ro)
    np.savez_compressed(os.path.join(OUT, "scores.npz"), **gen_scores(R))
    misc = {}
    misc.update(gen_assets(R))
    misc.update(gen_states(R))
    np.savez_compressed(os.path.join(OUT, "views.npz"), **misc)
    np.savez_compressed(os.path.join(OUT, "metrics.npz"), **gen_metrics(R))
    np.savez_compressed(os.path.join(OUT, "policy.npz"), **gen_policy(R))
    np.savez_compressed(os.path.join(OUT, "teacher.npz"), **gen_teacher(R))
    np.savez_compressed(os.path.join(OUT, "codec.npz"), **gen_codec(R))
    for f in ("levels", "rollouts", "scores", "views"):
        print(f, os.path.getsize(os.path.join(OUT, f + ".npz")))


if __name__ == "__main__":
    main()
