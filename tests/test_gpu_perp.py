"""PLR-perp / ACCEL-perp iterations vs the sequential oracle, the
parallel == sequential two-phase buffer equivalence, and the
buffer digest / checkpoint guards."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import amaze_np as onp  # noqa: E402
from oracle import plr_np  # noqa: E402
from tests.helpers import records_to_rows, tensor_rows  # noqa: E402

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, LevelBuffer, PlrConfig  # noqa: E402
from paper_2311_12716_b200.level import records_to_tensor  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR, SequentialPLR  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _assert_same(gpu: LevelBuffer, ref: plr_np.LevelBuffer):
    st = gpu.export()
    size, nxt = (int(x) for x in st["meta"].cpu())
    assert size == ref.size and nxt == ref.next_seq
    lv, sc, mx, ls, sq = ref.snapshot()
    assert np.array_equal(tensor_rows(st["levels"][:size]), records_to_rows(lv))
    assert np.array_equal(st["score"][:size].cpu().numpy(), sc)
    assert np.array_equal(st["max_return"][:size].cpu().numpy(), mx)
    assert np.array_equal(st["last_sampled"][:size].cpu().numpy(), ls)
    assert np.array_equal(st["seq"][:size].cpu().numpy(), sq)


def _oracle_rollout_score(inputs, gamma, lam, score_fn):
    """rollout_score callback for plr_np.plr_perp_iteration: HOME rollout of the packed
    levels with the harness's action/value streams, GAE + lane scores."""
    p = onp.Params()

    def run(levels, prior, reset_key, which):
        acts, values, last = inputs[which]
        L = len(levels)
        env = onp.AutoReset(L, p, "home")
        obs = env.reset_to_levels(inputs["seed"], reset_key, onp.unpack_levels(levels, p))
        _, _, rew, dn, _ = onp.rollout(env, obs, acts)
        adv, _ = onp.gae(rew, values, dn, last, gamma, lam)
        sc, mx, _ = onp.lane_scores(values, adv, rew, dn, prior, score_fn)
        return sc, mx

    return run


@pytest.mark.parametrize("accel", [None, (4, 20)])
@pytest.mark.parametrize("score_fn", ["maxmc", "pvl"])
def test_perp_iterations_match_oracle(accel, score_fn):
    n, T, K, seed = 40, 32, 48, 13
    gamma, lam = 0.999, 0.98
    cfg = PlrConfig(buffer_size=K, score_fn=score_fn, replay_rate=0.6, staleness_coef=0.3)
    ocfg = plr_np.PlrConfig(buffer_size=K, score_fn=score_fn, replay_rate=0.6, staleness_coef=0.3)
    plr = SequentialPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(seed),
                        AccelConfig(accel[1], accel[0]) if accel else None, gamma=gamma, lam=lam)
    ref = plr_np.LevelBuffer(K)
    rng = np.random.default_rng(2)
    branches = []
    for it in range(10):
        acts = rng.integers(0, 3, (T, n)).astype(np.uint8)
        values = rng.uniform(0, 0.3, (T, n))
        last = rng.uniform(0, 0.3, n)
        q = accel[0] if accel else 1
        macts, mvals, mlast = (rng.integers(0, 3, (T, q)).astype(np.uint8), rng.uniform(0, 0.3, (T, q)),
                               rng.uniform(0, 0.3, q))
        res = plr.iteration(it, torch.from_numpy(acts).cuda(), torch.from_numpy(values).cuda(),
                            torch.from_numpy(last).cuda(),
                            mutant_inputs=tuple(torch.from_numpy(x).cuda() for x in (macts, mvals, mlast)))
        inputs = {"seed": seed, "main": (acts, values, last), "mutants": (macts, mvals, mlast)}
        want = plr_np.plr_perp_iteration(ref, seed, (), it, n, onp.Params(), ocfg,
                                         _oracle_rollout_score(inputs, gamma, lam, score_fn), accel)
        branches.append(res.branch)
        assert res.branch == want["branch"]
        assert np.array_equal(tensor_rows(res.levels), records_to_rows(want["levels"]))
        assert np.array_equal(res.scores.cpu().numpy(), want["scores"])
        assert np.array_equal(res.max_returns.cpu().numpy(), want["max_returns"])
        if res.branch == "replay":
            assert np.array_equal(res.slots.cpu().numpy(), want["slots"])
            if accel:
                assert res.mutants.shape[0] == accel[0]  # exactly q mutants per replay
                assert np.array_equal(tensor_rows(res.mutants), records_to_rows(want["mutants"]))
                assert np.array_equal(res.mutant_scores.cpu().numpy(), want["mutant_scores"])
        _assert_same(plr.buffer, ref)
    assert branches[0] == "new" and "replay" in branches and branches.count("new") >= 2


def _copy_buffer(src: LevelBuffer, cfg) -> LevelBuffer:
    b = LevelBuffer(cfg)
    b.load(src.export())
    return b


@pytest.mark.parametrize("accel", [False, True])
def test_parallel_equals_sequential_two_phase(accel):
    """the PLR|| buffer equals sequential two-phase PLR-perp processing of
    the same candidate sets (NEW phase: the new lanes' candidates; REPLAY phase: the
    replay lanes' (and mutants') candidates) with the same draw."""
    n, T, K, seed = 300, 24, 400, 3
    cfg = PlrConfig(buffer_size=K, staleness_coef=0.5, replay_rate=0.5)
    plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(seed), AccelConfig(20, 4) if accel else None)
    rng = np.random.default_rng(4)
    for it in range(5):
        L = plr.L
        acts = torch.from_numpy(rng.integers(0, 3, (T, L)).astype(np.uint8)).cuda()
        vals = torch.from_numpy(rng.uniform(0, 0.3, (T, L))).cuda()
        last = torch.from_numpy(rng.uniform(0, 0.3, L)).cuda()
        before = _copy_buffer(plr.buffer, cfg)
        res = plr.iteration(it, acts, vals, last)
        seq = before
        if res.n_replay:
            seq.sample(plr.root.fold_in(it).fold_in(2), n, it)  # the same draw marks last_sampled
        parts = [(0, n), (n, plr.L)] if res.n_replay else [(0, plr.L)]
        for a, b in parts:  # phase NEW, then phase REPLAY (+ mutants)
            seq.update(res.levels[a:b], res.scores[a:b], res.max_returns[a:b], it)
        got, want = plr.buffer.export(), seq.export()
        for k in got:
            assert torch.equal(got[k], want[k]), (it, k)
        assert torch.equal(plr.buffer.digest(), seq.digest())


def test_digest_and_checkpoint_guards():
    cfg = PlrConfig(buffer_size=64)
    a = LevelBuffer(cfg)
    lv = amz.sample_levels(amz.RngStream(3, (0,)), 80, amz.StaticParams())
    sc = torch.rand(80, dtype=torch.float64, device="cuda")
    a.update(lv, sc, sc, 2)
    b = _copy_buffer(a, cfg)
    assert torch.equal(a.digest(), b.digest())
    st = b.export()
    st["max_return"][5] += 0.5
    b.load(st)
    assert not torch.equal(a.digest(), b.digest())
    bad = a.export()
    bad["meta"][0] = 65
    with pytest.raises(amz.ContractViolation):
        b.load(bad)
    bad = a.export()
    bad["seq"][3] = bad["seq"][4]
    with pytest.raises(amz.ContractViolation):
        b.load(bad)
    bad = a.export()
    bad["seq"][3] = int(bad["meta"][1])
    with pytest.raises(amz.ContractViolation):
        b.load(bad)


def test_wide_tie_keys_beyond_32_bits():
    """last_sampled / seq beyond 2^32 (long runs, imported checkpoints) keep the oracle's
    (score, last_sampled, seq) eviction order: no 32-bit truncation."""
    K = 8
    cfg = PlrConfig(buffer_size=K)
    gpu = LevelBuffer(cfg)
    ref = plr_np.LevelBuffer(K)
    p = onp.Params()
    recs = onp.pack_levels([onp.sample_level(5, (0, i), p) for i in range(40)], p)
    big = 1 << 33
    # fill with equal scores at iterations straddling 2^32, then evict by ties
    for j, it in enumerate([big - 3, 5, big + 7, (1 << 32) + 1]):
        sl = slice(2 * j, 2 * j + 2)
        sc = np.array([0.25, 0.25])
        gpu.update(records_to_tensor(recs[sl]), torch.from_numpy(sc), torch.from_numpy(sc), it)
        ref.update(recs[sl], sc, sc, it)
    _assert_same(gpu, ref)
    sc = np.full(6, 0.5)
    gpu.update(records_to_tensor(recs[20:26]), torch.from_numpy(sc), torch.from_numpy(sc), big + 9)
    ref.update(recs[20:26], sc, sc, big + 9)
    _assert_same(gpu, ref)


def test_reset_lanes_index_rules():
    p = amz.StaticParams()
    benv = amz.VectorBatchEnv(amz.MazeEnv(), amz.BatchShape(1, 1, 6))
    res = benv.reset(amz.RngStream(8, (0,)), p)
    fresh = amz.sample_levels(amz.RngStream(9, (0,)), 2, p)
    st, _ = benv.reset_lanes(res.state, [-1, 0], fresh, p)  # negative wraps like numpy
    lv = benv.lane_levels_tensor(st)
    assert torch.equal(lv[5], fresh[0]) and torch.equal(lv[0], fresh[1])
    mask = torch.tensor([False, True, False, False, True, False])
    st, _ = benv.reset_lanes(res.state, mask, fresh, p)  # bool mask selects its True lanes
    lv = benv.lane_levels_tensor(st)
    assert torch.equal(lv[1], fresh[0]) and torch.equal(lv[4], fresh[1])
    with pytest.raises(IndexError):
        benv.reset_lanes(res.state, [0, 6], fresh, p)
    with pytest.raises(IndexError):
        benv.reset_lanes(res.state, [-7, 0], fresh, p)
