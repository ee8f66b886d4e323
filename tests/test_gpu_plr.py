"""CUDA PLR buffer / sampler / parallel PLR-ACCEL iterations vs the sequential oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import amaze_np as onp  # noqa: E402
from oracle import plr_np  # noqa: E402
from tests.helpers import records_to_rows, tensor_rows  # noqa: E402

import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200.buffer import AccelConfig, LevelBuffer, PlrConfig, top_q  # noqa: E402
from paper_2311_12716_b200.errors import ContractViolation  # noqa: E402
from paper_2311_12716_b200.level import records_to_tensor  # noqa: E402
from paper_2311_12716_b200.plr import ParallelPLR  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _pool(n, seed=0):
    p = onp.Params()
    return onp.pack_levels([onp.sample_level(seed, (0, i), p) for i in range(n)], p)


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


@pytest.mark.parametrize("K,n,pool", [(2, 3, 4), (16, 40, 60), (100, 300, 500), (4000, 8192, 12000)])
def test_update_tie_heavy_matches_oracle(K, n, pool):
    rng = np.random.default_rng(K)
    recs = _pool(pool, seed=K)
    gpu = LevelBuffer(PlrConfig(buffer_size=K))
    ref = plr_np.LevelBuffer(K)
    for it in range(6):
        idx = rng.integers(0, pool, n)  # in-batch twins and buffer duplicates
        sc = rng.choice([0.0, 0.0, 0.0, -0.0, 0.05, 0.1, 0.1, 0.3, 0.7], n) + (it % 2) * rng.choice([0.0, 1e-3], n)
        mx = rng.uniform(0, 1, n)
        gpu.update(records_to_tensor(recs[idx]), torch.from_numpy(sc), torch.from_numpy(mx), it)
        ref.update(recs[idx], sc, mx, it)
        _assert_same(gpu, ref)


@pytest.mark.parametrize("K", [64, 500, 4000])
def test_update_inplace_runs_then_inserts(K):
    """Long runs of in-place updates (the PLR/ACCEL replay lanes) followed by inserts and
    evictions: the deferred heap repair must leave the same buffer as the sequential oracle."""
    rng = np.random.default_rng(K + 1)
    pool = 3 * K + 400
    recs = _pool(pool, seed=K + 1)
    gpu = LevelBuffer(PlrConfig(buffer_size=K))
    ref = plr_np.LevelBuffer(K)
    vals = [0.0, 0.0, -0.0, 0.05, 0.1, 0.1, 0.3, 0.7]
    keys = {r.tobytes(): i for i, r in enumerate(records_to_rows(recs))}
    for it in range(5):
        if it == 0:
            idx = rng.permutation(pool)[:K]
        else:
            lv, *_ = ref.snapshot()
            present = np.array([keys[r.tobytes()] for r in records_to_rows(lv)])
            runs = [rng.choice(present, K // 2 + 40),                 # in-place run (with twins)
                    rng.integers(0, pool, K // 4 + 33),               # new / mixed
                    rng.choice(present, 64),                          # another run
                    rng.integers(0, pool, 50)]
            idx = np.concatenate(runs)
        n = len(idx)
        sc = rng.choice(vals, n) + (it % 2) * rng.choice([0.0, 1e-3], n)
        mx = rng.uniform(0, 1, n)
        gpu.update(records_to_tensor(recs[idx]), torch.from_numpy(sc), torch.from_numpy(mx), it)
        ref.update(recs[idx], sc, mx, it)
        _assert_same(gpu, ref)


@pytest.mark.parametrize("K", [300, 4000])
def test_update_bulk_run_boundaries(K):
    """In-place runs of lengths around the bulk threshold (63/64/65 ...) separated by single
    inserts, with in-place scores that often drop below the minimum so the next insert
    evicts an entry the run just rewrote (bulk heap rebuild vs sequential sifts)."""
    rng = np.random.default_rng(K + 7)
    pool = 3 * K + 400
    recs = _pool(pool, seed=K + 7)
    gpu = LevelBuffer(PlrConfig(buffer_size=K))
    ref = plr_np.LevelBuffer(K)
    keys = {r.tobytes(): i for i, r in enumerate(records_to_rows(recs))}
    for it in range(4):
        if it == 0:
            idx = rng.permutation(pool)[:K]
        else:
            lv, *_ = ref.snapshot()
            present = np.array([keys[r.tobytes()] for r in records_to_rows(lv)])
            parts = []
            for L in [63, 64, 65, 1, 0, 128, 31, 64, 900, 2, 64, 1100]:
                parts.append(rng.choice(present, L))
                parts.append(rng.integers(0, pool, 1 + (L % 3)))
            idx = np.concatenate(parts)
        n = len(idx)
        sc = rng.choice([0.0, 0.01, 0.2, 0.5, 0.9], n) + rng.choice([0.0, 1e-3], n)
        mx = rng.uniform(0, 1, n)
        gpu.update(records_to_tensor(recs[idx]), torch.from_numpy(sc), torch.from_numpy(mx), it)
        ref.update(recs[idx], sc, mx, it)
        _assert_same(gpu, ref)


def test_spec_update_example():
    recs = _pool(3)
    gpu = LevelBuffer(PlrConfig(buffer_size=2))
    gpu.update(records_to_tensor(recs), torch.tensor([5.0, 1.0, 3.0]), torch.zeros(3), 0)
    st = gpu.export()
    assert sorted(st["score"][:2].cpu().tolist()) == [3.0, 5.0]


@pytest.mark.parametrize("K,rho,beta", [(5, 0.3, 0.3), (100, 0.0, 1.0), (4000, 0.3, 0.3), (4000, 0.5, 0.3),
                                        (777, 1.0, 0.5)])
def test_sample_matches_numpy_choice(K, rho, beta):
    rng = np.random.default_rng(K)
    recs = _pool(K + 50, seed=1)
    cfg = PlrConfig(buffer_size=K, staleness_coef=rho, temperature=beta)
    gpu = LevelBuffer(cfg)
    ref = plr_np.LevelBuffer(K)
    for it in range(3):
        idx = rng.permutation(K + 50)[:K]
        sc = rng.choice([0.0, 0.2, 0.2, 0.4, 0.9], K) * rng.uniform(0.5, 1, K)
        gpu.update(records_to_tensor(recs[idx]), torch.from_numpy(sc), torch.from_numpy(sc), it)
        ref.update(recs[idx], sc, sc, it)
    ocfg = plr_np.PlrConfig(buffer_size=K, staleness_coef=rho, temperature=beta)
    for it in range(3, 7):
        out = gpu.sample(amz.RngStream(11, (it, 2)), 2048, it)
        want = ref.sample(11, (it, 2), 2048, ocfg, it)
        assert np.array_equal(out["slots"].cpu().numpy(), want)
        lv = ref.levels[want]
        assert np.array_equal(tensor_rows(out["levels"]), records_to_rows(lv))
        assert np.array_equal(out["scores"].cpu().numpy(), ref.score[want])
    _assert_same(gpu, ref)


@pytest.mark.parametrize("K,rho,beta", [(100, 0.0, 0.3), (4000, 0.3, 0.3), (777, 0.5, 1.0)])
def test_sample_proportional_matches_numpy_choice(K, rho, beta):
    """SPEC.md:367 proportional prioritisation: P_S ~ score^(1/beta).  The weights come
    from CUDA's pow (within 2 ulp of numpy's np.power), so the probabilities are checked
    to 1e-13 relative and the draws for equality (a uniform would have to land inside
    that rounding of a cdf boundary to differ)."""
    rng = np.random.default_rng(K + 1)
    recs = _pool(K + 50, seed=2)
    cfg = PlrConfig(buffer_size=K, staleness_coef=rho, temperature=beta, prioritization="proportional")
    gpu = LevelBuffer(cfg)
    ref = plr_np.LevelBuffer(K)
    for it in range(3):
        idx = rng.permutation(K + 50)[:K]
        sc = rng.choice([0.0, 0.2, 0.2, 0.4, 0.9], K) * rng.uniform(0.5, 1, K)
        gpu.update(records_to_tensor(recs[idx]), torch.from_numpy(sc), torch.from_numpy(sc), it)
        ref.update(recs[idx], sc, sc, it)
    ocfg = plr_np.PlrConfig(buffer_size=K, staleness_coef=rho, temperature=beta, prioritization="proportional")
    w_gpu = torch.pow(torch.from_numpy(ref.score[:ref.size]).cuda(), 1.0 / beta).cpu().numpy()
    w_np = np.power(ref.score[:ref.size], 1.0 / beta)
    assert np.allclose(w_gpu, w_np, rtol=1e-13, atol=0)
    for it in range(3, 7):
        out = gpu.sample(amz.RngStream(13, (it, 2)), 2048, it)
        want = ref.sample(13, (it, 2), 2048, ocfg, it)
        assert np.array_equal(out["slots"].cpu().numpy(), want)
        assert np.array_equal(out["scores"].cpu().numpy(), ref.score[want])
    _assert_same(gpu, ref)


def test_sample_proportional_rejects_nan_probabilities():
    cfg = PlrConfig(buffer_size=16, prioritization="proportional")
    gpu = LevelBuffer(cfg)
    recs = _pool(16, seed=3)
    gpu.update(records_to_tensor(recs), torch.full((16,), -0.5, dtype=torch.float64), torch.zeros(16, dtype=torch.float64), 0)
    gpu.sample(amz.RngStream(1, (0,)), 8, 1)
    with pytest.raises(ContractViolation):
        gpu.size()


def test_top_q():
    rng = np.random.default_rng(0)
    s = rng.choice([0.0, 0.5, 0.5, 1.0, 0.25], 1000)
    got = top_q(torch.from_numpy(s).cuda(), 4).cpu().numpy()
    assert np.array_equal(got, plr_np.top_q(s, 4))


def _oracle_iteration(buf, seed, it, n, accel, cfg, acts, values, last):
    p = onp.Params()
    levels, prior, n_rep, _ = plr_np.compose_lanes(buf, seed, (), it, n, p, cfg, accel)
    L = len(levels)
    env = onp.AutoReset(L, p, "home")
    obs = env.reset_to_levels(seed, (it, 4), onp.unpack_levels(levels, p))
    view, dirs, rew, dn, _ = onp.rollout(env, obs, acts)
    adv, _ = onp.gae(rew, values, dn, last, 0.995, 0.95)
    sc, mx, _ = onp.lane_scores(values, adv, rew, dn, prior, cfg.score_fn)
    buf.update(levels, sc, mx, it)
    return levels, sc, mx, n_rep


@pytest.mark.parametrize("accel", [None, (4, 20)])
@pytest.mark.parametrize("score_fn", ["maxmc", "pvl"])
def test_parallel_iterations_match_oracle(accel, score_fn):
    n, T, K, seed = 48, 40, 64, 5
    cfg = PlrConfig(buffer_size=K, score_fn=score_fn)
    ocfg = plr_np.PlrConfig(buffer_size=K, score_fn=score_fn)
    plr = ParallelPLR(n, amz.StaticParams(), cfg, amz.RngStream.from_seed(seed),
                      AccelConfig(accel[1], accel[0]) if accel else None)
    ref = plr_np.LevelBuffer(K)
    rng = np.random.default_rng(1)
    L = plr.L
    for it in range(5):
        acts = rng.integers(0, 3, (T, L)).astype(np.uint8)
        values = rng.uniform(0, 0.3, (T, L))
        last = rng.uniform(0, 0.3, L)
        res = plr.iteration(it, torch.from_numpy(acts).cuda(), torch.from_numpy(values).cuda(),
                            torch.from_numpy(last).cuda())
        lv, sc, mx, n_rep = _oracle_iteration(ref, seed, it, n, accel, ocfg, acts, values, last)
        assert res.n_replay == n_rep
        assert np.array_equal(tensor_rows(res.levels), records_to_rows(lv))
        assert np.array_equal(res.scores.cpu().numpy(), sc)
        assert np.array_equal(res.max_returns.cpu().numpy(), mx)
        _assert_same(plr.buffer, ref)


def test_string_device_arguments():
    """device="cuda:0" strings resolve to the right stream (str has an .index method too)."""
    lv = amz.sample_levels(amz.RngStream(3, (0,)), 64, amz.StaticParams(), device="cuda:0")
    ref = amz.sample_levels(amz.RngStream(3, (0,)), 64, amz.StaticParams(), device=torch.device("cuda", 0))
    assert torch.equal(lv, ref)
    buf = LevelBuffer(PlrConfig(buffer_size=16), device="cuda:0")
    buf.update(lv, torch.rand(64, dtype=torch.float64), torch.zeros(64, dtype=torch.float64), 1)
    out = buf.sample(amz.RngStream(5, (0,)), 8, 2)
    assert out["slots"].shape == (8,) and int(out["slots"].max()) < 16


@pytest.mark.parametrize("K,n,digits", [(64, 200, 1), (500, 1500, 2), (4000, 4096, 3), (4000, 6000, 1), (1000, 3000, 16)])
def test_update_insert_runs_match_oracle(K, n, digits):
    """Mostly-new candidates (the parallel insert-run path): fills, evictions, evictions of
    entries inserted earlier in the same batch, rounded scores so candidates often tie the
    running minimum (the run stops and the tie goes through the sequential rule), a few
    twins and replays mixed in, and replay marks (last_sampled = iter) between updates."""
    rng = np.random.default_rng(K + n + digits)
    pool = _pool(3 * n + 64, seed=digits)
    gpu = LevelBuffer(PlrConfig(buffer_size=K))
    ref = plr_np.LevelBuffer(K)
    nxt = 0
    for it in range(5):
        idx = np.arange(nxt, nxt + n) % len(pool)
        nxt += n
        dup = rng.uniform(size=n) < 0.03  # a few twins / buffered levels
        idx[dup] = rng.integers(0, len(pool), int(dup.sum()))
        sc = np.round(rng.uniform(0, 1, n), digits)
        sc[rng.uniform(size=n) < 0.1] = 0.0
        mx = rng.uniform(0, 1, n)
        gpu.update(records_to_tensor(pool[idx]), torch.from_numpy(sc), torch.from_numpy(mx), it)
        ref.update(pool[idx], sc, mx, it)
        _assert_same(gpu, ref)
        if ref.size:
            out = gpu.sample(amz.RngStream(3, (it,)), 64, it)
            want = ref.sample(3, (it,), 64, plr_np.PlrConfig(buffer_size=K), it)
            assert np.array_equal(out["slots"].cpu().numpy(), want)
            _assert_same(gpu, ref)


def test_prepare_then_update_matches_oracle():
    """amz_plr_prepare on a side stream, then the update with the same batch, equals the
    oracle; a prepared batch is consumed once and ignored by an update with another batch."""
    K, n = 200, 600
    rng = np.random.default_rng(7)
    recs = _pool(900, seed=7)
    gpu = LevelBuffer(PlrConfig(buffer_size=K))
    ref = plr_np.LevelBuffer(K)
    side = torch.cuda.Stream()
    for it in range(6):
        idx = rng.integers(0, len(recs), n)
        sc = rng.choice([0.0, 0.1, 0.2, 0.5], n)
        mx = rng.uniform(0, 1, n)
        lv = records_to_tensor(recs[idx]).cuda()
        if it % 3 == 2:  # prepared for a different batch: must not be used
            other = records_to_tensor(recs[rng.integers(0, len(recs), n)]).cuda()
            gpu.prepare(other)
        else:
            side.wait_stream(torch.cuda.current_stream())
            gpu.prepare(lv, stream=side)
            torch.cuda.current_stream().wait_stream(side)
        gpu.update(lv, torch.from_numpy(sc), torch.from_numpy(mx), it)
        ref.update(recs[idx], sc, mx, it)
        _assert_same(gpu, ref)
    with pytest.raises(ContractViolation):
        gpu.prepare(lv.to(torch.int64))
