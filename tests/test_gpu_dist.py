"""Parallel PLR/ACCEL with 2 ranks on one GPU (gloo carries the candidate records):
every rank's lanes, scores and replicated buffer equal the 1-rank run lane for lane
(SPEC.md:400-417), and the drift check (on-device digest +
all-reduce) passes on equal replicas and fires on a diverged one."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_NEW, T, K, SEED, ITERS = 24, 24, 40, 9, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(L):
    rng = np.random.default_rng(17)
    out = []
    for _ in range(ITERS):
        out.append((rng.integers(0, 3, (T, L)).astype(np.uint8), rng.uniform(0, 0.3, (T, L)), rng.uniform(0, 0.3, L)))
    return out


def _make(accel):
    import paper_2311_12716_b200 as amz
    from paper_2311_12716_b200.buffer import AccelConfig, PlrConfig
    from paper_2311_12716_b200.plr import ParallelPLR

    cfg = PlrConfig(buffer_size=K, score_fn="maxmc", staleness_coef=0.5, replay_rate=0.8)
    return ParallelPLR(N_NEW, amz.StaticParams(), cfg, amz.RngStream.from_seed(SEED),
                       AccelConfig(20, 4) if accel else None, device="cuda:0", check_every=2)


def _run(plr):
    L = plr.L
    res = []
    for it, (a, v, l) in enumerate(_inputs(L)):
        sl = slice(plr.lo, plr.hi)
        r = plr.iteration(it, torch.from_numpy(a[:, sl].copy()).cuda(), torch.from_numpy(v[:, sl].copy()).cuda(),
                          torch.from_numpy(l[sl].copy()).cuda())
        res.append((r.levels.cpu().numpy(), r.scores.cpu().numpy(), r.max_returns.cpu().numpy()))
    st = {k: v.cpu().numpy() for k, v in plr.buffer.export().items()}
    return res, st


def _worker(rank, world, port, accel, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as tdist

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plr = _make(accel)
        res, st = _run(plr)
        plr.check_replicas()
        q.put(("ok", rank, plr.lo, plr.hi, res, st))
        # a diverged replica must be caught by the drift check
        if rank == 1:
            lv = plr.buffer.export()
            lv["score"][0] += 1.0
            plr.buffer.load(lv)
        try:
            plr.check_replicas()
            q.put(("fault", rank, "none"))
        except Exception as e:  # RunnerFault
            q.put(("fault", rank, type(e).__name__))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("accel", [False, True])
def test_two_ranks_equal_one_rank(accel):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, accel, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    msgs = [q.get(timeout=300) for _ in range(4)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    ok = sorted((m for m in msgs if m[0] == "ok"), key=lambda m: m[1])
    faults = {m[1]: m[2] for m in msgs if m[0] == "fault"}
    assert faults == {0: "RunnerFault", 1: "RunnerFault"}

    one = _make(accel)
    res1, st1 = _run(one)
    for it in range(ITERS):
        for f in range(3):
            got = np.concatenate([ok[0][4][it][f], ok[1][4][it][f]])
            assert np.array_equal(got, res1[it][f]), (it, f)
    for r in range(2):
        for k in st1:
            assert np.array_equal(ok[r][5][k], st1[k]), (r, k)
    assert ok[0][2:4] == (0, one.L // 2) and ok[1][2:4] == (one.L // 2, one.L)


# -- SDP gradient mean on device tensors (agents/ppo.py:308-313) -------------------------
def _grad_model(r):
    torch.manual_seed(100)  # identical initial parameters on every shard
    m = torch.nn.Sequential(torch.nn.Linear(5, 7), torch.nn.Tanh(), torch.nn.Linear(7, 3)).cuda()
    torch.manual_seed(200 + r)  # shard-specific minibatch
    x = (torch.randn(11, 5, dtype=torch.float32) * (r + 1)).cuda()
    m(x).pow(2).sum().backward()
    m[2].bias.grad = None  # a parameter without a gradient counts as zeros
    return m


def _sdp_worker(rank, world, port, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as tdist

    torch.cuda.set_device(0)
    try:
        tdist.init_process_group(backend, rank=rank, world_size=world)
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, False, False, False, repr(e)))
        return
    try:
        from paper_2311_12716_b200 import dist

        out = {}
        for exact in (True, False):
            m = _grad_model(rank)
            dist.sdp_average_gradients(m.parameters(), exact=exact)
            out[exact] = [p.grad.clone() for p in m.parameters()]
        shards = [[p.grad.detach() if p.grad is not None else torch.zeros_like(p) for p in _grad_model(r).parameters()]
                  for r in range(world)]
        want = [sum(g[i] for g in shards) / world for i in range(len(shards[0]))]
        on_dev = all(g.is_cuda for g in out[True] + out[False])
        exact_ok = all(torch.equal(a, b) for a, b in zip(out[True], want))
        close_ok = all(torch.allclose(a, b, rtol=1e-6, atol=1e-7) for a, b in zip(out[False], want))
        drift0 = dist.check_param_sync(_grad_model(rank).parameters())
        q.put((rank, on_dev, exact_ok, close_ok, drift0))
    except Exception as e:
        import traceback

        q.put((rank, False, False, False, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1)])
def test_sdp_gradient_mean_on_device(backend, world):
    """Device gradients: gloo with 2 ranks on the one GPU (host-staged exchange), NCCL with
    the world this box has (1 GPU: the call must be the identity and stay on the device)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sdp_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    msgs = sorted((q.get(timeout=180) for _ in range(world)), key=lambda m: m[0])
    for pr in procs:
        pr.join(timeout=120)
    for rank, on_dev, exact_ok, close_ok, drift0 in msgs:
        assert on_dev and exact_ok and close_ok and drift0 == 0.0, (rank, drift0)
    for pr in procs:
        assert pr.exitcode == 0
