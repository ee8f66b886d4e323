"""Multi-rank host logic of the parallel PLR path on CPU (gloo, world_size 2).

Each rank builds the candidate records of its lane shard with the oracle, all-gathers
them through paper_2311_12716_b200.dist, applies the (oracle) buffer update and checks
the replicas agree -- the same plumbing the NCCL path runs between GPU kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist_
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist_.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import amaze_np as onp
        from oracle import plr_np
        from paper_2311_12716_b200 import dist

        p = onp.Params()
        L = 24
        lo, hi = dist.shard(L, rank, world)
        # candidate levels keyed by GLOBAL lane index -> identical to a 1-rank run
        recs = onp.pack_levels([onp.sample_level(3, (1, i), p) for i in range(lo, hi)], p)
        lv = torch.from_numpy(np.ascontiguousarray(recs).view(np.int32).reshape(-1, 8).copy())
        sc = torch.tensor([float((i * 7) % 5) / 4 for i in range(lo, hi)], dtype=torch.float64)
        mx = torch.tensor([float(i) / 100 for i in range(lo, hi)], dtype=torch.float64)
        g_lv, g_sc, g_mx = dist.gather_candidates(lv, sc, mx)
        buf = plr_np.LevelBuffer(10)
        buf.update(g_lv.numpy().reshape(-1).view(onp.LEVEL_DTYPE), g_sc.numpy(), g_mx.numpy(), it=0)
        state = {"levels": torch.from_numpy(np.ascontiguousarray(buf.levels).view(np.int32).reshape(-1, 8).copy()),
                 "score": torch.from_numpy(buf.score.copy()), "max_return": torch.from_numpy(buf.max_return.copy()),
                 "last_sampled": torch.from_numpy(buf.last_sampled.copy()), "seq": torch.from_numpy(buf.seq.copy()),
                 "meta": torch.tensor([buf.size, buf.next_seq])}
        dist.check_replicas(dist.buffer_digest(state))
        q.put((rank, g_lv.numpy().tobytes(), g_sc.numpy().tolist(), dist.buffer_digest(state)))
        # a diverged replica must be caught
        if rank == 1:
            state["score"][0] += 1.0
        try:
            dist.check_replicas(dist.buffer_digest(state))
            q.put((rank, "no-fault"))
        except Exception as e:  # RunnerFault
            q.put((rank, type(e).__name__))
    finally:
        dist_.destroy_process_group()


def test_two_rank_candidate_gather_and_replicated_update():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    msgs = [q.get(timeout=120) for _ in range(4)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    data = sorted([m for m in msgs if len(m) == 4])
    faults = sorted([m for m in msgs if len(m) == 2])
    assert data[0][1] == data[1][1] and data[0][2] == data[1][2] and data[0][3] == data[1][3]
    # gathered order == global lane order of a single-rank run
    from oracle import amaze_np as onp

    p = onp.Params()
    want = onp.pack_levels([onp.sample_level(3, (1, i), p) for i in range(24)], p)
    assert data[0][1] == np.ascontiguousarray(want).view(np.int32).tobytes()
    assert [f[1] for f in faults] == ["RunnerFault", "RunnerFault"]


def test_shard_math():
    from paper_2311_12716_b200 import dist
    from paper_2311_12716_b200.errors import ShapeError

    assert [dist.shard(96, r, 4) for r in range(4)] == [(0, 24), (24, 48), (48, 72), (72, 96)]
    with pytest.raises(ShapeError):
        dist.shard(10, 0, 4)


def test_record_pack_roundtrip():
    from paper_2311_12716_b200 import dist

    lv = torch.randint(-2**31, 2**31 - 1, (7, 8), dtype=torch.int32)
    sc = torch.randn(7, dtype=torch.float64)
    mx = torch.randn(7, dtype=torch.float64)
    a, b, c = dist.unpack_candidates(dist.pack_candidates(lv, sc, mx))
    assert torch.equal(a, lv) and torch.equal(b, sc) and torch.equal(c, mx)


def _grad_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist_.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_12716_b200 import dist

        def model_and_grads(r):
            torch.manual_seed(100)  # identical initial parameters on every shard
            m = torch.nn.Sequential(torch.nn.Linear(5, 7), torch.nn.Tanh(), torch.nn.Linear(7, 3))
            torch.manual_seed(200 + r)  # shard-specific minibatch
            x = torch.randn(11, 5, dtype=torch.float32) * (r + 1)
            m(x).pow(2).sum().backward()
            m[2].bias.grad = None  # a parameter without a gradient counts as zeros
            return m

        out = {}
        for exact in (True, False):
            m = model_and_grads(rank)
            dist.sdp_average_gradients(m.parameters(), exact=exact)
            out[exact] = [p.grad.clone() for p in m.parameters()]
        # the reference's in-process mean: sum(g[i] for g in shard_grads) / n_shards
        shards = [[p.grad.detach() if p.grad is not None else torch.zeros_like(p) for p in model_and_grads(r).parameters()]
                  for r in range(world)]
        want = [sum(g[i] for g in shards) / world for i in range(len(shards[0]))]
        exact_ok = all(torch.equal(a, b) for a, b in zip(out[True], want))
        close_ok = all(torch.allclose(a, b, rtol=1e-6, atol=1e-7) for a, b in zip(out[False], want))
        m = model_and_grads(rank)
        drift0 = dist.check_param_sync(m.parameters())
        if rank == 1:
            with torch.no_grad():
                m[0].weight[0, 0] += 1.0
        try:
            dist.check_param_sync(m.parameters())
            fault = "no-fault"
        except Exception as e:  # RunnerFault
            fault = type(e).__name__
        q.put((rank, exact_ok, close_ok, drift0, fault))
    finally:
        dist_.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sdp_gradient_average_matches_reference_mean(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    msgs = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, exact_ok, close_ok, drift0, fault in msgs:
        assert exact_ok and close_ok and drift0 == 0.0 and fault == "RunnerFault"
