"""Multi-GPU plumbing for the parallel PLR/ACCEL hot path.

Lanes shard by global lane index: rank r of D owns global lanes [r*L/D, (r+1)*L/D) of
the iteration's lane layout, and every level key is a function of the global index,
so a D-GPU iteration equals the 1-GPU iteration lane for lane.  The one exchange step
is the candidate records (level 32 B + score f64 + max return f64 = 48 B per lane),
all-gathered in global lane order once per iteration; every rank then applies the same
deterministic buffer update, keeping the buffer replicated.  ``buffer_digest`` +
``check_replicas`` is the drift check (the analogue of the shard-sync check at
agents/ppo.py:323-328).

torch.distributed carries the bytes: NCCL (NVLink/NVSwitch) on GPUs, gloo on CPU for
the host-logic tests.
"""

from __future__ import annotations

import hashlib

from .errors import RunnerFault, ShapeError

RECORD_WORDS = 12  # int32 words per candidate record


def _torch():
    import torch

    return torch


def world():
    torch = _torch()
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        return torch.distributed.get_rank(), torch.distributed.get_world_size()
    return 0, 1


def shard(n_lanes: int, rank: int, world_size: int) -> tuple[int, int]:
    """Global [lo, hi) lane range of ``rank`` (equal shards; L must divide evenly)."""
    if n_lanes % world_size:
        raise ShapeError(f"{n_lanes} lanes do not split evenly over {world_size} ranks")
    per = n_lanes // world_size
    return rank * per, (rank + 1) * per


def pack_candidates(levels, scores, max_returns):
    """[n, 8] int32 levels + f64 scores + f64 max returns -> [n, 12] int32 records."""
    torch = _torch()
    n = levels.shape[0]
    rec = torch.empty((n, RECORD_WORDS), dtype=torch.int32, device=levels.device)
    rec[:, :8] = levels
    rec[:, 8:10] = scores.to(torch.float64).contiguous().view(torch.int32).reshape(n, 2)
    rec[:, 10:12] = max_returns.to(torch.float64).contiguous().view(torch.int32).reshape(n, 2)
    return rec


def unpack_candidates(rec):
    torch = _torch()
    n = rec.shape[0]
    levels = rec[:, :8].contiguous()
    scores = rec[:, 8:10].contiguous().view(torch.float64).reshape(n)
    max_returns = rec[:, 10:12].contiguous().view(torch.float64).reshape(n)
    return levels, scores, max_returns


def all_gather_records(rec):
    """Concatenate every rank's [n, 12] records in rank order (= global lane order)."""
    torch = _torch()
    rank, ws = world()
    if ws == 1:
        return rec
    rec = rec.contiguous()
    if torch.distributed.get_backend() == "nccl":
        out = torch.empty((rec.shape[0] * ws, rec.shape[1]), dtype=rec.dtype, device=rec.device)
        torch.distributed.all_gather_into_tensor(out, rec)
        return out
    # gloo (CPU test worlds, several ranks on one device): gather host copies
    dev = rec.device
    host = rec.cpu()
    parts = [torch.empty_like(host) for _ in range(ws)]
    torch.distributed.all_gather(parts, host)
    return torch.cat(parts).to(dev)


def gather_candidates(levels, scores, max_returns):
    """Every rank's candidates in global lane order; a 1-rank world passes them through
    (no record packing: it cost 6 device copies per iteration)."""
    if world()[1] == 1:
        return levels, scores, max_returns
    return unpack_candidates(all_gather_records(pack_candidates(levels, scores, max_returns)))


def buffer_digest(state: dict) -> int:
    """64-bit digest of a buffer state (valid slots only)."""
    size = int(state["meta"][0].item())
    h = hashlib.blake2b(digest_size=8)
    for k in ("levels", "score", "max_return", "last_sampled", "seq"):
        h.update(state[k][:size].detach().cpu().contiguous().numpy().tobytes())
    h.update(state["meta"].detach().cpu().numpy().tobytes())
    return int.from_bytes(h.digest(), "little") & 0x7FFFFFFFFFFFFFFF


def check_replicas(digest, device=None) -> None:
    """Raise RunnerFault if the ranks' buffers differ: one all-reduce of [d, -d] with MAX
    gives max and -min of the digests in one collective.  ``digest`` is an int or a
    device int64 tensor (``LevelBuffer.digest()``, computed on the GPU; with NCCL it
    never leaves the device until the final comparison)."""
    torch = _torch()
    rank, ws = world()
    if ws == 1:
        return
    nccl = torch.distributed.get_backend() == "nccl"
    if torch.is_tensor(digest):
        d = digest.reshape(1).to(torch.int64)
        dev = d.device if nccl else "cpu"
        d = d.to(dev)
    else:
        dev = device if device is not None and nccl else "cpu"
        d = torch.tensor([int(digest)], dtype=torch.int64, device=dev)
    # -d overflows only for INT64_MIN; the digest is masked to 63 bits first
    d = d & 0x7FFFFFFFFFFFFFFF
    both = torch.cat([d, -d])
    torch.distributed.all_reduce(both, op=torch.distributed.ReduceOp.MAX)
    hi, neg_lo = (int(x) for x in both.cpu())
    if hi != -neg_lo:
        raise RunnerFault(f"PLR buffer replicas diverged (rank {rank})")


# ------------------------------------------------------------------------------------
# SDP gradient averaging for PPO shards (agents/ppo.py:267-330)
# ------------------------------------------------------------------------------------

def _flat(tensors):
    torch = _torch()
    return torch.cat([t.reshape(-1) for t in tensors]) if tensors else torch.zeros(0)


def sdp_average_gradients(params, exact: bool = False, group=None) -> None:
    """Replace every parameter's gradient by the mean over ranks (one rank per shard),
    the in-process shard mean of agents/ppo.py:308-313 (missing gradients count as
    zeros, :260-263).  ``exact=False``: one all-reduce(SUM) of a flat bucket (NCCL over
    NVLink on GPUs), then / D -- identical on every rank.  ``exact=True``: all-gather the
    flat gradients and sum them in rank order from 0 like the reference's Python
    ``sum(...) / n_shards``, bit-identical to the single-process result for any D."""
    torch = _torch()
    dist = torch.distributed
    params = list(params)
    grads = [p.grad.detach() if p.grad is not None else torch.zeros_like(p) for p in params]
    flat = _flat(grads).contiguous()
    D = dist.get_world_size(group)
    if D == 1:  # the mean of one shard; a missing gradient still reads as zeros
        for p, g in zip(params, grads):
            if p.grad is None:
                p.grad = g
        return
    dev = flat.device
    # gloo has no all-gather of device tensors: its worlds (tests, several ranks on one
    # GPU) exchange host copies; the arithmetic stays on the gradients' device
    wire = flat.cpu() if (flat.is_cuda and dist.get_backend(group) == "gloo") else flat
    if exact:
        parts = [torch.empty_like(wire) for _ in range(D)]
        dist.all_gather(parts, wire, group=group)
        acc = torch.zeros_like(flat)
        for part in parts:
            acc = acc + part.to(dev)
        mean = acc / D
    else:
        dist.all_reduce(wire, op=dist.ReduceOp.SUM, group=group)
        mean = wire.to(dev) / D
    off = 0
    with torch.no_grad():
        for p in params:
            n = p.numel()
            p.grad = mean[off:off + n].view_as(p).clone()
            off += n


def check_param_sync(params, tol: float = 1e-6, group=None) -> float:
    """agents/ppo.py:322-328 across ranks: max |params - rank 0's params| (all-reduce
    MAX); raises RunnerFault above ``tol``."""
    torch = _torch()
    dist = torch.distributed
    with torch.no_grad():
        vec = _flat([p.detach().double() for p in params]).contiguous()
        if vec.is_cuda and dist.get_backend(group) == "gloo":
            vec = vec.cpu()  # gloo worlds exchange host copies
        ref = vec.clone()
        dist.broadcast(ref, src=0, group=group)
        drift = (vec - ref).abs().max() if vec.numel() else torch.zeros((), dtype=torch.float64)
        d = drift.reshape(1).clone()
        dist.all_reduce(d, op=dist.ReduceOp.MAX, group=group)
    val = float(d.item())
    if val > tol:
        raise RunnerFault(f"shard parameters diverged by {val:.3e}")
    return val
