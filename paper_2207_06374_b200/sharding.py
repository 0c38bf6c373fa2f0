"""Multi-GPU trial sharding: one process per GPU, trials are
independent, so the only exchange is the final best-of selection of solve()
(solver.hpp:256-267) — an allgather of (best mu, global trial id) and a
broadcast of the winning frame from its owner.  Pure data movement: every
floating-point value is computed on exactly one rank, so results are
bit-identical for any GPU count.

Works with any torch.distributed backend (NCCL on the GPU box, gloo in the
CPU tests).
"""
import math

import torch
import torch.distributed as dist


def shard(total, world, rank):
    """Contiguous block of global trial ids [lo, hi) for `rank` (trial i goes to
    GPU floor(i * world / total))."""
    lo = (total * rank) // world
    hi = (total * (rank + 1)) // world
    return lo, hi


def local_best(coherences, ok, first):
    """min mu over succeeded local trials, lowest global id on ties
    (solver.hpp:256-263).  Returns (mu, global id) or (inf, -1)."""
    best, bi = math.inf, -1
    for t, (mu, good) in enumerate(zip(coherences, ok)):
        if good and (bi < 0 or mu < best):
            best, bi = mu, first + t
    return best, bi


def global_best(best, best_id, frame, device):
    """Allgather (mu, id) over ranks, pick min mu / lowest id, broadcast the
    owner's frame.  Returns (mu, id, frame) identical on every rank."""
    world = dist.get_world_size()
    cand = torch.tensor([best, float(best_id)], dtype=torch.float64, device=device)
    allc = [torch.empty_like(cand) for _ in range(world)]
    dist.all_gather(allc, cand)
    vals = [(c[0].item(), c[1].item(), r) for r, c in enumerate(allc)]
    ok = [v for v in vals if v[1] >= 0]
    if not ok:
        raise RuntimeError("solve: all restarts failed")
    mu, gid, owner = min(ok, key=lambda v: (v[0], v[1]))
    buf = frame.clone() if dist.get_rank() == owner else torch.empty_like(frame)
    dist.broadcast(buf, src=owner)
    return mu, int(gid), buf
