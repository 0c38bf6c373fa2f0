"""Multi-GPU trial sharding — Python view of the product's
host logic in csrc/sharding.cu.

One process per GPU; trials are independent, so the only exchange is the
final best-of selection of solve() (solver.hpp:256-267): an allgather of
(best mu, global trial id) and a broadcast of the winning frame from its
owner.  `shard` and `select_best` call the library's own
trstmi_shard_range / trstmi_select_best (pure host functions, no GPU), so
the partition and the tie rule tested here are the ones trstmi_solve_sharded
and trstmi_best_of_ranks run over NCCL on the GPU box.  `global_best` is the
same exchange written with torch.distributed, for backends without the
library's NCCL communicator (the gloo CPU tests).
"""
import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import api


def shard(total, world, rank):
    """Contiguous block [lo, hi) of global trial ids for `rank`: trial i goes
    to rank floor(i * world / total) (trstmi_shard_range)."""
    lib = api.load_library()
    f, c = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.trstmi_shard_range(total, world, rank, ctypes.byref(f), ctypes.byref(c))
    if rc:
        raise ValueError("shard_range: bad arguments")
    return f.value, f.value + c.value


def select_best(mus, ids=None, ok=None):
    """Position of the minimum mu over ok entries (NaN = absent), lowest id on
    ties (trstmi_select_best, solver.hpp:256-263); -1 when none."""
    lib = api.load_library()
    mus = np.ascontiguousarray(mus, np.float64)
    idv = None if ids is None else np.ascontiguousarray(ids, np.int64)
    okv = None if ok is None else np.ascontiguousarray(ok, np.int32)
    pos = ctypes.c_int64()
    p = (lambda a: None if a is None else ctypes.c_void_p(a.ctypes.data))
    lib.trstmi_select_best(mus.size, p(mus), p(idv), p(okv), ctypes.byref(pos))
    return pos.value


def local_best(coherences, ok, first):
    """(mu, global id) of the rank's best trial, or (nan, -1)."""
    pos = select_best(coherences, None, ok)
    if pos < 0:
        return float("nan"), -1
    return float(coherences[pos]), first + pos


def global_best(best, best_id, frame, device):
    """Allgather (mu, id) over ranks, select with trstmi_select_best, broadcast
    the owner's frame.  Returns (mu, id, frame), identical on every rank."""
    world = dist.get_world_size()
    cand = torch.tensor([best, float(best_id)], dtype=torch.float64, device=device)
    allc = [torch.empty_like(cand) for _ in range(world)]
    dist.all_gather(allc, cand)
    mus = [c[0].item() for c in allc]
    ids = [int(c[1].item()) for c in allc]
    owner = select_best(mus, ids)
    if owner < 0:
        raise RuntimeError("solve: all restarts failed")
    buf = frame.clone() if dist.get_rank() == owner else torch.empty_like(frame)
    dist.broadcast(buf, src=owner)
    return mus[owner], ids[owner], buf
