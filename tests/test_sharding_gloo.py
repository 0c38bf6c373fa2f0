"""Multi-rank trial sharding on CPU (gloo, world_size 2): shards partition
the trial ids, and the best-of exchange (allgather + broadcast) returns the
same (mu, id, frame) as the single-process selection — GPU-count invariance
of solve()'s result (solver.hpp:256-267).  Per-trial anneals come from the
oracle here (no GPU); on the box the same code runs over NCCL."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_06374_b200 import abi, sharding

FIELD, D, N, TOTAL, MAX_OUTER = abi.COMPLEX, 2, 5, 6, 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _anneal(lo, hi):
    from tests import oracle_ffi as orc
    cfg = abi.default_cfg(FIELD, D, N, MAX_OUTER)
    starts, st = orc.random_frames(FIELD, D, N, 0, lo, hi - lo)
    r = orc.solve_batch(cfg, abi.lanes_for(FIELD, D, N), starts, st, threads=2)
    mus = [r["trials"][t].coherence for t in range(hi - lo)]
    ok = [r["trials"][t].status == abi.TRIAL_OK for t in range(hi - lo)]
    return mus, ok, r["frames"]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = sharding.shard(TOTAL, world, rank)
    mus, ok, frames = _anneal(lo, hi)
    mu, bid = sharding.local_best(mus, ok, lo)
    fr = torch.from_numpy(frames[bid - lo]) if bid >= 0 else torch.zeros(2 * D * N, dtype=torch.float64)
    gmu, gid, gframe = sharding.global_best(mu, bid, fr, "cpu")
    out[rank] = (gmu, gid, gframe.numpy().tobytes())
    dist.destroy_process_group()


def test_shards_partition_trials():
    for world in (1, 2, 3, 8):
        ids = []
        for r in range(world):
            lo, hi = sharding.shard(4096, world, r)
            ids.extend(range(lo, hi))
        assert ids == list(range(4096))


def test_two_rank_best_equals_single_process():
    mus, ok, frames = _anneal(0, TOTAL)
    mu1, id1 = sharding.local_best(mus, ok, 0)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1]
    gmu, gid, gframe = res[0]
    assert gmu == mu1 and gid == id1
    assert np.frombuffer(gframe, np.float64).tobytes() == frames[id1].tobytes()
