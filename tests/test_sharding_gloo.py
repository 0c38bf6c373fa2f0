"""Multi-rank trial sharding on CPU (gloo, world_size 2): the product's
partition (trstmi_shard_range) covers the trial ids in contiguous blocks, and
the best-of exchange with the product's selection rule (trstmi_select_best)
returns the same (mu, id, frame) as the single-process selection — GPU-count
invariance of solve()'s result (solver.hpp:256-267).  Per-trial anneals come
from the oracle here (no GPU); on the box trstmi_solve_sharded runs the same
host logic over NCCL (tests/test_gpu_sharded.py)."""
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
    for total in (1, 5, 64, 1000, 4096):
        for world in (1, 2, 3, 8):
            ids = []
            for r in range(world):
                lo, hi = sharding.shard(total, world, r)
                assert all(i * world // total == r for i in range(lo, hi))  # trial i on rank floor(i G / T)
                ids.extend(range(lo, hi))
            assert ids == list(range(total))


def test_select_best_rule():
    # strict < in index order: the lowest index wins ties; failed / NaN entries are skipped
    assert sharding.select_best([0.5, 0.4, 0.4, 0.7]) == 1
    assert sharding.select_best([0.5, 0.4, 0.4], ids=[9, 7, 3]) == 2
    assert sharding.select_best([0.1, 0.4, 0.3], ok=[0, 1, 1]) == 2
    assert sharding.select_best([float("nan"), 0.4]) == 1
    assert sharding.select_best([float("nan")]) == -1


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
