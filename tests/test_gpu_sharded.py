"""trstmi_solve_sharded / trstmi_best_of_ranks on one GPU (world size 1):
the multi-GPU solve() must return exactly what the single-GPU trstmi_solve
returns (same best frame bits, coherence and restart).  The cross-rank host
logic (partition, selection rule, allgather + broadcast) runs over gloo with
world size 2 in tests/test_sharding_gloo.py; only one GPU is available to
this build, so NCCL with world > 1 is not run here."""
import ctypes

import numpy as np
import pytest

from paper_2207_06374_b200 import abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2207_06374_b200 import api
    c = api.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("field,d,N,restarts", [(abi.COMPLEX, 2, 4, 20), (abi.REAL, 3, 7, 9)])
def test_solve_sharded_world1_equals_solve(ctx, field, d, N, restarts):
    lib = ctx.lib
    cfg = abi.default_cfg(field, d, N, 60)
    dim = abi.dim_of(field, d, N)
    f1, bc1, br1 = np.empty(dim), ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.trstmi_solve(ctx.h, ctypes.byref(cfg), restarts, 7, 0, ctypes.c_void_p(f1.ctypes.data),
                               ctypes.byref(bc1), ctypes.byref(br1), None, None), "solve")
    ctx.check(lib.trstmi_comm_init(ctx.h, 1, 0, None), "comm_init")
    f2, bc2, br2 = np.empty(dim), ctypes.c_double(), ctypes.c_int64()
    to = (abi.TrialOut * restarts)()
    first, count = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(lib.trstmi_solve_sharded(ctx.h, ctypes.byref(cfg), restarts, 7, ctypes.c_void_p(f2.ctypes.data),
                                       ctypes.byref(bc2), ctypes.byref(br2), ctypes.cast(to, ctypes.c_void_p),
                                       ctypes.byref(first), ctypes.byref(count)), "solve_sharded")
    assert (first.value, count.value) == (0, restarts)
    assert br1.value == br2.value and bc1.value == bc2.value
    assert f1.tobytes() == f2.tobytes()
    mus = [to[t].coherence for t in range(restarts)]
    assert min(mus) == bc2.value and mus.index(min(mus)) == br2.value


def test_best_of_ranks_world1_copies_local(ctx):
    import torch
    lib = ctx.lib
    ctx.check(lib.trstmi_comm_init(ctx.h, 1, 0, None), "comm_init")
    src = torch.arange(12, dtype=torch.float64, device="cuda")
    dst = torch.zeros_like(src)
    mu, idx = ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.trstmi_best_of_ranks(ctx.h, 12, 0.25, 42, ctypes.c_void_p(src.data_ptr()),
                                       ctypes.c_void_p(dst.data_ptr()), ctypes.byref(mu), ctypes.byref(idx), None),
              "best_of_ranks")
    assert mu.value == 0.25 and idx.value == 42 and torch.equal(src, dst)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_solve_devices_equals_single_gpu_solve(devices):
    """trstmi_solve_devices (one process, a host thread and a context per listed GPU, restart blocks by
    trstmi_shard_range, best-of on the host) returns trstmi_solve's result bit for bit for any device list —
    here the one GPU of the box listed several times, so the blocks anneal concurrently."""
    import ctypes
    from paper_2207_06374_b200 import abi, api
    from paper_2207_06374_b200 import records as rec
    cfg = abi.default_cfg(abi.COMPLEX, 3, 9, 40)
    restarts, seed = 11, 20240607
    ref = rec.solve(cfg, restarts=restarts, seed=seed)
    best, mu, idx, to, so = api.solve_devices(cfg, restarts, seed, devices)
    assert mu == ref.best_coherence and idx == ref.best_restart
    assert np.array_equal(best.view(np.uint64), ref.best_frame.view(np.uint64))
    for i in range(restarts):
        assert to[i].status == abi.TRIAL_OK
        assert to[i].coherence == ref.per_restart[i].coherence
        assert to[i].stages_done == len(ref.per_restart[i].stages)
