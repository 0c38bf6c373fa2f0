"""Alternating-projection baseline on the GPU: the host mirror of
/root/reference/proj/include/trstmi/baseline.hpp — `AltProjConfig` (:22-26), `alternating_projection` (:68-167),
`solve_altproj` (:172-199) — over the C ABI entry `trstmi_altproj_batch` (csrc/altproj.cu: one CTA per restart, the
Hermitian eigendecomposition as a round-robin Jacobi method).  Results take the solver's record shapes
(records.SolveResult / RestartRecord / StageRecord) so both methods share one run-record format, as in the reference.
No CPU fallback: without the CUDA library the import of `api` fails.
"""
import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import abi, api
from . import records as rec


@dataclass
class AltProjConfig:
    """baseline.hpp:22-26."""
    max_iters: int = 300
    mu_target: float = 0.0   # 0 -> max(welch_bound(d, N), 1e-12)
    tol: float = 1e-10       # max-entry change of the Gram between iterations


def _validate(d, N, cfg):
    """The reference's std::invalid_argument cases (baseline.hpp:72-82)."""
    if d > N:
        raise ValueError("alternating_projection: need d <= N")
    if cfg.max_iters < 1:
        raise ValueError("alternating_projection: need max_iters >= 1")
    target = cfg.mu_target if cfg.mu_target > 0.0 else max(rec.bounds_report(d, N)["welch"] if N > d else 0.0, 1e-12)
    if target >= 1.0:
        raise ValueError("alternating_projection: mu_target must be < 1")


def altproj_batch(d, N, cfg, starts):
    """alternating_projection from each row of `starts` (restarts x 2dN): (frames, coherences, iterations, sweeps)."""
    _validate(d, N, cfg)
    lib = api.load_library()
    starts = np.ascontiguousarray(starts, dtype=np.float64)
    R = starts.shape[0]
    frames = np.empty_like(starts)
    mu = np.empty(R)
    it = np.empty(R, np.int32)
    sw = np.empty(R, np.int32)
    rc = lib.trstmi_altproj_batch(d, N, cfg.max_iters, cfg.mu_target, cfg.tol, R, api._p(starts), api._p(frames),
                                  api._p(mu), api._p(it), api._p(sw))
    if rc == abi.TRSTMI_ERR_INVALID_ARG:
        raise ValueError("alternating_projection: invalid argument (d <= N <= 256, max_iters >= 1, mu_target < 1)")
    if rc:
        raise api.CudaError("trstmi_altproj_batch failed with status %d" % rc)
    return frames, mu, it, sw


def _result(d, N, seed, restarts, frames, mu, it, seeds, wall):
    cfg = abi.default_cfg(abi.COMPLEX, d, N, 200)
    per = []
    best = -1
    for i in range(restarts):
        stage = rec.StageRecord(0.0, float(mu[i]) * float(mu[i]), float(mu[i]), int(it[i]))  # baseline.hpp:152-156
        per.append(rec.RestartRecord(i, seeds[i], float(mu[i]), True, "", [stage]))
        if best < 0 or mu[i] < mu[best]:  # strict <: ties break by restart index (baseline.hpp:189)
            best = i
    return rec.SolveResult(cfg, restarts, seed, frames[best].copy(), float(mu[best]), best, per, wall)


def alternating_projection(d, N, cfg, rng_seed):
    """baseline.hpp:68-167 with the generator SplitMix64(rng_seed): the start is random_frame(d, N, rng)."""
    _validate(d, N, cfg)
    lib = api.load_library()
    dim = abi.dim_of(abi.COMPLEX, d, N)
    start = np.empty((1, dim))
    rc = lib.trstmi_random_frame_seeded(abi.COMPLEX, d, N, ctypes.c_uint64(rng_seed), api._p(start))
    if rc:
        raise ValueError("random_frame: need d, N >= 1")
    t0 = time.time()
    frames, mu, it, _ = altproj_batch(d, N, cfg, start)
    return _result(d, N, rng_seed, 1, frames, mu, it, [rng_seed], time.time() - t0)


def solve_altproj(d, N, cfg, restarts, seed):
    """baseline.hpp:172-199: restart i starts from random_frame(SplitMix64(mix_seed(seed, i))); all restarts run as
    one GPU batch; the best run wins, ties break by restart index."""
    if restarts < 1:
        raise ValueError("solve_altproj: restarts >= 1")
    _validate(d, N, cfg)
    t0 = time.time()
    starts, _ = api.random_frames(abi.COMPLEX, d, N, seed, 0, restarts)
    frames, mu, it, _ = altproj_batch(d, N, cfg, starts)
    seeds = [rec.mix_seed(seed, i) for i in range(restarts)]
    return _result(d, N, seed, restarts, frames, mu, it, seeds, time.time() - t0)


def altproj_config_to_json(d, N, cfg, restarts, seed):
    """main.cpp:65-71."""
    return {"d": d, "N": N, "max_iters": cfg.max_iters, "mu_target": cfg.mu_target, "tol": cfg.tol,
            "restarts": restarts, "seed": seed}
