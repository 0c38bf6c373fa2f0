"""ctypes handle on the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU
arms use this — it is the checker, never the product.
"""
import ctypes
import os
import subprocess

import numpy as np

from paper_2207_06374_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "_build", "liboracle.so")

_lib = None


def build_oracle():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_LIB):
            build_oracle()
        L = ctypes.CDLL(ORACLE_LIB)
        i64, c_int, dbl, vp, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_uint64
        L.orc_exp.argtypes = [dbl]
        L.orc_exp.restype = dbl
        L.orc_log.argtypes = [dbl]
        L.orc_log.restype = dbl
        L.orc_exp_array.argtypes = [vp, vp, i64]
        L.orc_hypot.argtypes = [dbl, dbl]
        L.orc_hypot.restype = dbl
        L.orc_log_array.argtypes = [vp, vp, i64]
        L.orc_cas_sum.argtypes = [vp, i64, c_int]
        L.orc_cas_sum.restype = dbl
        L.orc_cas_dot.argtypes = [vp, vp, i64, c_int]
        L.orc_cas_dot.restype = dbl
        L.orc_mix_seed.argtypes = [u64, u64]
        L.orc_mix_seed.restype = u64
        L.orc_welch_bound.argtypes = [i64, i64]
        L.orc_welch_bound.restype = dbl
        L.orc_default_schedule.argtypes = [i64, dbl, vp, c_int]
        L.orc_rng_uniform.argtypes = [u64, vp, i64]
        L.orc_rng_normal.argtypes = [u64, vp, i64]
        L.orc_random_frames.argtypes = [c_int, i64, i64, u64, i64, i64, vp, vp]
        L.orc_random_test_frame.argtypes = [c_int, i64, i64, u64, vp]
        L.orc_eval.argtypes = [c_int, i64, i64, c_int, vp, vp, dbl, dbl, c_int, vp, vp, vp, vp]
        L.orc_eval.restype = i64
        L.orc_hvp.argtypes = [c_int, i64, i64, c_int, vp, vp, dbl, vp, vp]
        L.orc_hvp.restype = i64
        L.orc_coherence.argtypes = [c_int, i64, i64, vp, c_int, vp, vp]
        L.orc_coherence.restype = i64
        L.orc_offdiag_magnitudes.argtypes = [c_int, i64, i64, vp, vp]
        L.orc_distortion_mc.argtypes = [i64, i64, vp, u64, u64, vp, vp]
        L.orc_altproj_batch.argtypes = [i64, i64, c_int, dbl, dbl, i64, vp, vp, vp, vp, vp]
        L.orc_solve_batch.argtypes = [vp, c_int, i64, vp, vp, vp, vp, vp, vp, c_int]
        L.orc_time_solve_batch.argtypes = [vp, c_int, i64, vp, vp, c_int, vp, vp]
        L.orc_time_solve_batch.restype = dbl
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def exp(x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().orc_exp_array(_p(x), _p(y), x.size)
    return y


def hypot(x, y):
    f = np.frompyfunc(lib().orc_hypot, 2, 1)
    return np.asarray(f(np.asarray(x, np.float64), np.asarray(y, np.float64)), np.float64)


def log(x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().orc_log_array(_p(x), _p(y), x.size)
    return y


def cas_sum(v, S):
    v = np.ascontiguousarray(v, np.float64)
    return lib().orc_cas_sum(_p(v), v.size, S)


def cas_dot(a, b, S):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().orc_cas_dot(_p(a), _p(b), a.size, S)


def schedule(N, eps=1e-7):
    buf = np.zeros(64)
    n = lib().orc_default_schedule(N, eps, _p(buf), 64)
    if n < 0:
        raise ValueError("bad schedule args")
    return list(buf[:n])


def uniforms(seed, n):
    out = np.empty(n)
    lib().orc_rng_uniform(seed, _p(out), n)
    return out


def normals(seed, n):
    out = np.empty(n)
    lib().orc_rng_normal(seed, _p(out), n)
    return out


def random_frames(field, d, N, seed, first, count):
    dim = abi.dim_of(field, d, N)
    f = np.empty((count, dim))
    st = np.empty((count, 3), np.uint64)
    rc = lib().orc_random_frames(field, d, N, seed, first, count, _p(f), _p(st))
    assert rc == 0
    return f, st


def random_test_frame(field, d, N, seed):
    f = np.empty(abi.dim_of(field, d, N))
    lib().orc_random_test_frame(field, d, N, seed, _p(f))
    return f


def eval_objective(field, d, N, S, x, delta, squared=True, direction=None, sc=0.0, want_weights=False):
    x = np.ascontiguousarray(x, np.float64)
    dirv = None if direction is None else np.ascontiguousarray(direction, np.float64)
    F = ctypes.c_double()
    s = ctypes.c_double()
    g = np.empty(abi.dim_of(field, d, N))
    w = np.empty(N * (N - 1) // 2) if want_weights else None
    zc = lib().orc_eval(field, d, N, S, _p(x), _p(dirv), sc, delta, int(squared), ctypes.byref(F), ctypes.byref(s),
                        _p(g), _p(w))
    return F.value, s.value, g, w, zc


def hvp(field, d, N, S, x, direction, delta):
    x = np.ascontiguousarray(x, np.float64)
    dirv = np.ascontiguousarray(direction, np.float64)
    hv = np.empty(abi.dim_of(field, d, N))
    path = ctypes.c_int()
    zc = lib().orc_hvp(field, d, N, S, _p(x), _p(dirv), delta, _p(hv), ctypes.byref(path))
    return hv, path.value, zc


def coherence(field, d, N, frame, normalize=False):
    frame = np.ascontiguousarray(frame, np.float64)
    mu = ctypes.c_double()
    arg = ctypes.c_int64()
    zc = lib().orc_coherence(field, d, N, _p(frame), int(normalize), ctypes.byref(mu), ctypes.byref(arg))
    return mu.value, arg.value, zc


def solve_batch(cfg, S, params, rng_state=None, threads=8, want_frames=True):
    dim = abi.dim_of(cfg.field, cfg.d, cfg.N)
    params = np.ascontiguousarray(params, np.float64).reshape(-1, dim).copy()
    T = params.shape[0]
    ns = cfg.n_stages or len(schedule(cfg.N, cfg.eps_target))
    frames = np.zeros_like(params) if want_frames else None
    to = (abi.TrialOut * max(T, 1))()
    so = (abi.StageOut * max(T * ns, 1))()
    cap = cfg.record_cap
    oo = (abi.OuterOut * max(T * cap, 1))() if cap > 0 else None
    rng = None
    if rng_state is not None:
        rng = np.ascontiguousarray(rng_state, np.uint64).reshape(-1).copy()
    rc = lib().orc_solve_batch(ctypes.byref(cfg), S, T, _p(params), _p(rng), _p(frames),
                               ctypes.cast(to, ctypes.c_void_p), ctypes.cast(so, ctypes.c_void_p),
                               ctypes.cast(oo, ctypes.c_void_p) if oo is not None else None, threads)
    assert rc == 0
    return dict(params=params, frames=frames, trials=to, stages=so, outer=oo, n_stages=ns, rng=rng)


def offdiag_magnitudes(field, d, N, frame):
    frame = np.ascontiguousarray(frame, np.float64)
    out = np.empty(N * (N - 1) // 2)
    lib().orc_offdiag_magnitudes(field, d, N, _p(frame), _p(out))
    return out


def mix_seed(seed, index):
    return int(lib().orc_mix_seed(seed, index))


def distortion_mc(d, N, book, samples, seed):
    book = np.ascontiguousarray(book, np.float64)
    est, se = ctypes.c_double(), ctypes.c_double()
    assert lib().orc_distortion_mc(d, N, _p(book), samples, seed, ctypes.byref(est), ctypes.byref(se)) == 0
    return est.value, se.value


def altproj_batch(d, N, starts, max_iters=300, mu_target=0.0, tol=1e-10):
    """alternating_projection (baseline.hpp:68-167) from each start frame: (frames, coherences, iterations, sweeps)."""
    starts = np.ascontiguousarray(starts, np.float64)
    R = starts.shape[0]
    frames = np.empty_like(starts)
    mu = np.empty(R)
    it = np.empty(R, np.int32)
    sw = np.empty(R, np.int32)
    rc = lib().orc_altproj_batch(d, N, max_iters, mu_target, tol, R, _p(starts), _p(frames), _p(mu), _p(it), _p(sw))
    assert rc == 0, rc
    return frames, mu, it, sw
