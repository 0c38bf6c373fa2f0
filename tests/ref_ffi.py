"""ctypes handle on oracle/_ref/libtrstmi_ref.so: the reference's own hot-path
headers compiled unchanged against oracle/eigen_shim (see oracle/ref_capi.cpp).

TEST INFRASTRUCTURE: only tests/ and bench.py's CPU arms use this — it pins
the CAS oracle to the reference and is the CPU baseline; never the product.
The library is built in the container that holds /root/reference (make -C
oracle) and travels prebuilt to the GPU box; where it is missing, callers skip.
"""
import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libtrstmi_ref.so")

_lib = None


def available():
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_LIB)
        i64, c_int, dbl, vp, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_uint64
        L.ref_eval.argtypes = [c_int, i64, i64, vp, dbl, c_int, vp, vp, vp, vp]
        L.ref_eval.restype = i64
        L.ref_hvp.argtypes = [c_int, i64, i64, vp, vp, dbl, vp]
        L.ref_hvp.restype = i64
        L.ref_offdiag_magnitudes.argtypes = [c_int, i64, i64, vp, vp]
        L.ref_coherence.argtypes = [c_int, i64, i64, vp, c_int, vp, vp]
        L.ref_coherence.restype = i64
        L.ref_default_schedule.argtypes = [i64, dbl, vp, c_int]
        L.ref_batch_create.argtypes = [c_int, i64, i64, u64, i64, i64, vp]
        L.ref_batch_create.restype = vp
        L.ref_batch_destroy.argtypes = [vp]
        L.ref_batch_run_stages.argtypes = [vp, vp, c_int, c_int, c_int, vp, vp, c_int, vp, vp, vp, vp]
        L.ref_batch_run_stages.restype = dbl
        L.ref_batch_params.argtypes = [vp, vp, vp]
        L.ref_batch_keep_history.argtypes = [vp, c_int]
        L.ref_batch_history.argtypes = [vp, i64, i64, vp, vp]
        L.ref_batch_history.restype = i64
        L.ref_anneal.argtypes = [i64, i64, vp, c_int, vp, vp, u64, i64, vp, vp, vp]
        L.ref_solve.argtypes = [i64, i64, c_int, u64, dbl, vp, vp, c_int, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dim(field, d, N):
    return (2 if field == 0 else 1) * d * N


def eval_objective(field, d, N, x, delta, squared=True, want_weights=False):
    x = np.ascontiguousarray(x, np.float64)
    F, s = ctypes.c_double(), ctypes.c_double()
    g = np.empty(_dim(field, d, N))
    w = np.empty(N * (N - 1) // 2) if want_weights else None
    zc = lib().ref_eval(field, d, N, _p(x), delta, int(squared), ctypes.byref(F), ctypes.byref(s), _p(g), _p(w))
    return F.value, s.value, g, w, zc


def hvp(field, d, N, x, direction, delta):
    x = np.ascontiguousarray(x, np.float64)
    v = np.ascontiguousarray(direction, np.float64)
    hv = np.empty(_dim(field, d, N))
    zc = lib().ref_hvp(field, d, N, _p(x), _p(v), delta, _p(hv))
    return hv, zc


def offdiag_magnitudes(field, d, N, frame):
    frame = np.ascontiguousarray(frame, np.float64)
    out = np.empty(N * (N - 1) // 2)
    lib().ref_offdiag_magnitudes(field, d, N, _p(frame), _p(out))
    return out


def coherence(field, d, N, frame, normalize=False):
    frame = np.ascontiguousarray(frame, np.float64)
    mu, arg = ctypes.c_double(), ctypes.c_int64()
    zc = lib().ref_coherence(field, d, N, _p(frame), int(normalize), ctypes.byref(mu), ctypes.byref(arg))
    return mu.value, arg.value, zc


def schedule(N, eps=1e-7):
    buf = np.zeros(64)
    n = lib().ref_default_schedule(N, eps, _p(buf), 64)
    return list(buf[:n])


def tr_arrays(cfg):
    tr6 = np.array([cfg.delta0, cfg.delta_max, cfg.eta, cfg.shrink, cfg.grow, cfg.grad_tol, cfg.cg_force_c])
    tri = np.array([cfg.max_outer, cfg.max_cg], np.int32)
    return tr6, tri


class Batch:
    """Trials [first, first+count) of `seed` annealed stage by stage with the
    reference's own functions (solver.hpp:182-200)."""

    def __init__(self, cfg, seed, first, count, starts=None):
        self.cfg = cfg
        self.count = count
        self.sched = np.array(list(cfg.schedule)[:cfg.n_stages] if cfg.n_stages else schedule(cfg.N, cfg.eps_target))
        self.ns = len(self.sched)
        st = None if starts is None else np.ascontiguousarray(starts, np.float64)
        self.h = lib().ref_batch_create(cfg.field, cfg.d, cfg.N, seed, first, count, _p(st))
        self.tr6, self.tri = tr_arrays(cfg)
        self.rec = np.zeros((count, self.ns, 4))

    def run(self, k0, k1, threads):
        o, e, hv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        sec = lib().ref_batch_run_stages(self.h, _p(self.sched), self.ns, k0, k1, _p(self.tr6), _p(self.tri), threads,
                                         _p(self.rec), ctypes.byref(o), ctypes.byref(e), ctypes.byref(hv))
        return sec, o.value, e.value, hv.value

    def keep_history(self, on=True):
        lib().ref_batch_keep_history(self.h, int(on))

    def history(self, t, cap=100000):
        """OuterRecords of trial t: (ints[:, stage, iteration, cg_exit, cg_iterations, accepted],
        doubles[:, value, grad_norm, radius, rho, step_norm])."""
        ints = np.zeros((cap, 5), np.int32)
        dbl = np.zeros((cap, 5))
        n = lib().ref_batch_history(self.h, t, cap, _p(ints), _p(dbl))
        n = min(n, cap)
        return ints[:n], dbl[:n]

    def params(self):
        out = np.empty((self.count, _dim(self.cfg.field, self.cfg.d, self.cfg.N)))
        st = np.empty(self.count, np.int32)
        lib().ref_batch_params(self.h, _p(out), _p(st))
        return out, st

    def close(self):
        if self.h:
            lib().ref_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def anneal(cfg, seed, index, start=None):
    sched = np.array(list(cfg.schedule)[:cfg.n_stages] if cfg.n_stages else schedule(cfg.N, cfg.eps_target))
    tr6, tri = tr_arrays(cfg)
    frame = np.empty(_dim(0, cfg.d, cfg.N))
    rec = np.zeros((len(sched), 4))
    st = None if start is None else np.ascontiguousarray(start, np.float64)
    rc = lib().ref_anneal(cfg.d, cfg.N, _p(sched), len(sched), _p(tr6), _p(tri), seed, index, _p(st), _p(frame),
                          _p(rec))
    return rc, frame, rec


def solve(cfg, restarts, seed, threads):
    tr6, tri = tr_arrays(cfg)
    frame = np.empty(_dim(0, cfg.d, cfg.N))
    bc, br, wall = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
    per = np.empty(restarts)
    rc = lib().ref_solve(cfg.d, cfg.N, restarts, seed, cfg.eps_target, _p(tr6), _p(tri), threads, _p(frame),
                         ctypes.byref(bc), ctypes.byref(br), _p(per), ctypes.byref(wall))
    return dict(rc=rc, frame=frame, best_coherence=bc.value, best_restart=br.value, per_restart=per, wall_s=wall.value)
