"""Python binding of the C ABI (include/trstmi_b200.h) with the reference's
names and error behaviour (trstmi::eval_objective, hessian_vector_product,
coherence, anneal, solve; ZeroColumnError, DimensionMismatchError,
SolveError).  Used by the tests and bench.py; the C++ host mirror
(csrc/host/trstmi_host.hpp) is the native equivalent.

The CUDA library is mandatory: importing the binding on a machine without the
built library raises, and every compute call requires a CUDA device — there is
no CPU fallback.
"""
import ctypes
import os
from dataclasses import dataclass, field as dc_field
from typing import List, Optional

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtrstmi_b200.so")

_lib = None


class ZeroColumnError(RuntimeError):
    """frame.hpp:25-31: a column with norm below 1e-12."""

    def __init__(self, column):
        super().__init__("column %d has near-zero norm" % column)
        self.column = column


class DimensionMismatchError(ValueError):
    """frame.hpp:33-35."""


class SolveError(RuntimeError):
    """solver.hpp:56-58."""


class UnsupportedShapeError(ValueError):
    pass


class CudaError(RuntimeError):
    pass


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libtrstmi_b200.so not built: run __graft_entry__.build() "
                          "(python -m paper_2207_06374_b200.build)")
    try:
        # The library links libnccl.so.2; PyTorch bundles a newer NCCL under the same soname and needs ITS symbols.
        # Whichever loads first serves both, so let torch's copy in first when torch is installed (a later
        # `import torch` in the same process would otherwise fail with an undefined NCCL symbol).
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = ctypes.CDLL(LIB_PATH)
    c_i64, c_int, c_dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    lib.trstmi_ctx_create.argtypes = [c_int, ctypes.POINTER(vp)]
    lib.trstmi_ctx_destroy.argtypes = [vp]
    lib.trstmi_last_error.argtypes = [vp]
    lib.trstmi_last_error.restype = ctypes.c_char_p
    lib.trstmi_lanes.argtypes = [c_int, c_i64, c_i64]
    lib.trstmi_small_layout.argtypes = [c_int, c_i64, c_i64]
    lib.trstmi_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    lib.trstmi_mix_seed.restype = ctypes.c_uint64
    lib.trstmi_offdiag_magnitudes.argtypes = [c_int, c_i64, c_i64, vp, c_int, vp, vp, vp]
    lib.trstmi_cluster_sorted.argtypes = [vp, c_i64, c_dbl, vp, vp]
    lib.trstmi_frame_operator_deviation.argtypes = [c_int, c_i64, c_i64, vp, vp]
    lib.trstmi_normalize_columns.argtypes = [c_int, c_i64, c_i64, vp, vp]
    lib.trstmi_distortion_mc.argtypes = [c_i64, c_i64, vp, ctypes.c_uint64, ctypes.c_uint64, vp, vp]
    lib.trstmi_welch_bound.argtypes = [c_i64, c_i64]
    lib.trstmi_welch_bound.restype = c_dbl
    lib.trstmi_default_schedule.argtypes = [c_i64, c_dbl, vp, c_int]
    lib.trstmi_cfg_defaults.argtypes = [vp, c_int, c_int, c_int]
    lib.trstmi_random_frames.argtypes = [c_int, c_i64, c_i64, ctypes.c_uint64, c_i64, c_i64, vp, vp]
    lib.trstmi_eval_batch.argtypes = [vp, c_int, c_i64, c_i64, c_i64, vp, vp, c_int, vp, vp, vp, vp, vp]
    lib.trstmi_eval_batch_dev.argtypes = [vp, c_int, c_i64, c_i64, c_i64, vp, vp, c_int, vp, vp, vp, vp, vp, vp]
    lib.trstmi_hvp_batch.argtypes = [vp, c_int, c_i64, c_i64, c_i64, vp, vp, vp, vp, vp, vp]
    lib.trstmi_coherence_batch.argtypes = [vp, c_int, c_i64, c_i64, c_i64, vp, c_int, vp, vp, vp]
    lib.trstmi_solve_batch.argtypes = [vp, vp, c_i64, vp, vp, vp, vp, vp, vp]
    lib.trstmi_solve_batch_dev.argtypes = [vp, vp, c_i64, vp, vp, vp, vp, vp, vp, vp]
    lib.trstmi_solve.argtypes = [vp, vp, c_i64, ctypes.c_uint64, c_i64, vp, vp, vp, vp, vp]
    lib.trstmi_nccl_unique_id.argtypes = [vp]
    lib.trstmi_set_shard.argtypes = [vp, c_int, c_int, vp]
    lib.trstmi_shard_range.argtypes = [c_i64, c_int, c_int, vp, vp]
    lib.trstmi_select_best.argtypes = [c_i64, vp, vp, vp, vp]
    lib.trstmi_comm_init.argtypes = [vp, c_int, c_int, vp]
    lib.trstmi_best_of_ranks.argtypes = [vp, c_i64, c_dbl, c_i64, vp, vp, vp, vp, vp]
    lib.trstmi_solve_sharded.argtypes = [vp, vp, c_i64, ctypes.c_uint64, vp, vp, vp, vp, vp, vp]
    lib.trstmi_random_frame_seeded.argtypes = [c_int, c_i64, c_i64, ctypes.c_uint64, vp]
    lib.trstmi_altproj_batch.argtypes = [c_i64, c_i64, ctypes.c_int32, c_dbl, c_dbl, c_i64, vp, vp, vp, vp, vp]
    lib.trstmi_solve_devices.argtypes = [vp, c_int, vp, c_i64, ctypes.c_uint64, vp, vp, vp, vp, vp]
    lib.trstmi_launch_count.restype = ctypes.c_longlong
    lib.trstmi_measure_dfma_peak.argtypes = [vp, c_int, vp]
    _lib = lib
    return lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Context:
    """Owns a trstmi_ctx (device workspaces + stream) on one GPU."""

    def __init__(self, device=0):
        self.lib = load_library()
        h = ctypes.c_void_p()
        rc = self.lib.trstmi_ctx_create(device, ctypes.byref(h))
        if rc == abi.TRSTMI_ERR_NO_DEVICE:
            raise CudaError("no CUDA device: the TRST-MI B200 path has no CPU fallback")
        if rc != 0:
            raise CudaError("trstmi_ctx_create failed (%d)" % rc)
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.trstmi_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc, who=""):
        if rc == 0:
            return
        msg = self.lib.trstmi_last_error(self.h).decode()
        if rc == abi.TRSTMI_ERR_INVALID_ARG:
            raise ValueError(msg)
        if rc == abi.TRSTMI_ERR_DIM_MISMATCH:
            raise DimensionMismatchError(msg)
        if rc == abi.TRSTMI_ERR_ALL_FAILED:
            raise SolveError(msg)
        if rc == abi.TRSTMI_ERR_UNSUPPORTED:
            raise UnsupportedShapeError(msg)
        raise CudaError("%s: %s (code %d)" % (who, msg, rc))

    def set_shard(self, world, rank=0, nccl_id=None):
        """Row-block sharding of single large frames over `world` ranks
        (trstmi_set_shard); nccl_id None -> virtual ranks on this device."""
        buf = None
        if nccl_id is not None:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self.check(self.lib.trstmi_set_shard(self.h, world, rank, buf), "set_shard")

    # ---------------------------------------------------------------- objective
    def eval_batch(self, field, d, N, pts, delta, squared=True, want_weights=False):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, abi.dim_of(field, d, N))
        B = pts.shape[0]
        delta = np.ascontiguousarray(np.broadcast_to(np.asarray(delta, np.float64), (B,)))
        F = np.empty(B)
        s = np.empty(B)
        g = np.empty_like(pts)
        w = np.empty((B, N * (N - 1) // 2)) if want_weights else None
        zc = np.empty(B, np.int64)
        rc = self.lib.trstmi_eval_batch(self.h, field, d, N, B, _p(pts), _p(delta), int(squared), _p(F), _p(s),
                                        _p(g), _p(w), _p(zc))
        self.check(rc, "eval_batch")
        return F, s, g, w, zc

    def hvp_batch(self, field, d, N, pts, dirs, delta):
        dim = abi.dim_of(field, d, N)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, dim)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, dim)
        B = pts.shape[0]
        delta = np.ascontiguousarray(np.broadcast_to(np.asarray(delta, np.float64), (B,)))
        hv = np.empty_like(pts)
        path = np.empty(B, np.int32)
        zc = np.empty(B, np.int64)
        rc = self.lib.trstmi_hvp_batch(self.h, field, d, N, B, _p(pts), _p(dirs), _p(delta), _p(hv), _p(path), _p(zc))
        self.check(rc, "hvp_batch")
        return hv, path, zc

    def coherence_batch(self, field, d, N, frames, normalize=False):
        frames = np.ascontiguousarray(frames, dtype=np.float64).reshape(-1, abi.dim_of(field, d, N))
        B = frames.shape[0]
        mu = np.empty(B)
        arg = np.empty(B, np.int64)
        zc = np.empty(B, np.int64)
        rc = self.lib.trstmi_coherence_batch(self.h, field, d, N, B, _p(frames), int(normalize), _p(mu), _p(arg),
                                             _p(zc))
        self.check(rc, "coherence_batch")
        return mu, arg, zc

    # ---------------------------------------------------------------- anneal
    def solve_batch(self, cfg, params, rng_state=None, want_frames=True):
        """Batched anneal() of len(params) trials; returns dict of numpy outputs."""
        field, d, N = cfg.field, cfg.d, cfg.N
        dim = abi.dim_of(field, d, N)
        params = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, dim).copy()
        T = params.shape[0]
        ns = cfg.n_stages or default_schedule_len(N, cfg.eps_target)
        frames = np.zeros_like(params) if want_frames else None
        to = (abi.TrialOut * max(T, 1))()
        so = (abi.StageOut * max(T * ns, 1))()
        cap = cfg.record_cap
        oo = (abi.OuterOut * max(T * cap, 1))() if cap > 0 else None
        rng = None
        if rng_state is not None:
            rng = np.ascontiguousarray(rng_state, dtype=np.uint64).reshape(-1).copy()
        rc = self.lib.trstmi_solve_batch(self.h, ctypes.byref(cfg), T, _p(params), _p(rng), _p(frames),
                                         ctypes.cast(to, ctypes.c_void_p), ctypes.cast(so, ctypes.c_void_p),
                                         ctypes.cast(oo, ctypes.c_void_p) if oo is not None else None)
        self.check(rc, "solve_batch")
        return dict(params=params, frames=frames, trials=to, stages=so, outer=oo, n_stages=ns, rng=rng)


def nccl_unique_id():
    """128-byte ncclUniqueId (rank 0 creates it and shares it with the others)."""
    buf = ctypes.create_string_buffer(128)
    rc = load_library().trstmi_nccl_unique_id(buf)
    if rc:
        raise CudaError("ncclGetUniqueId failed (%d)" % rc)
    return buf.raw


def default_schedule(N, eps_target=1e-7):
    lib = load_library()
    buf = (ctypes.c_double * abi.MAX_STAGES)()
    n = lib.trstmi_default_schedule(N, eps_target, ctypes.cast(buf, ctypes.c_void_p), abi.MAX_STAGES)
    if n < 0:
        raise ValueError("default_delta_schedule: invalid input")
    return [buf[i] for i in range(n)]


def default_schedule_len(N, eps_target=1e-7):
    return len(default_schedule(N, eps_target))


def lanes(field, d, N):
    return load_library().trstmi_lanes(field, d, N)


def small_layout(field, d, N):
    """-1 large-frame path, 0 Gram recomputed, 1 stored Gram, 2 stored Gram in
    bank-padded rows (trstmi_small_layout; a pure function, no GPU needed)."""
    return load_library().trstmi_small_layout(field, d, N)


def welch_bound(d, N):
    return load_library().trstmi_welch_bound(d, N)


def random_frames(field, d, N, seed, first, count):
    lib = load_library()
    dim = abi.dim_of(field, d, N)
    f = np.empty((count, dim))
    st = np.empty((count, 3), np.uint64)
    rc = lib.trstmi_random_frames(field, d, N, seed, first, count, _p(f), _p(st))
    if rc:
        raise ValueError("random_frame: need d, N >= 1")
    return f, st


def solve_devices(cfg, restarts, seed, devices):
    """solve() (solver.hpp:210-273) over the listed GPUs of this process: one host thread and one context per entry
    (trstmi_solve_devices).  Returns (best_frame, best_coherence, best_restart, trial_out, stage_out)."""
    lib = load_library()
    dim = abi.dim_of(cfg.field, cfg.d, cfg.N)
    ns = cfg.n_stages or len(default_schedule(cfg.N, cfg.eps_target))
    devs = (ctypes.c_int * len(devices))(*devices)
    best = np.empty(dim)
    mu = ctypes.c_double()
    idx = ctypes.c_int64()
    to = (abi.TrialOut * max(restarts, 1))()
    so = (abi.StageOut * max(restarts * ns, 1))()
    rc = lib.trstmi_solve_devices(ctypes.cast(devs, ctypes.c_void_p), len(devices), ctypes.byref(cfg), restarts,
                                  ctypes.c_uint64(seed), _p(best), ctypes.byref(mu), ctypes.byref(idx),
                                  ctypes.cast(to, ctypes.c_void_p), ctypes.cast(so, ctypes.c_void_p))
    if rc == abi.TRSTMI_ERR_NO_DEVICE:
        raise CudaError("no CUDA device: the TRST-MI B200 path has no CPU fallback")
    if rc:
        raise CudaError("trstmi_solve_devices failed with status %d" % rc)
    return best, mu.value, int(idx.value), to, so


# ------------------------------------------------------------------ reference-named API
@dataclass
class SmoothObjective:
    """smoothing.hpp:27-34."""
    delta: float = 1e-2
    d: int = 0
    N: int = 0
    squared: bool = True
    field: int = abi.COMPLEX

    def pair_count(self):
        return self.N * (self.N - 1) // 2


@dataclass
class ObjectiveEval:
    """smoothing.hpp:36-41."""
    value: float
    s: float
    grad: np.ndarray
    softmax_weights: Optional[np.ndarray]


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def eval_objective(point, obj: SmoothObjective, ctx=None) -> ObjectiveEval:
    """eval_objective (smoothing.hpp:82-162) on the GPU; raises like the reference."""
    ctx = ctx or default_context()
    if obj.delta <= 0.0:
        raise ValueError("eval_objective: delta <= 0")
    if obj.N < 2:
        raise ValueError("eval_objective: need N >= 2")
    point = np.asarray(point, np.float64)
    if point.size != abi.dim_of(obj.field, obj.d, obj.N):
        raise DimensionMismatchError("eval_objective: point length mismatch")
    F, s, g, w, zc = ctx.eval_batch(obj.field, obj.d, obj.N, point[None], obj.delta, obj.squared, True)
    if zc[0] >= 0:
        raise ZeroColumnError(int(zc[0]))
    return ObjectiveEval(float(F[0]), float(s[0]), g[0], w[0])


def hessian_vector_product(point, direction, obj: SmoothObjective, ctx=None):
    """hessian_vector_product (smoothing.hpp:187-194): central difference;
    raises ZeroColumnError when a perturbed point hits a zero column."""
    ctx = ctx or default_context()
    point = np.asarray(point, np.float64)
    direction = np.asarray(direction, np.float64)
    if direction.size != point.size:
        raise DimensionMismatchError("fd_hessian_vector_product: length mismatch")
    hv, path, zc = ctx.hvp_batch(obj.field, obj.d, obj.N, point[None], direction[None], obj.delta)
    if path[0] in (abi.HVP_FORWARD, abi.HVP_BACKWARD, abi.HVP_FAILED):
        # the plain central difference threw; report the first failing column
        raise ZeroColumnError(int(zc[0]) if zc[0] >= 0 else -1)
    return hv[0]


def coherence(frame, field=abi.COMPLEX, d=None, N=None, ctx=None):
    """coherence (frame.hpp:138-145) of a column-major frame (d x N)."""
    ctx = ctx or default_context()
    mu, arg, zc = ctx.coherence_batch(field, d, N, np.asarray(frame, np.float64)[None], normalize=False)
    return float(mu[0]), int(arg[0])
