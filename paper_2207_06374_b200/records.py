"""Run records, frame files and post-solve analysis (SURVEY.md §8(f) ranks 1
and 3), mirroring the reference's io.hpp and analysis.hpp
(/root/reference/proj/include/trstmi):

  frame_to_json / frame_from_json      io.hpp:35-76   {"d", "N", "columns": [[re, im, ...]]}
  frame_to_csv / frame_from_csv        io.hpp:87-139  2d rows x N columns, %.17g
  save_frame / load_frame              io.hpp:146-172 format by extension
  FileFormatError                      io.hpp:22-24
  bounds_report                        analysis.hpp:43-72
  offdiagonal_magnitudes, angle_spectrum, gram_summary
                                       frame.hpp:80-147 (GPU magnitudes + device sort,
                                                         sequential clustering)
  check_tight                          analysis.hpp:76-84 (GPU frame operator)
  one_distance_report, check_etf, certificates
                                       analysis.hpp:86-271
  solve -> SolveResult                 solver.hpp:38-54, 210-273 (trstmi_solve)
  make_run_record, restart_to_json, solver_config_to_json, trust_region_config_to_json,
  bounds_to_json, certificate_to_json, iso8601_utc_now
                                       io.hpp:175-276

Frames are the reference's interleaved column-major layout (frame.hpp:37-40):
column j = [re_0, im_0, re_1, im_1, ...].  Real-field frames (the new real mode)
are written with zero imaginary parts, so the files stay readable by the
reference.  Magnitudes use the CAS |z| = sqrt(re^2 + im^2) (DESIGN.md §3 item
10); the reference's std::abs (hypot) is at most an ulp away.
"""
import ctypes
import datetime
import json
import math
import time
from dataclasses import dataclass, field as dc_field
from typing import List, Optional

import numpy as np

from . import abi
from .api import Context, SolveError, ZeroColumnError, default_context, default_schedule, load_library

kDefaultClusterTol = 1e-4      # frame.hpp:23
kDefaultCertificateTol = 1e-4  # analysis.hpp:19


class FileFormatError(RuntimeError):
    """io.hpp:22-24."""


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _complex_view(frame, d, N, field):
    """Interleaved complex d x N (2dN doubles) for any field."""
    f = np.ascontiguousarray(frame, np.float64).reshape(-1)
    if field == abi.COMPLEX:
        if f.size != 2 * d * N:
            raise ValueError("frame length %d != 2dN = %d" % (f.size, 2 * d * N))
        return f
    if f.size != d * N:
        raise ValueError("frame length %d != dN = %d" % (f.size, d * N))
    out = np.zeros(2 * d * N)
    out[0::2] = f
    return out


# ------------------------------------------------------------------ frame files
def frame_to_json(frame, d, N, field=abi.COMPLEX):
    """io.hpp:35-46."""
    f = _complex_view(frame, d, N, field)
    cols = [[float(v) for v in f[j * 2 * d:(j + 1) * 2 * d]] for j in range(N)]
    return {"d": int(d), "N": int(N), "columns": cols}


def frame_from_json(obj):
    """io.hpp:48-76: returns (interleaved complex frame, d, N)."""
    if not isinstance(obj, dict) or not all(k in obj for k in ("d", "N", "columns")):
        raise FileFormatError("frame json: expected keys d, N, columns")
    d, N = obj["d"], obj["N"]
    if not isinstance(d, int) or not isinstance(N, int) or d < 1 or N < 1:
        raise FileFormatError("frame json: d and N must be >= 1")
    cols = obj["columns"]
    if not isinstance(cols, list) or len(cols) != N:
        raise FileFormatError("frame json: expected %d columns" % N)
    f = np.empty(2 * d * N)
    for j, col in enumerate(cols):
        if not isinstance(col, list) or len(col) != 2 * d:
            raise FileFormatError("frame json: column %d must hold %d numbers" % (j, 2 * d))
        f[j * 2 * d:(j + 1) * 2 * d] = [float(v) for v in col]
    return f, d, N


def full_precision(v):
    """io.hpp:79-83: '%.17g' (round-trips every double)."""
    return "%.17g" % v


def frame_to_csv(frame, d, N, field=abi.COMPLEX):
    """io.hpp:87-101: row 2i = real parts of coordinate i across columns, 2i+1 imaginary."""
    f = _complex_view(frame, d, N, field).reshape(N, d, 2)
    lines = []
    for i in range(d):
        for part in (0, 1):
            lines.append(",".join(full_precision(v) for v in f[:, i, part]))
    return "\n".join(lines) + "\n"


def frame_from_csv(text):
    """io.hpp:103-139."""
    rows = []
    for line in text.split("\n"):
        if line == "" or line == "\r":
            continue
        row = []
        for cell in line.split(","):
            try:
                row.append(float(cell))
            except ValueError:
                raise FileFormatError("frame csv: bad number '%s'" % cell) from None
        rows.append(row)
    if not rows or len(rows) % 2:
        raise FileFormatError("frame csv: expected an even, positive row count")
    d, N = len(rows) // 2, len(rows[0])
    for r, row in enumerate(rows):
        if len(row) != N:
            raise FileFormatError("frame csv: ragged row %d" % r)
    f = np.empty((N, d, 2))
    for i in range(d):
        f[:, i, 0] = rows[2 * i]
        f[:, i, 1] = rows[2 * i + 1]
    return f.reshape(-1), d, N


def save_frame(path, frame, d, N, field=abi.COMPLEX):
    """io.hpp:161-172: CSV for '.csv', JSON (indent 2) otherwise."""
    try:
        with open(path, "w") as out:
            if str(path).endswith(".csv"):
                out.write(frame_to_csv(frame, d, N, field))
            else:
                out.write(json.dumps(frame_to_json(frame, d, N, field), indent=2) + "\n")
    except OSError:
        raise FileFormatError("cannot write '%s'" % path) from None


def load_frame(path):
    """io.hpp:146-159: returns (interleaved complex frame, d, N)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise FileFormatError("cannot open '%s'" % path) from None
    if str(path).endswith(".csv"):
        return frame_from_csv(text)
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as e:
        raise FileFormatError("frame json parse error in '%s': %s" % (path, e)) from None
    return frame_from_json(obj)


# ------------------------------------------------------------------ bounds / analysis
def gerzon_max_complex(d):
    return d * d


def bounds_report(d, N):
    """analysis.hpp:53-72."""
    if d < 1 or N < d:
        raise ValueError("bounds_report: need 1 <= d <= N")
    welch = 0.0 if N <= d else math.sqrt((N - d) / (d * (N - 1)))
    rep = {"d": d, "N": N, "welch": welch, "orthoplex": None, "levenshtein": None,
           "gerzon_max": gerzon_max_complex(d), "best_applicable": welch}
    if N > d * d:
        rep["orthoplex"] = 1.0 / math.sqrt(d)
        rep["levenshtein"] = math.sqrt((2 * N - d * (d + 1)) / ((N - d) * (d + 1)))
        rep["best_applicable"] = max(welch, rep["orthoplex"], rep["levenshtein"])
    return rep


def offdiagonal_magnitudes(frame, d, N, field=abi.COMPLEX, normalize=False, sort=False):
    """frame.hpp:80-91 on the GPU: |G(j,k)|, j < k, row-major (sort=True: ascending)."""
    lib = load_library()
    f = np.ascontiguousarray(frame, np.float64).reshape(-1)
    n = N * (N - 1) // 2
    out = np.empty(n)
    zc = ctypes.c_int64(-1)
    rc = lib.trstmi_offdiag_magnitudes(field, d, N, _p(f), int(normalize), None if sort else _p(out),
                                       _p(out) if sort else None, ctypes.byref(zc))
    if rc == abi.TRSTMI_ERR_ZERO_COLUMN:
        raise ZeroColumnError(zc.value)
    if rc:
        raise RuntimeError("trstmi_offdiag_magnitudes failed (%d)" % rc)
    return out


def cluster_sorted(sorted_mags, cluster_tol=kDefaultClusterTol):
    """frame.hpp:96-118 over an ascending array (sequential sums, the reference's order)."""
    if not cluster_tol > 0.0:
        raise ValueError("cluster_tol must be positive")
    s = np.ascontiguousarray(sorted_mags, np.float64)
    means = np.empty(max(s.size, 1))
    cnt = ctypes.c_int64()
    rc = load_library().trstmi_cluster_sorted(_p(s), s.size, cluster_tol, _p(means), ctypes.byref(cnt))
    if rc:
        raise ValueError("cluster_magnitudes failed (%d)" % rc)
    return means[:cnt.value].copy()


def cluster_magnitudes(mags, cluster_tol=kDefaultClusterTol):
    return cluster_sorted(np.sort(np.asarray(mags, np.float64)), cluster_tol)


def angle_spectrum(frame, d, N, field=abi.COMPLEX, cluster_tol=kDefaultClusterTol):
    """frame.hpp:147-150: clustered distinct off-diagonal magnitudes (device sort)."""
    if not cluster_tol > 0.0:
        raise ValueError("cluster_tol must be positive")
    return cluster_sorted(offdiagonal_magnitudes(frame, d, N, field, sort=True), cluster_tol)


def gram_summary(frame, d, N, field=abi.COMPLEX, cluster_tol=kDefaultClusterTol):
    """frame.hpp:120-136."""
    mags = offdiagonal_magnitudes(frame, d, N, field)
    mu = 0.0
    if mags.size:
        m = float(mags.max())
        mu = m if m > 0.0 else 0.0
    return {"offdiag_mags": mags, "coherence": mu,
            "angle_spectrum": cluster_sorted(np.sort(mags), cluster_tol)}


def check_tight(frame, d, N, field=abi.COMPLEX, tol=kDefaultCertificateTol):
    """analysis.hpp:76-84: (deviation <= tol, max |Phi Phi* - (N/d) I|)."""
    f = np.ascontiguousarray(frame, np.float64).reshape(-1)
    dev = ctypes.c_double()
    rc = load_library().trstmi_frame_operator_deviation(field, d, N, _p(f), ctypes.byref(dev))
    if rc:
        raise RuntimeError("trstmi_frame_operator_deviation failed (%d)" % rc)
    return dev.value <= tol, dev.value


def _coherence(frame, d, N, field):
    mags = offdiagonal_magnitudes(frame, d, N, field)
    return float(mags.max()) if mags.size and mags.max() > 0.0 else 0.0


def one_distance_report(frame, d, N, field=abi.COMPLEX, tol=kDefaultCertificateTol):
    """analysis.hpp:118-133."""
    mags = offdiagonal_magnitudes(frame, d, N, field)
    spectrum = cluster_sorted(np.sort(mags), tol)
    cert = {"kind": "none", "tolerance": tol, "witness": {"clusters": float(spectrum.size)}}
    if spectrum.size == 1:
        cert["kind"] = "one_distance"
        cert["witness"]["angle"] = float(spectrum[0])
        cert["witness"]["spread"] = float(mags.max() - mags.min())
    return cert


def check_etf(frame, d, N, field=abi.COMPLEX, tol=kDefaultCertificateTol):
    """analysis.hpp:135-155."""
    spectrum = angle_spectrum(frame, d, N, field, tol)
    tight, deviation = check_tight(frame, d, N, field, tol)
    welch = bounds_report(d, N)["welch"] if N >= d else 0.0
    cert = {"kind": "none", "tolerance": tol, "witness": {"tight_deviation": deviation, "welch": welch}}
    if spectrum.size == 1:
        cert["witness"]["angle"] = float(spectrum[0])
        cert["witness"]["welch_gap"] = abs(float(spectrum[0]) - welch)
        if tight and abs(float(spectrum[0]) - welch) <= tol:
            cert["kind"] = "etf"
    return cert


def certificates(frame, d, N, field=abi.COMPLEX, tol=kDefaultCertificateTol):
    """analysis.hpp:218-271: every certificate that passes at `tol`."""
    certs = []
    mu = _coherence(frame, d, N, field)
    b = bounds_report(d, N)
    tight, deviation = check_tight(frame, d, N, field, tol)
    if tight:
        certs.append({"kind": "tight_frame", "tolerance": tol, "witness": {"deviation": deviation}})
    etf = check_etf(frame, d, N, field, tol)
    if etf["kind"] == "etf":
        certs.append(etf)
    one = one_distance_report(frame, d, N, field, tol)
    if one["kind"] == "one_distance":
        certs.append(one)
    if N > d and abs(mu - b["welch"]) <= tol:
        certs.append({"kind": "welch_equality", "tolerance": tol,
                      "witness": {"coherence": mu, "welch": b["welch"]}})
    if b["orthoplex"] is not None and abs(mu - b["orthoplex"]) <= tol:
        certs.append({"kind": "orthoplex_equality", "tolerance": tol,
                      "witness": {"coherence": mu, "orthoplex": b["orthoplex"],
                                  "count_condition": 1.0 if N <= 2 * d * d - 1 else 0.0}})
    if b["levenshtein"] is not None and abs(mu - b["levenshtein"]) <= tol:
        spectrum = angle_spectrum(frame, d, N, field, tol)
        two_class = spectrum.size == 2 and spectrum[0] <= tol and abs(spectrum[-1] - mu) <= tol
        certs.append({"kind": "levenshtein_equality", "tolerance": tol,
                      "witness": {"coherence": mu, "levenshtein": b["levenshtein"],
                                  "tight_zero_mu_detector": 1.0 if (tight and two_class) else 0.0}})
    return certs


# ------------------------------------------------------------------ solve + run records
@dataclass
class StageRecord:  # solver.hpp:31-36
    delta: float
    objective: float
    coherence: float
    outer_iterations: int


@dataclass
class RestartRecord:  # solver.hpp:38-45
    restart_index: int
    seed: int
    coherence: float
    succeeded: bool
    error: str
    stages: List[StageRecord] = dc_field(default_factory=list)


@dataclass
class SolveResult:  # solver.hpp:47-54 (+ field)
    config: abi.Cfg
    restarts: int
    seed: int
    best_frame: np.ndarray
    best_coherence: float
    best_restart: int
    per_restart: List[RestartRecord]
    wall_time_seconds: float


_TRIAL_ERRORS = {abi.TRIAL_ZERO_COLUMN: "zero column", abi.TRIAL_NONFINITE_X0: "trust_region_minimize: non-finite x0"}


def mix_seed(seed, index):
    """rng.hpp:13 child seeds, as trstmi_random_frames uses them."""
    return int(load_library().trstmi_mix_seed(ctypes.c_uint64(seed), ctypes.c_uint64(index)))


def solve(cfg, restarts=20, seed=0, ctx: Optional[Context] = None):
    """solve (solver.hpp:210-273) on the GPU: restarts i = 0..restarts-1 from
    random_frame(SplitMix64(mix_seed(seed, i))), best = lowest coherence, lowest
    index on ties.  Raises SolveError when every restart failed."""
    ctx = ctx or default_context()
    lib = ctx.lib
    dim = abi.dim_of(cfg.field, cfg.d, cfg.N)
    ns = cfg.n_stages or len(default_schedule(cfg.N, cfg.eps_target))
    best = np.empty(dim)
    mu = ctypes.c_double()
    arg = ctypes.c_int64()
    to = (abi.TrialOut * max(restarts, 1))()
    so = (abi.StageOut * max(restarts * ns, 1))()
    t0 = time.time()
    rc = lib.trstmi_solve(ctx.h, ctypes.byref(cfg), restarts, ctypes.c_uint64(seed), 0, _p(best), ctypes.byref(mu),
                          ctypes.byref(arg), ctypes.cast(to, ctypes.c_void_p), ctypes.cast(so, ctypes.c_void_p))
    wall = time.time() - t0
    ctx.check(rc, "solve")
    per = []
    for i in range(restarts):
        t = to[i]
        ok = t.status == abi.TRIAL_OK
        stages = [StageRecord(so[i * ns + k].delta, so[i * ns + k].objective, so[i * ns + k].coherence,
                              int(so[i * ns + k].outer_iterations)) for k in range(t.stages_done)]
        per.append(RestartRecord(i, mix_seed(seed, i), t.coherence if ok else 0.0, ok,
                                 "" if ok else _TRIAL_ERRORS.get(t.status, "restart failed"), stages))
    return SolveResult(cfg, restarts, seed, best, mu.value, int(arg.value), per, wall)


def iso8601_utc_now():
    """io.hpp:175-183."""
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def trust_region_config_to_json(cfg):
    """io.hpp:185-191 (the configuration as given: delta0 = 0 / max_cg = 0 mean the solver defaults)."""
    return {"delta0": cfg.delta0, "delta_max": cfg.delta_max, "eta": cfg.eta, "shrink": cfg.shrink,
            "grow": cfg.grow, "grad_tol": cfg.grad_tol, "max_outer": cfg.max_outer,
            "cg_force_c": cfg.cg_force_c, "max_cg": cfg.max_cg}


def solver_config_to_json(cfg, restarts, seed):
    """io.hpp:193-205."""
    sched = [cfg.schedule[k] for k in range(cfg.n_stages)] if cfg.n_stages else default_schedule(cfg.N, cfg.eps_target)
    return {"d": cfg.d, "N": cfg.N, "delta_schedule": list(sched), "restarts": restarts, "seed": seed,
            "eps_target": cfg.eps_target, "tr": trust_region_config_to_json(cfg),
            "field": "complex" if cfg.field == abi.COMPLEX else "real"}


def bounds_to_json(b):
    """io.hpp:207-216."""
    return {k: b[k] for k in ("d", "N", "welch", "gerzon_max", "best_applicable", "orthoplex", "levenshtein")}


def certificate_to_json(c):
    """io.hpp:218-224."""
    return {"kind": c["kind"], "tolerance": c["tolerance"], "witness": dict(sorted(c["witness"].items()))}


def restart_to_json(r: RestartRecord):
    """io.hpp:226-246."""
    j = {"restart": r.restart_index, "seed": r.seed, "succeeded": r.succeeded,
         "stages": [{"delta": s.delta, "objective": s.objective, "coherence": s.coherence,
                     "outer_iterations": s.outer_iterations} for s in r.stages]}
    if r.succeeded:
        j["coherence"] = r.coherence
    else:
        j["error"] = r.error
    return j


def make_run_record(method, result: SolveResult, method_config, started, finished,
                    certificate_tol=kDefaultCertificateTol):
    """io.hpp:249-276: configuration echo, per-restart summaries, the winning
    frame, and the bounds / certificate analysis of that frame."""
    c = result.config
    return {
        "schema_version": 1,
        "method": method,
        "seed": result.seed,
        "config": method_config,
        "per_restart": [restart_to_json(r) for r in result.per_restart],
        "best_restart": result.best_restart,
        "best_coherence": result.best_coherence,
        "best_frame": frame_to_json(result.best_frame, c.d, c.N, c.field),
        "bounds": bounds_to_json(bounds_report(c.d, c.N)),
        "certificates": [certificate_to_json(x) for x in
                         certificates(result.best_frame, c.d, c.N, c.field, certificate_tol)],
        "timestamps": {"started": started, "finished": finished},
        "wall_time_seconds": result.wall_time_seconds,
    }


# ------------------------------------------------------------------ targets (analysis.hpp:181-216)
def conjecture1_target(d, N):
    """analysis.hpp:181-187: 1/sqrt(d+1) for N in [d^2-d+2, d^2]."""
    if d < 2:
        return None
    return 1.0 / math.sqrt(d + 1) if d * d - d + 2 <= N <= d * d else None


def is_prime_power(n):
    """analysis.hpp:189-204."""
    if n < 2:
        return False
    p = 0
    f = 2
    while f * f <= n:
        if n % f == 0:
            p = f
            break
        f += 1
    if p == 0:
        return True
    while n % p == 0:
        n //= p
    return n == 1


def mub_removal_target(d, N):
    """analysis.hpp:206-216: 1/sqrt(d) for prime-power d and N in [d^2+1, d^2+d]."""
    if d < 2 or not is_prime_power(d):
        return None
    return 1.0 / math.sqrt(d) if d * d + 1 <= N <= d * (d + 1) else None


def column_norms(frame, d, N, field=abi.COMPLEX):
    f = _complex_view(frame, d, N, field).reshape(N, 2 * d)
    return np.sqrt((f * f).sum(axis=1))


def is_normalized(frame, d, N, field=abi.COMPLEX, tol=1e-12):
    """frame.hpp:51-56."""
    return bool(np.all(np.abs(column_norms(frame, d, N, field) - 1.0) <= tol))


def normalize_columns(frame, d, N, field=abi.COMPLEX):
    """frame.hpp:60-69 on the GPU (raises ZeroColumnError like the reference)."""
    f = np.ascontiguousarray(frame, np.float64).reshape(-1).copy()
    zc = ctypes.c_int64(-1)
    rc = load_library().trstmi_normalize_columns(field, d, N, _p(f), ctypes.byref(zc))
    if rc == abi.TRSTMI_ERR_ZERO_COLUMN:
        raise ZeroColumnError(zc.value)
    if rc:
        raise RuntimeError("trstmi_normalize_columns failed (%d)" % rc)
    return f


def distortion_mc(codebook, d, N, samples, seed, field=abi.COMPLEX):
    """beamforming.hpp:78-163 on the GPU: {"estimate", "std_error", "samples"}."""
    if samples < 1:
        raise ValueError("distortion_mc: samples >= 1")
    if N < 1:
        raise ValueError("distortion_mc: empty codebook")
    f = np.ascontiguousarray(_complex_view(codebook, d, N, field))
    est, se = ctypes.c_double(), ctypes.c_double()
    rc = load_library().trstmi_distortion_mc(d, N, _p(f), ctypes.c_uint64(samples), ctypes.c_uint64(seed),
                                             ctypes.byref(est), ctypes.byref(se))
    if rc:
        raise RuntimeError("trstmi_distortion_mc failed (%d)" % rc)
    return {"estimate": est.value, "std_error": se.value, "samples": int(samples)}
