"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

The small-frame path computes in the Canonical Arithmetic Spec, so values,
gradients, Hessian-vector products, coherences, argmax pairs and whole
anneal trajectories (every OuterRecord / StageRecord field) must be
BIT-IDENTICAL to the oracle on the same seeded inputs.
"""
import numpy as np
import pytest

from paper_2207_06374_b200 import abi
from tests import oracle_ffi as orc

pytestmark = pytest.mark.gpu

C, R = abi.COMPLEX, abi.REAL

SHAPES = [(C, 2, 4), (C, 3, 6), (C, 4, 10), (C, 2, 100), (C, 6, 36), (R, 4, 10), (C, 1, 2), (R, 3, 5),
          (R, 2, 40), (C, 11, 20), (R, 13, 30), (C, 8, 9), (R, 1, 3)]


@pytest.fixture(scope="module")
def ctx():
    from paper_2207_06374_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def frames_for(field, d, N, seeds):
    return np.stack([orc.random_test_frame(field, d, N, s) for s in seeds])


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("field,d,N", SHAPES)
@pytest.mark.parametrize("delta", [1e-1, 1e-3, 2e-8])
def test_eval_bit_exact(ctx, field, d, N, delta):
    from paper_2207_06374_b200 import api
    S = api.lanes(field, d, N)
    pts = frames_for(field, d, N, range(11, 15))
    pts[1] *= 3.7  # unnormalised columns exercise the normalisation chain rule
    F, s, g, w, zc = ctx.eval_batch(field, d, N, pts, delta, True, True)
    for b in range(pts.shape[0]):
        Fo, so, go, wo, zo = orc.eval_objective(field, d, N, S, pts[b], delta, want_weights=True)
        assert zc[b] == -1 and zo == -1
        assert bits(F[b]) == bits(Fo), (F[b], Fo)
        assert bits(s[b]) == bits(so)
        assert np.array_equal(bits(g[b]), bits(go)), np.max(np.abs(g[b] - go))
        assert np.array_equal(bits(w[b]), bits(wo))


@pytest.mark.parametrize("field,d,N", [(C, 3, 5), (R, 4, 10), (C, 2, 100)])
def test_eval_magnitude_mode_bit_exact(ctx, field, d, N):
    from paper_2207_06374_b200 import api
    S = api.lanes(field, d, N)
    pts = frames_for(field, d, N, [4096, 7])
    F, s, g, w, zc = ctx.eval_batch(field, d, N, pts, 1e-1, False, True)
    for b in range(2):
        Fo, so, go, wo, zo = orc.eval_objective(field, d, N, S, pts[b], 1e-1, squared=False, want_weights=True)
        assert bits(F[b]) == bits(Fo)
        assert np.array_equal(bits(g[b]), bits(go))


def test_eval_zero_column(ctx):
    # test_smoothing.cpp:148-153: column 1 is zero -> ZeroColumnError(1)
    from paper_2207_06374_b200 import api
    pt = np.zeros(8)
    pt[0] = 1.0
    with pytest.raises(api.ZeroColumnError) as e:
        api.eval_objective(pt, api.SmoothObjective(0.1, 2, 2, True), ctx)
    assert e.value.column == 1
    F, s, g, w, zc = ctx.eval_batch(C, 2, 2, pt[None], 0.1)
    assert zc[0] == 1 and np.isinf(F[0]) and not g.any()


def test_eval_closed_forms(ctx):
    # test_smoothing.cpp:16-34: orthogonal pair F = s = 0; coincident pair F = 1
    from paper_2207_06374_b200 import api
    ident = np.array([1.0, 0, 0, 0, 0, 0, 1.0, 0])
    for delta in (1.0, 1e-2, 1e-6):
        e = api.eval_objective(ident, api.SmoothObjective(delta, 2, 2, True), ctx)
        assert e.s == 0.0 and e.value == 0.0
    coinc = np.array([1.0, 0, 0, 0, 1.0, 0, 0, 0])
    e = api.eval_objective(coinc, api.SmoothObjective(0.1, 2, 2, True), ctx)
    assert abs(e.value - 1.0) <= 1e-15


@pytest.mark.parametrize("field,d,N", SHAPES)
def test_hvp_bit_exact(ctx, field, d, N):
    from paper_2207_06374_b200 import api
    S = api.lanes(field, d, N)
    pts = frames_for(field, d, N, [3, 5, 8])
    rng = np.random.default_rng(d * 1000 + N)
    dirs = rng.standard_normal(pts.shape)
    dirs[2] = 0.0  # zero direction -> zero product
    for delta in (1e-2, 1e-5):
        hv, path, zc = ctx.hvp_batch(field, d, N, pts, dirs, delta)
        for b in range(3):
            ho, po, zo = orc.hvp(field, d, N, S, pts[b], dirs[b], delta)
            assert path[b] == po
            assert np.array_equal(bits(hv[b]), bits(ho))
    assert path[2] == abi.HVP_ZERO_DIR and not hv[2].any()


def test_hvp_one_sided_fallback(ctx):
    # test_solver.cpp:212-230: a column at the FD step size forces the fallback
    from paper_2207_06374_b200 import api
    kfd = float.fromhex('0x1.965fea53d6e3dp-18')
    point = np.array([1e-3, 0.0, 1.0, 0.0])
    direction = np.array([-1.0, 0.0, 0.0, 0.0])
    for _ in range(3):
        point[0] = kfd * (1.0 + np.linalg.norm(point)) / np.linalg.norm(direction)
    obj = api.SmoothObjective(1e-1, 1, 2, True)
    with pytest.raises(api.ZeroColumnError):
        api.hessian_vector_product(point, direction, obj, ctx)
    hv, path, zc = ctx.hvp_batch(C, 1, 2, point[None], direction[None], 1e-1)
    ho, po, zo = orc.hvp(C, 1, 2, api.lanes(C, 1, 2), point, direction, 1e-1)
    assert path[0] == po and po in (abi.HVP_FORWARD, abi.HVP_BACKWARD)
    assert np.all(np.isfinite(hv[0]))
    assert np.array_equal(bits(hv[0]), bits(ho))


@pytest.mark.parametrize("field,d,N", SHAPES)
def test_coherence_bit_exact(ctx, field, d, N):
    pts = frames_for(field, d, N, [21, 22, 23])
    pts[0] *= 0.25
    for normalize in (False, True):
        mu, arg, zc = ctx.coherence_batch(field, d, N, pts, normalize)
        for b in range(3):
            mo, ao, zo = orc.coherence(field, d, N, pts[b], normalize)
            assert bits(mu[b]) == bits(mo)
            assert arg[b] == ao


def _cmp_solve(g, o, T, ns, cap):
    for t in range(T):
        a, b = g["trials"][t], o["trials"][t]
        assert a.status == b.status, (t, a.status, b.status)
        assert a.outer_iterations == b.outer_iterations, (t, a.outer_iterations, b.outer_iterations)
        assert a.evals == b.evals and a.hvps == b.hvps, (t, a.evals, b.evals, a.hvps, b.hvps)
        assert bits(a.coherence) == bits(b.coherence)
        assert a.argmax_pair == b.argmax_pair
        for k in range(ns):
            sa, sb = g["stages"][t * ns + k], o["stages"][t * ns + k]
            assert (sa.outer_iterations, sa.status, sa.argmax_pair) == (sb.outer_iterations, sb.status, sb.argmax_pair)
            assert bits(sa.objective) == bits(sb.objective) and bits(sa.coherence) == bits(sb.coherence)
        if cap:
            assert a.records == b.records
            for i in range(a.records):
                ra, rb = g["outer"][t * cap + i], o["outer"][t * cap + i]
                assert (ra.stage, ra.iteration, ra.cg_exit, ra.cg_iterations, ra.accepted) == \
                       (rb.stage, rb.iteration, rb.cg_exit, rb.cg_iterations, rb.accepted), (t, i)
                for f in ("value", "grad_norm", "radius", "rho", "step_norm"):
                    assert bits(getattr(ra, f)) == bits(getattr(rb, f)), (t, i, f)
    assert np.array_equal(bits(g["params"]), bits(o["params"]))
    assert np.array_equal(bits(g["frames"]), bits(o["frames"]))


@pytest.mark.parametrize("field,d,N,trials,max_outer,cap", [
    (R, 4, 10, 16, 200, 4000),     # BASELINE config 1 (full budget, 16 of its 64 trials)
    (C, 2, 4, 8, 200, 1000),
    (C, 6, 36, 2, 30, 2000),       # config 3 shape, reduced budget
    (C, 2, 100, 2, 12, 1000),      # config 2 shape, reduced budget
    (C, 3, 7, 6, 200, 0),
])
def test_solve_batch_trajectory_bit_exact(ctx, field, d, N, trials, max_outer, cap):
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(field, d, N, max_outer)
    cfg.record_cap = cap
    S = api.lanes(field, d, N)
    starts, st = api.random_frames(field, d, N, 0, 0, trials)
    so, sto = orc.random_frames(field, d, N, 0, 0, trials)
    assert np.array_equal(bits(starts), bits(so)) and np.array_equal(st, sto)
    g = ctx.solve_batch(cfg, starts, st)
    o = orc.solve_batch(cfg, S, starts, st)
    _cmp_solve(g, o, trials, g["n_stages"], cap)


@pytest.mark.parametrize("field,d,N,trials,max_outer", [
    (C, 6, 36, 4, 1000),   # BASELINE config 3: the config's full budget (8 stages, max_outer 1000 + 50k)
    (C, 2, 100, 4, 500),   # BASELINE config 2: the config's full budget (~2.5e5 evaluations per trial)
])
def test_full_budget_trajectories_bit_exact(ctx, field, d, N, trials, max_outer):
    """Whole anneals at the headline configs' own budgets: every stage record, iteration / evaluation /
    HVP count, final parameters and frames identical to the oracle (~50 s of CPU oracle time)."""
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(field, d, N, max_outer)
    S = api.lanes(field, d, N)
    starts, st = api.random_frames(field, d, N, 0, 0, trials)
    g = ctx.solve_batch(cfg, starts, st)
    o = orc.solve_batch(cfg, S, starts, st, threads=trials)
    _cmp_solve(g, o, trials, g["n_stages"], 0)


@pytest.mark.parametrize("field,d,N,trials,max_outer", [
    (C, 2, 100, 3, 10),   # config 2 shape: the fused central difference (dual layout) is on by default
    (C, 6, 36, 3, 20),    # config 3 shape
    (R, 4, 10, 4, 50),
])
def test_fused_central_difference_bit_exact(ctx, field, d, N, trials, max_outer, monkeypatch):
    """The fused central difference of the anneal kernel (hvp_cta_gs: both points normalised side by side, the +
    point's combine inside the - point's Gram phase) against the step-by-step path (TRSTMI_NO_DUAL) and the oracle:
    every record, parameter and frame identical."""
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(field, d, N, max_outer)
    cfg.record_cap = 600
    S = api.lanes(field, d, N)
    starts, st = api.random_frames(field, d, N, 0, 0, trials)
    g = ctx.solve_batch(cfg, starts, st)
    monkeypatch.setenv("TRSTMI_NO_DUAL", "1")
    g0 = ctx.solve_batch(cfg, starts, st)
    monkeypatch.delenv("TRSTMI_NO_DUAL")
    o = orc.solve_batch(cfg, S, starts, st, threads=trials)
    _cmp_solve(g, o, trials, g["n_stages"], 600)
    _cmp_solve(g0, o, trials, g0["n_stages"], 600)


@pytest.mark.parametrize("field,d,N", [(C, 3, 100), (C, 2, 80), (C, 3, 44), (C, 2, 65), (C, 1, 35), (R, 4, 40),
                                       (C, 2, 110), (C, 8, 12), (R, 3, 7)])
def test_fused_central_difference_every_layout(ctx, field, d, N, monkeypatch):
    """The fused central difference against the step-by-step path on one shape per stored-Gram kernel family and CAS
    width (and on shapes where the dual layout is not taken): identical records, parameters and frames."""
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(field, d, N, 6)
    cfg.record_cap = 100
    starts, st = api.random_frames(field, d, N, 3, 0, 3)
    g = ctx.solve_batch(cfg, starts, st)
    monkeypatch.setenv("TRSTMI_NO_DUAL", "1")
    g0 = ctx.solve_batch(cfg, starts, st)
    monkeypatch.delenv("TRSTMI_NO_DUAL")
    _cmp_solve(g, g0, 3, g["n_stages"], 100)
    # and the single-point HVP entry, which takes the same fused path
    pts = frames_for(field, d, N, [31, 32])
    dirs = frames_for(field, d, N, [41, 42])
    hv, path, zc = ctx.hvp_batch(field, d, N, pts, dirs, 1e-2)
    monkeypatch.setenv("TRSTMI_NO_DUAL", "1")
    hv0, path0, zc0 = ctx.hvp_batch(field, d, N, pts, dirs, 1e-2)
    monkeypatch.delenv("TRSTMI_NO_DUAL")
    assert np.array_equal(bits(hv), bits(hv0)) and np.array_equal(path, path0) and np.array_equal(zc, zc0)


def test_stage_boundary_rescue(ctx):
    # test_solver.cpp:232-250: column 2 is zero; with a generator the anneal
    # recovers, without one the restart fails with ZeroColumnError(2)
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(C, 2, 3, 200, eps_target=1e-4)
    start = np.array([1.0, 0, 0, 0, 0, 0, 1.0, 0, 0, 0, 0, 0])
    from tests.oracle_ffi import lib  # noqa: F401
    rng = np.array([[8, 0, 0]], np.uint64)
    g = ctx.solve_batch(cfg, start[None], rng)
    o = orc.solve_batch(cfg, api.lanes(C, 2, 3), start[None], rng)
    assert g["trials"][0].status == abi.TRIAL_OK
    _cmp_solve(g, o, 1, g["n_stages"], 0)
    assert np.array_equal(g["rng"], o["rng"])
    g2 = ctx.solve_batch(cfg, start[None], None)
    assert g2["trials"][0].status == abi.TRIAL_ZERO_COLUMN and g2["trials"][0].zero_col == 2


def test_device_cas_math_bit_identical_to_oracle(ctx):
    import ctypes
    lib = ctx.lib
    lib.trstmi_selftest_cas_math.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int64]
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-746, 710, 400000), rng.uniform(-50, 1, 400000), -(10 ** rng.uniform(-300, 3, 100000)),
                        np.array([0.0, -0.0, -745.2, -745.13, 709.78, np.inf, -np.inf, np.nan])])
    y = np.empty_like(x)
    assert lib.trstmi_selftest_cas_math(ctx.h, 0, x.ctypes.data, y.ctypes.data, x.size) == 0
    assert np.array_equal(y.view(np.uint64), orc.exp(x).view(np.uint64))
    z = np.concatenate([rng.uniform(1, 5000, 400000), 10 ** rng.uniform(-300, 300, 400000), np.array([1.0, 2.0])])
    w = np.empty_like(z)
    assert lib.trstmi_selftest_cas_math(ctx.h, 1, z.ctypes.data, w.ctypes.data, z.size) == 0
    assert np.array_equal(w.view(np.uint64), orc.log(z).view(np.uint64))
    # hypot (coherence magnitudes, frame.hpp:87): device == oracle == the host libm, bit for bit
    pr = hypot_inputs(rng, 300000)
    h = np.empty(pr.shape[0])
    assert lib.trstmi_selftest_cas_math(ctx.h, 2, pr.ctypes.data, h.ctypes.data, pr.shape[0]) == 0
    assert np.array_equal(h.view(np.uint64), orc.hypot(pr[:, 0], pr[:, 1]).view(np.uint64))
    assert np.array_equal(h.view(np.uint64), np.hypot(pr[:, 0], pr[:, 1]).view(np.uint64))


def hypot_inputs(rng, n):
    """(x, y) pairs: coherence-range magnitudes plus the whole exponent range,
    zeros, infinities and NaN."""
    e1 = rng.integers(-1070, 1020, n)
    e2 = np.clip(e1 + rng.integers(-60, 60, n), -1074, 1020)
    a = rng.uniform(-1, 1, n) * np.ldexp(1.0, e1)
    b = rng.uniform(-1, 1, n) * np.ldexp(1.0, e2)
    m = rng.uniform(-1, 1, (n, 2))
    special = np.array([[0.0, 0.0], [-0.0, 3.0], [np.inf, np.nan], [np.nan, 1.0], [1e-320, 1e-321], [1e308, 1e308]])
    return np.ascontiguousarray(np.concatenate([np.stack([a, b], 1), m, special]))


def test_markstein_division_matches_ieee(ctx):
    """The kernels divide by delta, z and alpha through a precomputed
    reciprocal + one fma correction; it must equal IEEE division bit for bit."""
    import ctypes
    lib = ctx.lib
    lib.trstmi_selftest_division.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
    bad = ctypes.c_uint64()
    assert lib.trstmi_selftest_division(ctx.h, 1 << 31, 20250809, ctypes.byref(bad)) == 0
    assert bad.value == 0


@pytest.mark.parametrize("field,d,N", [(C, 1, 2), (R, 1, 2), (C, 5, 2), (R, 16, 3), (C, 16, 17)])
def test_edge_shapes_bit_exact(ctx, field, d, N):
    """Smallest pair counts (N = 2: one pair), d = 1, and the runtime-d kernel family (d = 16)."""
    from paper_2207_06374_b200 import api
    S = api.lanes(field, d, N)
    pts = np.stack([orc.random_test_frame(field, d, N, s) for s in (1, 2)])
    for delta in (1e-1, 1e-7):
        F, s, g, w, zc = ctx.eval_batch(field, d, N, pts, delta, True, True)
        for b in range(2):
            Fo, so, go, wo, zo = orc.eval_objective(field, d, N, S, pts[b], delta, want_weights=True)
            assert bits(F[b]) == bits(Fo) and np.array_equal(bits(g[b]), bits(go))
    cfg = abi.default_cfg(field, d, N, 30)
    cfg.record_cap = 300
    starts, st = api.random_frames(field, d, N, 0, 0, 3)
    _cmp_solve(ctx.solve_batch(cfg, starts, st), orc.solve_batch(cfg, S, starts, st, threads=3), 3,
               api.default_schedule_len(N), 300)


def test_nonfinite_start_fails_like_the_reference(ctx):
    """A NaN entry makes the stage's x0 evaluation non-finite:
    trust_region_minimize throws invalid_argument (trust_region.hpp:206-209)."""
    from paper_2207_06374_b200 import api
    cfg = abi.default_cfg(C, 2, 6, 10)
    starts, st = api.random_frames(C, 2, 6, 0, 0, 2)
    starts[1, 3] = np.nan
    g = ctx.solve_batch(cfg, starts, st)
    o = orc.solve_batch(cfg, api.lanes(C, 2, 6), starts, st, threads=2)
    assert g["trials"][0].status == o["trials"][0].status == abi.TRIAL_OK
    assert g["trials"][1].status == o["trials"][1].status


# one shape per (kernel layout, CAS width) the dispatcher can pick
# (trstmi_small_layout: 0 Gram recomputed, 1 stored Gram, 2 stored Gram in
# bank-padded rows): the same bits whichever layout runs
LAYOUTS = [(C, 1, 128, 0, 128), (C, 1, 140, 0, 256), (C, 1, 116, 1, 128), (C, 2, 110, 1, 256),
           (C, 3, 100, 1, 512), (C, 2, 80, 2, 512), (C, 3, 44, 2, 128), (C, 2, 65, 2, 256), (C, 1, 35, 2, 128),
           (R, 4, 10, 2, 64),
           (R, 2, 150, 0, 256), (R, 4, 40, 2, 128)]


@pytest.mark.parametrize("field,d,N,layout,lanes", LAYOUTS)
def test_every_layout_bit_exact(ctx, field, d, N, layout, lanes):
    from paper_2207_06374_b200 import api
    assert api.small_layout(field, d, N) == layout and api.lanes(field, d, N) == lanes
    S = lanes
    pts = frames_for(field, d, N, [21, 22])
    for delta in (1e-1, 1e-5):
        F, s, g, w, zc = ctx.eval_batch(field, d, N, pts, delta, True, True)
        for b in range(pts.shape[0]):
            Fo, so, go, wo, zo = orc.eval_objective(field, d, N, S, pts[b], delta, want_weights=True)
            assert bits(F[b]) == bits(Fo) and np.array_equal(bits(g[b]), bits(go))
            assert np.array_equal(bits(w[b]), bits(wo))
    dirs = frames_for(field, d, N, [31, 32])
    hv, path, zc = ctx.hvp_batch(field, d, N, pts, dirs, 1e-3)
    for b in range(pts.shape[0]):
        ho, po, zo = orc.hvp(field, d, N, S, pts[b], dirs[b], 1e-3)
        assert path[b] == po and np.array_equal(bits(hv[b]), bits(ho))
    cfg = abi.default_cfg(field, d, N, 8)
    cfg.record_cap = 400
    starts, st = api.random_frames(field, d, N, 0, 0, 2)
    gr = ctx.solve_batch(cfg, starts, st)
    o = orc.solve_batch(cfg, S, starts, st)
    _cmp_solve(gr, o, 2, gr["n_stages"], 400)
