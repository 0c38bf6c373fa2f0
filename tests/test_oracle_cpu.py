"""CPU tests of the oracle (test infrastructure) against the reference's own
known-answer / property tests and against independent restatements."""
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2207_06374_b200 import abi
from tests import oracle_ffi as orc

C, R = abi.COMPLEX, abi.REAL


def test_ported_reference_unit_tests():
    """oracle/tests/oracle_tests.cpp ports test_smoothing / test_trust_region /
    test_solver / test_frames / acceptance criteria 1 and 7."""
    orc.build_oracle()
    exe = os.path.join(orc.ORACLE_DIR, "_build", "oracle_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 failures" in r.stdout


def test_cas_hypot_matches_libm():
    """CAS |G| for coherence is glibc's hypot restated (std::abs(complex),
    frame.hpp:87): bit-identical to this host's libm over the exponent range."""
    from tests.test_gpu_parity import hypot_inputs
    pr = hypot_inputs(np.random.default_rng(11), 400000)
    h = orc.hypot(pr[:, 0], pr[:, 1])
    assert np.array_equal(h.view(np.uint64), np.hypot(pr[:, 0], pr[:, 1]).view(np.uint64))


def test_cas_exp_accuracy_vs_mpmath():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 160
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-745.1, 709.7, 3000), rng.uniform(-40, 0, 3000), rng.uniform(-1, 1, 2000),
                        rng.uniform(-745.13, -708, 1000)])
    y = orc.exp(x)
    worst = 0.0
    for xi, yi in zip(x, y):
        ref = mpmath.exp(mpmath.mpf(float(xi)))
        u = math.ulp(float(ref)) if float(ref) != 0 else 5e-324
        worst = max(worst, float(abs(mpmath.mpf(float(yi)) - ref) / u))
    assert worst <= 1.0, worst
    assert orc.exp(np.array([0.0]))[0] == 1.0
    assert orc.exp(np.array([-746.0]))[0] == 0.0      # the underflow cut is exact
    assert np.isinf(orc.exp(np.array([710.0]))[0])


def test_cas_log_accuracy_vs_mpmath():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 160
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.uniform(1, 1e4, 3000), 10 ** rng.uniform(-300, 300, 3000), rng.uniform(0.5, 2, 2000)])
    y = orc.log(x)
    worst = 0.0
    for xi, yi in zip(x, y):
        ref = mpmath.log(mpmath.mpf(float(xi)))
        worst = max(worst, float(abs(mpmath.mpf(float(yi)) - ref) / math.ulp(float(ref))))
    assert worst <= 2.0, worst
    assert orc.log(np.array([1.0]))[0] == 0.0


def _fma(a, b, c):
    """correctly rounded a*b+c (exact rational arithmetic, one rounding)"""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _py_cas_sum(v, S, dot_with=None):
    lane = [0.0] * S
    for p, x in enumerate(v):
        if dot_with is None:
            lane[p % S] = lane[p % S] + x
        else:
            lane[p % S] = _fma(x, dot_with[p], lane[p % S])
    tot = []
    for w in range(S // 32):
        a = lane[32 * w:32 * w + 32]
        for off in (16, 8, 4, 2, 1):
            a = [a[l] + a[l ^ off] for l in range(32)]
        tot.append(a[0])
    off = 1
    while off < len(tot):
        tot = [tot[w] + tot[w ^ off] for w in range(len(tot))]
        off *= 2
    return tot[0]


@pytest.mark.parametrize("S", [32, 128, 256, 512])
def test_cas_reduction_shape(S):
    rng = np.random.default_rng(S)
    for n in (1, 31, 400, 4950):
        v = rng.standard_normal(n) * 10.0 ** rng.uniform(-5, 5, n)
        w = rng.standard_normal(n)
        assert orc.cas_sum(v, S) == _py_cas_sum(list(v), S)
        assert orc.cas_dot(v, w, S) == _py_cas_sum(list(v), S, list(w))


def _py_splitmix(seed, n):
    M = (1 << 64) - 1
    s = seed
    out = []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append((z ^ (z >> 31)) >> 11)
    return [x * 2.0 ** -53 for x in out]


def test_rng_matches_independent_splitmix():
    """rng.hpp:26-34 restated independently in Python."""
    assert list(orc.uniforms(12345, 50)) == _py_splitmix(12345, 50)
    u = _py_splitmix(7, 2)
    r = math.sqrt(-2.0 * math.log(u[0]))
    n = orc.normals(7, 2)
    assert abs(n[0] - r * math.cos(2 * math.pi * u[1])) < 1e-15
    assert abs(n[1] - r * math.sin(2 * math.pi * u[1])) < 1e-15


def test_mix_seed_and_schedule():
    L = orc.lib()
    assert L.orc_mix_seed(0, 0) == 0xE220A8397B1DCDAF  # splitmix64 of the golden-ratio increment
    s = orc.schedule(100, 1e-7)
    assert len(s) == 8 and s[0] == 0.1
    assert abs(s[-1] - 1e-7 / (2 * math.log(100))) < 1e-22


def test_welch():
    L = orc.lib()
    assert abs(L.orc_welch_bound(6, 36) - 1 / math.sqrt(7)) < 1e-15
    assert L.orc_welch_bound(3, 3) == 0.0


@pytest.mark.parametrize("d,N", [(3, 6), (4, 10), (2, 7)])
def test_real_mode_equals_complex_embedding(d, N):
    """real lines == complex code with Im == 0 (value and
    gradient to 1e-12; identical Gram, so identical coherence)."""
    S = 32
    xr = orc.normals(d * 100 + N, d * N)
    xc = np.zeros(2 * d * N)
    xc[0::2] = xr
    for delta in (1e-1, 1e-3):
        Fr, sr, gr, _, _ = orc.eval_objective(R, d, N, S, xr, delta)
        Fc, sc, gc, _, _ = orc.eval_objective(C, d, N, S, xc, delta)
        assert abs(Fr - Fc) <= 1e-12 * max(1.0, abs(Fc))
        assert sr == sc
        assert np.max(np.abs(gr - gc[0::2])) <= 1e-12 * max(1.0, np.max(np.abs(gc)))
        assert np.all(gc[1::2] == 0.0)
    mr, ar, _ = orc.coherence(R, d, N, xr, True)
    mc, ac, _ = orc.coherence(C, d, N, xc, True)
    assert mr == mc and ar == ac


def test_gradient_vs_numpy_reference_formula():
    """An independent float64 numpy restatement of smoothing.hpp:82-162."""
    d, N, delta = 3, 7, 1e-2
    x = orc.random_test_frame(C, d, N, 99) * 1.3
    F, s, g, w, _ = orc.eval_objective(C, d, N, 32, x, delta, want_weights=True)
    A = (x[0::2] + 1j * x[1::2]).reshape(N, d).T
    alpha = np.linalg.norm(A, axis=0)
    phi = A / alpha
    G = phi.conj().T @ phi
    iu = np.triu_indices(N, 1)
    u = np.abs(G[iu]) ** 2
    smax = u.max()
    ww = np.exp((u - smax) / delta)
    z = ww.sum()
    c = ww / z
    Fn = smax + delta * np.log(z)
    C_ = np.zeros((N, N), complex)
    C_[iu] = c * G[iu]
    C_[(iu[1], iu[0])] = c * G[(iu[1], iu[0])]
    t = np.zeros(N)
    np.add.at(t, iu[0], c * u)
    np.add.at(t, iu[1], c * u)
    D = (phi @ C_ - phi * t) / alpha
    gn = np.empty(2 * d * N)
    gn[0::2] = 2 * D.T.reshape(-1).real
    gn[1::2] = 2 * D.T.reshape(-1).imag
    assert abs(F - Fn) < 1e-14 and s == pytest.approx(smax, abs=1e-15)
    assert np.max(np.abs(g - gn)) < 1e-12
    assert np.max(np.abs(w - c)) < 1e-14
