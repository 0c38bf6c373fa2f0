"""Alternating-projection baseline, CPU side: the oracle restatement (oracle/altproj_oracle.hpp) against the
reference's own expectations for the path (/root/reference/proj/tests/test_baseline.cpp) and against an independent
numpy restatement of baseline.hpp:68-167 that uses numpy.linalg.eigh where the reference uses Eigen's
SelfAdjointEigenSolver.  (The reference's baseline cannot be compiled here: DESIGN.md §5.)"""
import math

import numpy as np
import pytest

from paper_2207_06374_b200 import abi
from tests import oracle_ffi as orc

C = abi.COMPLEX


def _cplx(frame, d, N):
    return frame.reshape(N, d, 2)[..., 0].T + 1j * frame.reshape(N, d, 2)[..., 1].T  # d x N


def _welch(d, N):
    return 0.0 if N <= d else math.sqrt((N - d) / (d * (N - 1)))


def numpy_altproj(d, N, start, max_iters=300, mu_target=0.0, tol=1e-10):
    """baseline.hpp:84-150 with numpy.linalg.eigh; returns (best_coherence, +-iterations)."""
    target = mu_target if mu_target > 0 else max(_welch(d, N), 1e-12)
    F = _cplx(start, d, N)
    G = F.conj().T @ F

    def coh(Fm):
        A = np.abs(Fm.conj().T @ Fm)
        np.fill_diagonal(A, 0.0)
        return A.max() if N > 1 else 0.0

    best = last = coh(F)
    for it in range(max_iters):
        mag = np.abs(G)
        scale = np.where(mag > target, target / np.maximum(mag, 1e-300), 1.0)
        G = G * scale
        np.fill_diagonal(G, 1.0)
        lam, vec = np.linalg.eigh(G)
        lam_top = np.maximum(lam[::-1][:d], 0.0)
        V = vec[:, ::-1][:, :d]
        P = (V * lam_top) @ V.conj().T
        fac = (np.sqrt(lam_top)[:, None] * V.conj().T)
        norms = np.linalg.norm(fac, axis=0)
        if norms.min() >= 1e-12:
            last = coh(fac / norms)
            best = min(best, last)
        change = np.abs(P - G).max()
        G = P
        if change <= tol:
            return last, it + 1
    return best, -max_iters


@pytest.mark.parametrize("d,N,seed,restarts", [(2, 4, 7, 3), (3, 7, 1, 2), (3, 9, 42, 2), (4, 6, 3, 2), (2, 2, 5, 1)])
def test_oracle_matches_numpy_restatement(d, N, seed, restarts):
    starts, _ = orc.random_frames(C, d, N, seed, 0, restarts)
    frames, mu, it, _ = orc.altproj_batch(d, N, starts, max_iters=40)
    for r in range(restarts):
        mu_np, it_np = numpy_altproj(d, N, starts[r], max_iters=40)
        assert it[r] == it_np
        assert abs(mu[r] - mu_np) <= 1e-8, (mu[r], mu_np)
        # the returned frame has unit columns and the reported coherence (test_baseline.cpp:24-35)
        F = _cplx(frames[r], d, N)
        assert np.allclose(np.linalg.norm(F, axis=0), 1.0, atol=1e-10)
        A = np.abs(F.conj().T @ F)
        np.fill_diagonal(A, 0.0)
        assert abs(A.max() - mu[r]) <= 1e-12


def test_orthonormal_basis_at_N_equals_d():
    # test_baseline.cpp:12-17 (generator SplitMix64(17))
    start = orc.random_test_frame(C, 3, 3, 17)
    frames, mu, it, _ = orc.altproj_batch(3, 3, start[None])
    assert mu[0] <= 1e-6 and it[0] > 0
    F = _cplx(frames[0], 3, 3)
    assert np.allclose(np.linalg.norm(F, axis=0), 1.0, atol=1e-10)


def test_reaches_the_2_4_optimum():
    # test_baseline.cpp:19-22: solve_altproj(2, 4, {}, 3, 7)
    starts, _ = orc.random_frames(C, 2, 4, 7, 0, 3)
    _, mu, _, _ = orc.altproj_batch(2, 4, starts)
    assert mu.min() <= 0.5774 + 5e-3


def test_respects_the_welch_bound():
    # test_baseline.cpp:24-35
    for seed in (1, 2):
        start = orc.random_test_frame(C, 3, 7, seed)
        _, mu, _, _ = orc.altproj_batch(3, 7, start[None])
        assert mu[0] >= _welch(3, 7) - 1e-9


def test_budget_quality_at_5_25():
    # baseline.hpp:17-21: the 300-iteration budget leaves (5, 25) near 0.45; acceptance criterion 6 needs a gap
    # of >= 0.02 to the solver's ~0.41 (acceptance_main.cpp:158-168)
    starts, _ = orc.random_frames(C, 5, 25, 20240607, 0, 1)
    _, mu, it, _ = orc.altproj_batch(5, 25, starts)
    assert it[0] == -300 and 0.43 <= mu[0] <= 0.47
