"""Alternating-projection baseline on the GPU (csrc/altproj.cu, paper_2207_06374_b200/baseline.py): bit-exact against
the CPU oracle (oracle/altproj_oracle.hpp) and the reference's own test cases for the path
(/root/reference/proj/tests/test_baseline.cpp, tests/test_cli.cpp:226-240)."""
import json
import math

import numpy as np
import pytest

from paper_2207_06374_b200 import abi
from tests import oracle_ffi as orc

pytestmark = pytest.mark.gpu
C = abi.COMPLEX


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _cplx(frame, d, N):
    return frame.reshape(N, d, 2)[..., 0].T + 1j * frame.reshape(N, d, 2)[..., 1].T


def _coh(frame, d, N):
    F = _cplx(frame, d, N)
    A = np.abs(F.conj().T @ F)
    np.fill_diagonal(A, 0.0)
    return A.max()


@pytest.mark.parametrize("d,N,seed,restarts,max_iters", [
    (2, 4, 7, 3, 300), (3, 3, 17, 2, 300), (3, 7, 1, 3, 300), (3, 9, 42, 2, 300), (5, 25, 20240607, 2, 300),
    (4, 16, 3, 2, 60), (2, 33, 9, 2, 25), (6, 36, 11, 1, 20),   # odd N (padded round-robin), config-3 shape
])
def test_altproj_bit_exact_vs_oracle(d, N, seed, restarts, max_iters):
    from paper_2207_06374_b200 import api, baseline
    starts, _ = api.random_frames(C, d, N, seed, 0, restarts)
    cfg = baseline.AltProjConfig(max_iters=max_iters)
    frames, mu, it, sw = baseline.altproj_batch(d, N, cfg, starts)
    fo, muo, ito, swo = orc.altproj_batch(d, N, starts, max_iters=max_iters)
    assert np.array_equal(it, ito) and np.array_equal(sw, swo)
    assert np.array_equal(bits(mu), bits(muo))
    assert np.array_equal(bits(frames), bits(fo))


def test_custom_target_and_tolerance_bit_exact():
    from paper_2207_06374_b200 import api, baseline
    starts, _ = api.random_frames(C, 3, 8, 5, 0, 2)
    cfg = baseline.AltProjConfig(max_iters=80, mu_target=0.55, tol=1e-6)
    frames, mu, it, _ = baseline.altproj_batch(3, 8, cfg, starts)
    fo, muo, ito, _ = orc.altproj_batch(3, 8, starts, max_iters=80, mu_target=0.55, tol=1e-6)
    assert np.array_equal(it, ito) and np.array_equal(bits(mu), bits(muo)) and np.array_equal(bits(frames), bits(fo))


def test_orthonormal_basis_at_N_equals_d():
    # test_baseline.cpp:12-17
    from paper_2207_06374_b200 import baseline
    res = baseline.alternating_projection(3, 3, baseline.AltProjConfig(), 17)
    assert res.best_coherence <= 1e-6
    assert np.allclose(np.linalg.norm(_cplx(res.best_frame, 3, 3), axis=0), 1.0, atol=1e-10)


def test_reaches_the_2_4_optimum():
    # test_baseline.cpp:19-22
    from paper_2207_06374_b200 import baseline
    res = baseline.solve_altproj(2, 4, baseline.AltProjConfig(), 3, 7)
    assert res.best_coherence <= 0.5774 + 5e-3
    assert res.best_restart == int(np.argmin([r.coherence for r in res.per_restart]))


def test_normalized_and_welch_bound():
    # test_baseline.cpp:24-35
    from paper_2207_06374_b200 import baseline
    for seed in (1, 2):
        res = baseline.alternating_projection(3, 7, baseline.AltProjConfig(), seed)
        assert np.allclose(np.linalg.norm(_cplx(res.best_frame, 3, 7), axis=0), 1.0, atol=1e-10)
        assert res.best_coherence >= math.sqrt(4 / 18) - 1e-9
        assert abs(res.best_coherence - _coh(res.best_frame, 3, 7)) <= 1e-12


def test_deterministic_given_the_seed():
    # test_baseline.cpp:65-70
    from paper_2207_06374_b200 import baseline
    a = baseline.solve_altproj(3, 9, baseline.AltProjConfig(), 2, 42)
    b = baseline.solve_altproj(3, 9, baseline.AltProjConfig(), 2, 42)
    assert a.best_coherence == b.best_coherence and np.array_equal(bits(a.best_frame), bits(b.best_frame))
    assert [r.seed for r in a.per_restart] == [orc.mix_seed(42, 0), orc.mix_seed(42, 1)]
    st = a.per_restart[0].stages[0]
    assert st.delta == 0.0 and st.objective == a.per_restart[0].coherence ** 2 and st.outer_iterations == -300


def test_config_validation():
    # test_baseline.cpp:72-84: the reference throws std::invalid_argument
    from paper_2207_06374_b200 import baseline
    with pytest.raises(ValueError):
        baseline.alternating_projection(2, 4, baseline.AltProjConfig(max_iters=0), 1)
    with pytest.raises(ValueError):
        baseline.alternating_projection(2, 4, baseline.AltProjConfig(mu_target=1.5), 1)
    with pytest.raises(ValueError):
        baseline.alternating_projection(4, 3, baseline.AltProjConfig(), 1)
    with pytest.raises(ValueError):
        baseline.solve_altproj(2, 4, baseline.AltProjConfig(), 0, 1)


def test_gap_to_the_solver_at_5_25():
    # acceptance criterion 6 (acceptance_main.cpp:158-168): altproj(5,25) - trstmi(5,25) >= 0.02
    from paper_2207_06374_b200 import baseline
    from paper_2207_06374_b200 import records as rec
    base = baseline.solve_altproj(5, 25, baseline.AltProjConfig(), 1, 20240607)
    cfg = abi.default_cfg(C, 5, 25, 200)
    ours = rec.solve(cfg, restarts=8, seed=20240607)
    assert base.best_coherence - ours.best_coherence >= 0.02


def test_cli_altproj_record(tmp_path, capsys):
    # test_cli.cpp:226-240
    from paper_2207_06374_b200 import cli
    out = tmp_path / "ap.json"
    rc = cli.main(["solve", "--d", "2", "--N", "4", "--method", "altproj", "--restarts", "2", "--seed", "5",
                   "--out", str(out)])
    assert rc == 0
    record = json.loads(out.read_text())
    assert record["method"] == "altproj"
    assert record["config"]["max_iters"] == 300 and record["config"]["restarts"] == 2
    assert len(record["per_restart"]) == 2
    assert record["best_coherence"] <= 0.5774 + 5e-2
