"""GPU parity at the five BASELINE.json config shapes, at FULL size
(config 5: d = 128, N = 4096), against both oracles:

  * the CAS oracle, bit for bit — through sha256 digests of its outputs
    committed in tests/golden/reference_pin.json (the CPU oracle takes ~8 s per
    config-5 evaluation, so the digests are generated once, here:
    tests/golden/make_reference_pin.py);
  * the reference itself (its headers compiled unchanged against the
    Eigen-API shim, oracle/_ref) at the north star's tolerances: objective
    and gradient within 1e-10 relative, coherence within 1e-12 absolute,
    argmax pair exact.

The delta values are the first, middle and terminal stages of each config's
default schedule (terminal: 2.2e-8 .. 6.0e-9).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from tests.test_reference_pin import rel_checks

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_pin.json")
PIN = json.load(open(GOLDEN))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ctx():
    from paper_2207_06374_b200 import api
    c = api.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_eval_full_size_vs_oracle_and_reference(ctx, name):
    from paper_2207_06374_b200 import api
    c = PIN["configs"][name]
    field, d, N = c["field"], c["d"], c["N"]
    x = api.random_frames(field, d, N, 0, 0, 1)[0][0]
    assert sha(x) == c["frame_sha256"]
    idx = np.asarray(c["sample_idx"])
    for e in c["evals"]:
        F, s, g, _, zc = ctx.eval_batch(field, d, N, x[None], e["delta"], True, False)
        assert zc[0] == -1
        assert sha([F[0], s[0]]) == e["cas"]["F_bits_sha256"], (F[0], e["cas"]["F"])
        assert sha(g[0]) == e["cas"]["grad_sha256"], "gradient not bit-identical to the CAS oracle"
        assert abs(F[0] - e["ref"]["F"]) <= 1e-10 * abs(e["ref"]["F"])
        rel_checks(g[0], e, idx)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_coherence_full_size_vs_reference(ctx, name):
    from paper_2207_06374_b200 import api
    c = PIN["configs"][name]
    field, d, N = c["field"], c["d"], c["N"]
    x = api.random_frames(field, d, N, 0, 0, 1)[0][0]
    mu, arg, zc = ctx.coherence_batch(field, d, N, x[None], normalize=False)
    assert zc[0] == -1
    assert abs(mu[0] - c["mu"]) <= 1e-12 and arg[0] == c["argmax_pair"]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_hvp_full_size_vs_oracle_and_reference(ctx, name):
    from paper_2207_06374_b200 import abi, api
    c = PIN["configs"][name]
    field, d, N = c["field"], c["d"], c["N"]
    x = api.random_frames(field, d, N, 0, 0, 1)[0][0]
    r0 = np.random.default_rng(1000).standard_normal(x.size)
    v = r0 * 0.00390625  # as the generator: exact scaling (a BLAS norm may differ by an ulp across hosts)
    idx = np.asarray(c["sample_idx"])
    for e in c["evals"]:
        hv, path, zc = ctx.hvp_batch(field, d, N, x[None], v[None], e["delta"])
        assert path[0] == abi.HVP_CENTRAL
        assert sha(hv[0]) == e["hvp"]["cas_sha256"], "HVP not bit-identical to the CAS oracle"
        hs = np.asarray(e["hvp"]["ref_samples"])
        # the 1/(2h) ~ 1e5 FD amplification of ulp-level gradient differences
        assert abs(np.linalg.norm(hv[0]) - e["hvp"]["ref_norm"]) <= 1e-7 * e["hvp"]["ref_norm"]
        assert np.linalg.norm(hv[0][idx] - hs) <= 1e-6 * max(np.linalg.norm(hs), 1e-300)
