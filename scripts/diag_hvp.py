"""Diagnostic: large-path HVP vs the oracle at several shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_06374_b200 import api, abi
from tests import oracle_ffi as orc
ctx = api.Context(0)
for (field, d, N) in [(1, 64, 1024), (1, 20, 300), (0, 17, 200), (1, 64, 256), (1, 17, 1024)]:
    S = api.lanes(field, d, N)
    x = orc.random_test_frame(field, d, N, 5)
    v = np.random.default_rng(1).standard_normal(x.size); v /= np.linalg.norm(v)
    for delta in (0.1, 1e-5):
        hv, path, zc = ctx.hvp_batch(field, d, N, x[None], v[None], delta)
        ho, po, zo = orc.hvp(field, d, N, S, x, v, delta)
        F, s, g, _, z = ctx.eval_batch(field, d, N, x[None], delta, True, False)
        Fo, so, go, _, zo2 = orc.eval_objective(field, d, N, S, x, delta)
        print((field, d, N, S, delta), "hvp equal:", np.array_equal(hv[0], ho), "maxrel", np.max(np.abs(hv[0]-ho))/np.max(np.abs(ho)),
              "eval equal:", np.array_equal(g[0], go), F[0] == Fo, flush=True)
