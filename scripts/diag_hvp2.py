import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_06374_b200 import api, abi
from tests import oracle_ffi as orc
ctx = api.Context(0)
field, d, N = 1, 64, 1024
S = api.lanes(field, d, N)
x = api.random_frames(field, d, N, 0, 0, 1)[0][0]
r0 = np.random.default_rng(1000).standard_normal(x.size); v = r0 / np.linalg.norm(r0)
delta = 0.1
hv, path, zc = ctx.hvp_batch(field, d, N, x[None], v[None], delta)
ho, po, zo = orc.hvp(field, d, N, S, x, v, delta)
bad = np.nonzero(hv[0] != ho)[0]
print("hvp mismatches", bad.size, bad[:10], np.max(np.abs(hv[0]-ho)) if bad.size else 0)
dn = np.sqrt(orc.cas_dot(v, v, S)); xn = np.sqrt(orc.cas_dot(x, x, S))
h = 6.0554544523933395e-06 * (1.0 + xn) / max(dn, 1e-300)
print("h", repr(h), "dn", repr(dn), "xn", repr(xn))
for sgn in (1, -1):
    p = x + (sgn * h) * v
    F, s, g, _, z = ctx.eval_batch(field, d, N, p[None], delta, True, False)
    Fo, so, go, _, z2 = orc.eval_objective(field, d, N, S, p, delta)
    print(sgn, "eval at materialised point equal:", np.array_equal(g[0], go), F[0] == Fo, s[0] == so)
    Fd, sd, gd, _, zd = orc.eval_objective(field, d, N, S, x, delta, direction=v, sc=sgn * h)
    print(sgn, "oracle direction form == materialised:", np.array_equal(gd, go))
