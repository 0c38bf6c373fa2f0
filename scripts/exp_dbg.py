import sys, ctypes, numpy as np
sys.path.insert(0, '.')
from paper_2207_06374_b200 import api
from tests import oracle_ffi as orc
ctx = api.Context(0); lib = ctx.lib
lib.trstmi_selftest_cas_math.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
rng = np.random.default_rng(7)
x = np.concatenate([rng.uniform(-746, 710, 400000), rng.uniform(-50, 1, 400000), -(10 ** rng.uniform(-300, 3, 100000)),
                    np.array([0.0, -0.0, -745.2, -745.13, 709.78, np.inf, -np.inf, np.nan])])
y = np.empty_like(x)
lib.trstmi_selftest_cas_math(ctx.h, 0, x.ctypes.data, y.ctypes.data, x.size)
o = orc.exp(x)
bad = np.nonzero(y.view(np.uint64) != o.view(np.uint64))[0]
print("mismatches", len(bad))
for i in bad[:20]: print(repr(x[i]), repr(y[i]), repr(o[i]), np.exp(x[i]))
z = np.concatenate([rng.uniform(1, 5000, 400000), 10 ** rng.uniform(-300, 300, 400000), np.array([1.0, 2.0])])
w = np.empty_like(z)
print("rc", lib.trstmi_selftest_cas_math(ctx.h, 1, z.ctypes.data, w.ctypes.data, z.size))
ol = orc.log(z)
bad = np.nonzero(w.view(np.uint64) != ol.view(np.uint64))[0]
print("log mismatches", len(bad))
for i in bad[:10]: print(repr(z[i]), repr(w[i]), repr(ol[i]))
