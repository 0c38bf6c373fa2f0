"""Times a few outer iterations of the large-frame path and prints CG lengths.
python scripts/large_probe.py FIELD D N TRIALS MAX_OUTER N_STAGES"""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2207_06374_b200 import abi, api  # noqa: E402

field, d, N, T, mo, ns = (int(a) for a in sys.argv[1:7])
ctx = api.Context(0)
cfg = abi.default_cfg(field, d, N, mo)
sched = api.default_schedule(N)
cfg.n_stages = ns
for k in range(ns):
    cfg.schedule[k] = sched[k]
cfg.record_cap = 64
starts, st = api.random_frames(field, d, N, 0, 0, T)
t0 = time.time()
g = ctx.solve_batch(cfg, starts, st)
dt = time.time() - t0
outer = sum(g["trials"][t].outer_iterations for t in range(T))
ev = sum(g["trials"][t].evals for t in range(T))
print(f"{field},{d},{N} T={T}: {dt:.2f}s outer={outer} evals={ev} TRit/s={outer / dt:.3g} evals/s={ev / dt:.3g} "
      f"alg TFLOP/s={ev * (16 if field == 0 else 4) * d * N * N / dt / 1e12:.2f}")
for t in range(min(T, 3)):
    r = g["trials"][t]
    recs = [(g["outer"][t * 64 + i].cg_iterations, g["outer"][t * 64 + i].cg_exit) for i in range(r.records)]
    print("  trial", t, "status", r.status, "mu", r.coherence, "cg", recs[:12])
