"""Runs one batched anneal (for ncu / sanitizer captures).  Usage:
python scripts/run_solve.py FIELD D N TRIALS MAX_OUTER [N_STAGES]"""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2207_06374_b200 import abi, api  # noqa: E402

field, d, N, T, mo = (int(a) for a in sys.argv[1:6])
ns = int(sys.argv[6]) if len(sys.argv) > 6 else 0
ctx = api.Context(0)
cfg = abi.default_cfg(field, d, N, mo)
if ns:
    sched = api.default_schedule(N)[:ns]
    cfg.n_stages = ns
    for k, v in enumerate(sched):
        cfg.schedule[k] = v
starts, st = api.random_frames(field, d, N, 0, 0, T)
t0 = time.time()
g = ctx.solve_batch(cfg, starts, st)
dt = time.time() - t0
outer = sum(g["trials"][t].outer_iterations for t in range(T))
ev = sum(g["trials"][t].evals for t in range(T))
print(f"{dt:.3f}s outer={outer} evals={ev} evals/s={ev / dt:.3g}")
