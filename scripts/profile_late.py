"""Two anneal launches: (1) a short full anneal of T trials to get converged
frames, (2) a single terminal-delta stage from those frames (the regime that
dominates a full C2 solve).  Profile launch (2) with ncu -k regex:anneal -s 1 -c 1."""
import sys
import time

sys.path.insert(0, '.')
from paper_2207_06374_b200 import abi, api  # noqa: E402

field, d, N, T = (int(a) for a in sys.argv[1:5])
mo2 = int(sys.argv[5]) if len(sys.argv) > 5 else 20
ctx = api.Context(0)
cfg = abi.default_cfg(field, d, N, 60)
starts, st = api.random_frames(field, d, N, 0, 0, T)
g = ctx.solve_batch(cfg, starts, st)
sched = api.default_schedule(N)
cfg2 = abi.default_cfg(field, d, N, mo2)
cfg2.n_stages = 1
cfg2.schedule[0] = sched[-1]
t0 = time.time()
g2 = ctx.solve_batch(cfg2, g["params"], g["rng"])
dt = time.time() - t0
ev = sum(g2["trials"][t].evals for t in range(T))
outer = sum(g2["trials"][t].outer_iterations for t in range(T))
print(f"late stage: {dt:.3f}s outer={outer} evals={ev} evals/s={ev/dt:.3g} evals/outer={ev/max(outer,1):.1f}")
