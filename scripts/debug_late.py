import sys, time, ctypes
sys.path.insert(0, '.')
from paper_2207_06374_b200 import abi, api
field, d, N, T = (int(a) for a in sys.argv[1:5])
mo2 = int(sys.argv[5]) if len(sys.argv) > 5 else 20
lib = api.load_library(); lib.trstmi_launch_count.restype = ctypes.c_longlong
ctx = api.Context(0)
cfg = abi.default_cfg(field, d, N, 60)
starts, st = api.random_frames(field, d, N, 0, 0, T)
t0 = time.time(); g = ctx.solve_batch(cfg, starts, st); print("first", time.time()-t0, "launches", lib.trstmi_launch_count(), flush=True)
sched = api.default_schedule(N)
cfg2 = abi.default_cfg(field, d, N, mo2)
cfg2.n_stages = 1
cfg2.schedule[0] = sched[-1]
t0 = time.time()
g2 = ctx.solve_batch(cfg2, g["params"], g["rng"])
dt = time.time() - t0
print("second", dt, "launches", lib.trstmi_launch_count(), flush=True)
from collections import Counter
print(Counter(g2["trials"][t].status for t in range(T)))
ev = [g2["trials"][t].evals for t in range(T)]; ou=[g2["trials"][t].outer_iterations for t in range(T)]
print("evals min/max", min(ev), max(ev), "outer min/max", min(ou), max(ou))
