import time, numpy as np, sys
sys.path.insert(0,'.')
from paper_2207_06374_b200 import api, abi
ctx = api.Context(0)
for (field,d,N,T,mo) in [(abi.REAL,4,10,64,200),(abi.COMPLEX,6,36,1024,1000),(abi.COMPLEX,2,100,4096,500)]:
    cfg = abi.default_cfg(field,d,N,mo)
    starts, st = api.random_frames(field,d,N,0,0,T)
    t0=time.time(); g = ctx.solve_batch(cfg, starts, st); dt=time.time()-t0
    outer = sum(g["trials"][t].outer_iterations for t in range(T)); ev = sum(g["trials"][t].evals for t in range(T))
    mus = np.array([g["trials"][t].coherence for t in range(T)])
    print(f"{field},{d},{N} T={T}: {dt:.2f}s outer={outer} evals={ev} TRit/s={outer/dt:.3g} evals/s={ev/dt:.3g} best mu={mus.min():.9f} statuses={set(g['trials'][t].status for t in range(T))}", flush=True)
