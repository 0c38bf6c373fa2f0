"""Times the single-point eval kernel (one CTA per point) in isolation.
python scripts/bench_eval.py FIELD D N DELTA [B]"""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2207_06374_b200 import abi, api  # noqa: E402

field, d, N = (int(a) for a in sys.argv[1:4])
delta = float(sys.argv[4])
B = int(sys.argv[5]) if len(sys.argv) > 5 else 148 * 64
ctx = api.Context(0)
lib = ctx.lib
f, _ = api.random_frames(field, d, N, 0, 0, 64)
dim = abi.dim_of(field, d, N)
pts = torch.from_numpy(f).cuda().repeat((B + 63) // 64, 1)[:B].contiguous()
dl = torch.full((B,), delta, dtype=torch.float64, device="cuda")
F = torch.empty(B, dtype=torch.float64, device="cuda")
s = torch.empty_like(F)
g = torch.empty_like(pts)
zc = torch.empty(B, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()


def run():
    rc = lib.trstmi_eval_batch_dev(ctx.h, field, d, N, B, ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                                   1, ctypes.c_void_p(F.data_ptr()), ctypes.c_void_p(s.data_ptr()),
                                   ctypes.c_void_p(g.data_ptr()), None, ctypes.c_void_p(zc.data_ptr()),
                                   ctypes.c_void_p(st.cuda_stream))
    assert rc == 0, lib.trstmi_last_error(ctx.h)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
n = N * (N - 1) // 2
fl = (16 if field == abi.COMPLEX else 4) * d * N * N
print(f"eval {field},{d},{N} delta={delta} B={B}: {ms:.3f} ms  {B / ms * 1e3:.3g} evals/s  "
      f"{B * fl / ms / 1e9:.2f} TFLOP/s(alg)  {ms * 1e-3 * 148 * 1.965e9 / B:.0f} SM-cycles/eval")
torch.cuda.synchronize()
print("F[:3]", F[:3].tolist(), "zc", zc[:3].tolist(), "err", torch.cuda.is_available())
from tests import oracle_ffi as orc
Fo, so, go, _, _ = orc.eval_objective(field, d, N, api.lanes(field, d, N), f[0], delta)
print("oracle F", Fo, "match", Fo == F[0].item(), bool((g[0].cpu().numpy() == go).all()))
