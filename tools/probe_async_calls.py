"""K5 per-call overhead: 10 x 1000-step async_advance calls with / without the
stats read-back, against one 10000-step call (device-timed)."""
import torch
from paper_1510_08982_b200 import heat as H, _lib
import ctypes as C
n = 1 << 30
s = torch.cuda.Stream()
p = H.Plan(n, 0); p.set_stream(s.cuda_stream); p.fill_sine()
bc = H.BoundaryCondition.dirichlet(0, 0); r = H.SolverParams.from_r(0.4).r()
per = n // 512
p.async_advance(r, bc, per, 8, 1000); p.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("stats", "nostats", "one", "stats", "nostats", "one"):
    e0.record(s)
    if mode == "one":
        p.async_advance(r, bc, per, 8, 10000)
    else:
        for _ in range(10):
            if mode == "stats":
                p.async_advance(r, bc, per, 8, 1000)
            else:
                _lib.check(_lib.lib().heat_plan_async_advance(p._h, r, bc.kind, bc.c1, bc.c2, per, 8, 1000, None), "x")
    e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(mode, round(ms, 2), "ms", round(n * 10000 / (ms * 1e-3) / 1e9, 1), "GLUPS")
