"""K1 pass time vs steps per pass at N=2^30 (one advance of s <= 32 steps is
one pass): fits t(s) = a + b*s to split per-tile fixed cost from stepping."""
import torch
from paper_1510_08982_b200 import heat as H

n = 1 << 30
s = torch.cuda.Stream()
p = H.Plan(n, 0)
p.set_stream(s.cuda_stream)
p.fill_sine()
bc = H.BoundaryCondition.dirichlet(0, 0)
r = H.SolverParams.from_r(0.4).r()
for _ in range(20):
    p.sync_advance(r, bc, 32)
p.synchronize()
res = []
for steps in (1, 4, 8, 16, 24, 32):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(s)
    for _ in range(reps):
        p.sync_advance(r, bc, steps)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res.append((steps, ms))
    print(f"s={steps:2d}: {ms:.3f} ms/pass  {n * steps / (ms * 1e-3) / 1e9:.0f} GLUPS")
import numpy as np
x = np.array([a for a, _ in res if a >= 8], float)
y = np.array([b for a, b in res if a >= 8])
b, a = np.polyfit(x, y, 1)
print(f"fit (s>=8): t = {a:.3f} ms + {b:.4f} ms * s ; fixed share at s=32: {a / (a + 32 * b):.3f}")
