"""Wall time of BASELINE configs[1] (N=1024, 8 PEs, uniform q=2, seed 1, r=0.25,
1000 steps, trajectory every 100 steps) through the public API, best of 30,
and of the same run at 20000 steps (per-step kernel cost)."""
import time

import numpy as np

from paper_1510_08982_b200 import heat as H

n = 1024
u0 = np.sin(np.pi * np.arange(n) / (n - 1))
u0[-1] = 0.0
f = H.TemperatureField(u0)
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
part = H.PartitionSpec(n, n // 8)
m = H.DelayModel.uniform(2, 1)
for k, stride in ((1000, 100), (20000, 20000)):
    ts = []
    for _ in range(30 if k == 1000 else 5):
        t0 = time.perf_counter()
        H.async_run(f, p, bc, part, m, k, stride).final()
        ts.append(time.perf_counter() - t0)
    print(f"async_run cfg2 k={k}: best {min(ts) * 1e6:.1f} us, {min(ts) / k * 1e9:.1f} ns/step")
