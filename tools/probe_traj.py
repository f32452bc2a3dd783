"""Wall time of a recorded large sync_run (N = 2^26, 1000 steps, stride 100:
11 snapshots of 512 MiB) with snapshot downloads overlapped (default) or in
line (HEAT_NO_OVERLAP_SNAPS=1); pageable numpy destination, as the mirror uses."""
import os
import time

import numpy as np

from paper_1510_08982_b200 import heat as H

n = 1 << 26
u = np.sin(np.pi * np.arange(n) / (n - 1))
u[0] = u[-1] = 0.0
p = H.SolverParams.from_r(0.4)
bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
H.sync_run(H.TemperatureField(np.zeros(4096)), p, bc, 10, 5)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    t = H.sync_run(H.TemperatureField(u), p, bc, 1000, 100)
    ts.append(time.perf_counter() - t0)
mode = "in line" if os.environ.get("HEAT_NO_OVERLAP_SNAPS") else "overlapped"
print(f"{mode}: best {min(ts):.3f} s for 1000 steps + {len(t.snapshots)} snapshots")
