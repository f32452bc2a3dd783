"""Where the wall time of a small public-API call goes (cfg1 shape, N=1024):
full trajectory call vs final-state call vs k_end=1, sync and async (best of 50)."""
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


def best(fn, reps=50):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e6


for k in (1, 1000):
    print(f"k={k:5d} sync_run+traj {best(lambda: H.sync_run(f, p, bc, k, 100)):7.1f} us  "
          f"sync_final {best(lambda: H.sync_final(u0, p, bc, k)):7.1f} us  "
          f"async_run+traj {best(lambda: H.async_run(f, p, bc, part, m, k, 100)):7.1f} us  "
          f"async_final {best(lambda: H.async_final(u0, p, bc, part, m, k)):7.1f} us")
