"""Small-N synchronous path (exec_run(Barriered) -> heat_sync_run -> K7, or K1
with HEAT_NO_SMALL_SYNC=1): device ns/step at N = 100, 1024, 4096."""
import os
import sys
import numpy as np
from paper_1510_08982_b200 import heat as H

K = 20000
for n in (100, 1024, 4096):
    u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
    best = None
    for _ in range(5):
        res = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(0.25),
                         H.BoundaryCondition.dirichlet(0, 0), H.PartitionSpec(n, n // 4),
                         H.ExecConfig(4, K, H.ExecMode.Barriered, False, 0))
        best = res.duration_ns if best is None else min(best, res.duration_ns)
    path = "K1" if os.environ.get("HEAT_NO_SMALL_SYNC") else "K7"
    print(f"{path} n={n}: {best / K:.1f} ns/step")
