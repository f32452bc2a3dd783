"""Small-N synchronous path (heat_sync_run -> K3 barrier mode): device ns/step
for the PE count HEAT_SMALL_SYNC_PES caps (A/B helper)."""
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
    print(f"PES<={os.environ.get('HEAT_SMALL_SYNC_PES', '16')} n={n}: {best / K:.1f} ns/step")
