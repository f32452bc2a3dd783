"""One free-running exec_run at N=1024, 8 PEs, 1000 steps (ncu target)."""
import numpy as np
from paper_1510_08982_b200 import heat as H
n, P, K = 1024, 8, 1000
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
for _ in range(3):
    res = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(0.25), H.BoundaryCondition.dirichlet(0, 0),
                     H.PartitionSpec(n, n // P), H.ExecConfig(P, K, H.ExecMode.BarrierFree, True, 8))
print("ok", res.duration_ns)
