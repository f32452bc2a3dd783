"""One barriered exec_run at the paper's N=1024 / 8 PEs for a profiler capture."""
import sys
import numpy as np
from paper_1510_08982_b200 import heat as H

mode = H.ExecMode.Barriered if (len(sys.argv) < 2 or sys.argv[1] == "b") else H.ExecMode.BarrierFree
n, P, K = 1024, 8, 20000
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
res = H.exec_run(H.TemperatureField(u0), H.SolverParams.from_r(0.25), H.BoundaryCondition.dirichlet(0, 0),
                 H.PartitionSpec(n, n // P), H.ExecConfig(P, K, mode, True, 2))
print(res.duration_ns / K, "ns/step")
