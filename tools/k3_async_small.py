"""One deterministic async_run at the paper's cfg2 shape (N=1024, 8 PEs, q=2),
20000 steps, for a profiler capture of the lockstep K3 kernel."""
import numpy as np
from paper_1510_08982_b200 import heat as H

n, P, K = 1024, 8, 20000
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
H.async_final(u0, H.SolverParams.from_r(0.25), H.BoundaryCondition.dirichlet(0, 0),
              H.PartitionSpec(n, n // P), H.DelayModel.uniform(2, 1), K)
print("ok")
