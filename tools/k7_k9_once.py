"""One K7 (cfg1 shape) and one K9 (cfg2 shape) launch of 20000 steps, for ncu."""
import numpy as np
from paper_1510_08982_b200 import heat as H
n = 1024
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[-1] = 0
p = H.SolverParams.from_r(0.25); bc = H.BoundaryCondition.dirichlet(0, 0)
H.sync_final(u0, p, bc, 20000)
H.async_final(u0, p, bc, H.PartitionSpec(n, n // 8), H.DelayModel.uniform(2, 1), 20000)
