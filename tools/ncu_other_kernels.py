"""One launch of each kernel besides K1/K5, at the sizes the public API uses them,
for `ncu --set full` captures (profiles/ncu_summary.json):

  K7 sync_small_kernel   cfg1: sync_run, N=1024, r=0.25, 1000 steps (BASELINE configs[0])
  K3 async_pe_kernel     cfg2: async_run, N=1024, 8 PEs, uniform q=2, seed 1, 1000 steps (configs[1])
  K6 ensemble_kernel     the paper's ensemble: 50 members, N=1024, 8 PEs, q=2, 2*10^4 steps
  K8a step_body_kernel / K8b step_edges_kernel
                         one async_step over a device HistoryRing, N=2^26, 512 PEs, q=4
"""
import numpy as np

from paper_1510_08982_b200 import heat as H

n = 1024
u0 = np.sin(np.pi * np.arange(n) / (n - 1))
u0[-1] = 0.0
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
part = H.PartitionSpec(n, n // 8)
H.sync_final(u0, p, bc, 1000)                                        # K7
H.async_final(u0, p, bc, part, H.DelayModel.uniform(2, 1), 1000)     # K3
cfg = H.EnsembleConfig(H.TemperatureField(u0), p, bc, part, H.DelayModel.uniform(2, 1),
                       k_end=20000, stride=1000)
H.ensemble_run(cfg, 50, 1, keep_terminals=False)                     # K6
N = 1 << 26
big = np.sin(np.pi * np.arange(N) / (N - 1))
big[-1] = 0.0
ring = H.HistoryRing(4, big, 0)
ring.push_async_step(H.SolverParams.from_r(0.4), bc, H.PartitionSpec(N, N // 512),
                     H.DelayModel.uniform(4, 7), H.SplitMix64(7))     # K8a + K8b
print("ok")
