"""Per-step time of the ensemble kernel (K6) with ONE member at cfg2's shape
(N=1024, 8 PEs, q=2) vs the K3 path of async_run: is K6 a better small-N
async_run engine?"""
import time
import numpy as np
from paper_1510_08982_b200 import heat as H

n, P, q = 1024, 8, 2
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0, 0)
for K in (1000, 20000):
    cfg = H.EnsembleConfig(H.TemperatureField(u0), p, bc, H.PartitionSpec(n, n // P),
                           H.DelayModel.uniform(q, 1), K, K)
    H.ensemble_run(cfg, 1, 1)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); H.ensemble_run(cfg, 1, 1); ts.append(time.perf_counter() - t0)
    t_k6 = min(ts)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        H.async_final(u0, p, bc, H.PartitionSpec(n, n // P), H.DelayModel.uniform(q, 1), K)
        ts.append(time.perf_counter() - t0)
    t_k3 = min(ts)
    print(f"K={K}: K6 one member {t_k6 * 1e6:.0f} us ({t_k6 / K * 1e9:.0f} ns/step), "
          f"async_run (K3) {t_k3 * 1e6:.0f} us ({t_k3 / K * 1e9:.0f} ns/step)")
