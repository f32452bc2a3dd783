"""Paper-regime probe (N=1024, 8 PEs): sync vs deterministic async vs free-running,
device time from exec_run's CUDA events and wall time around async_run."""
import sys, time
import numpy as np
from paper_1510_08982_b200 import heat as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0, 0)
part = H.PartitionSpec(n, n // P)
for mode, q in ((H.ExecMode.Barriered, 0), (H.ExecMode.BarrierFree, 2), (H.ExecMode.BarrierFree, 8)):
    best = None
    for _ in range(5):
        res = H.exec_run(H.TemperatureField(u0), p, bc, part, H.ExecConfig(P, K, mode, True, q))
        best = res.duration_ns if best is None else min(best, res.duration_ns)
    extra = ""
    if res.stats:
        extra = f" maxdelay={res.stats.max_delay} waits={res.stats.waits}/{res.stats.reads}"
    print(f"exec {H.to_string(mode):13s} q={q}: {best/1e3:9.1f} us  {n*K/best:8.3f} GLUPS{extra}")
for q in (1, 2, 3):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); H.async_final(u0, p, bc, part, H.DelayModel.uniform(q, 1), K); ts.append(time.perf_counter() - t0)
    print(f"async_run det q={q}: wall {min(ts)*1e6:9.1f} us (incl. H2D/D2H + launch)")
ts = []
for _ in range(5):
    t0 = time.perf_counter(); H.sync_final(u0, p, bc, K); ts.append(time.perf_counter() - t0)
print(f"sync_run          : wall {min(ts)*1e6:9.1f} us")
