"""Paper-regime probe (N=1024, 8 PEs): sync vs deterministic async vs free-running.

Small runs are latency-bound and the B200 idles at ~120 MHz between them, so a
~1 s heavy kernel runs first to bring SM clocks up; each config is repeated and
the minimum device time (exec_run's CUDA events) is reported."""
import sys, time
import numpy as np
from paper_1510_08982_b200 import heat as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
warm = H.Plan(1 << 27)
warm.fill_sine()
t0 = time.time()
while time.time() - t0 < 1.0:
    warm.sync_advance(0.4, H.BoundaryCondition.dirichlet(0, 0), 320)
    warm.synchronize()
u0 = np.sin(np.pi * np.arange(n) / (n - 1)); u0[0] = 0; u0[-1] = 0
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0, 0)
part = H.PartitionSpec(n, n // P)
for mode, q in ((H.ExecMode.Barriered, 0), (H.ExecMode.BarrierFree, 2), (H.ExecMode.BarrierFree, 8)):
    best = None
    for _ in range(20):
        res = H.exec_run(H.TemperatureField(u0), p, bc, part, H.ExecConfig(P, K, mode, True, q))
        best = res.duration_ns if best is None else min(best, res.duration_ns)
    extra = f" maxdelay={res.stats.max_delay} waits={res.stats.waits}/{res.stats.reads}" if res.stats else ""
    print(f"exec {H.to_string(mode):13s} q={q}: {best/1e3:9.1f} us  {best/K:7.1f} ns/step {n*K/best:8.3f} GLUPS{extra}")
for q in (1, 2, 3):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); H.async_final(u0, p, bc, part, H.DelayModel.uniform(q, 1), K); ts.append(time.perf_counter() - t0)
    print(f"async_run det q={q}: wall {min(ts)*1e6:9.1f} us (incl. H2D/D2H + launch)")
ts = []
for _ in range(10):
    t0 = time.perf_counter(); H.sync_final(u0, p, bc, K); ts.append(time.perf_counter() - t0)
print(f"sync_run          : wall {min(ts)*1e6:9.1f} us")
