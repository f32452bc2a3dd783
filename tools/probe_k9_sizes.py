import time, numpy as np
from paper_1510_08982_b200 import heat as H
for n, pe in ((2048, 256), (4096, 512), (8192, 1024)):
    u0 = np.sin(np.pi*np.arange(n)/(n-1)); u0[-1] = 0
    f = H.TemperatureField(u0); p = H.SolverParams.from_r(0.25); bc = H.BoundaryCondition.dirichlet(0, 0)
    part = H.PartitionSpec(n, pe); m = H.DelayModel.uniform(2, 1)
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter(); H.async_run(f, p, bc, part, m, 5000, 5000).final(); best = min(best, time.perf_counter() - t0)
    print(f"async_run N={n} P={n//pe} q=2 5000 steps: {best*1e6:.0f} us, {best/5000*1e9:.1f} ns/step")
