"""One member of the paper's Fig. 3/6 experiment as a plain async_run (N = 100,
one point per PE, q = 5, uniform delays, 2e5 steps, Dirichlet(1, 0), cosine
IC), and the same with rows every 1000 steps, against K6 running it as a
one-member ensemble."""
import time

from paper_1510_08982_b200 import heat as H

u0 = H.cosine_init(100)
p = H.SolverParams.checked(0.5, 0.01, 0.1)
bc = H.BoundaryCondition.dirichlet(1.0, 0.0)
part = H.PartitionSpec(100, 1)
m = H.DelayModel.uniform(5, 7)
for k, stride in ((20000, 20000), (200000, 1000)):
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        H.async_run(u0, p, bc, part, m, k, stride).final()
        best = min(best, time.perf_counter() - t0)
    print(f"async_run N=100 P=100 q=5 k={k} stride={stride}: {best * 1e3:.2f} ms, {best / k * 1e9:.0f} ns/step")
cfg = H.EnsembleConfig(u0, p, bc, part, m, 200000, 1000)
H.ensemble_run(cfg, 1, 7)
t0 = time.perf_counter()
H.ensemble_run(cfg, 1, 7)
dt = time.perf_counter() - t0
print(f"ensemble_run M=1 k=200000: {dt * 1e3:.2f} ms, {dt / 2e5 * 1e9:.0f} ns/step")
