"""async_run of shapes K9 does not lay out: K6 as one member (default) against
K3 (HEAT_NO_MEMBER_ASYNC=1), ns/step over 20000 steps."""
import sys
import time

from paper_1510_08982_b200 import heat as H

for n, pe, q in ((100, 1, 5), (100, 10, 3), (1000, 10, 4), (1000, 100, 8), (1000, 125, 2),
                 (1024, 4, 2), (600, 600 // 8, 6)):
    u0 = H.cosine_init(n)
    p = H.SolverParams.from_r(0.3)
    bc = H.BoundaryCondition.dirichlet(u0.values()[0], u0.values()[-1])
    m = H.DelayModel.uniform(q, 3)
    k = 20000
    H.async_run(u0, p, bc, H.PartitionSpec(n, pe), m, 100, 100)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        H.async_run(u0, p, bc, H.PartitionSpec(n, pe), m, k, k).final()
        best = min(best, time.perf_counter() - t0)
    print(f"N={n} per_pe={pe} q={q}: {best / k * 1e9:.0f} ns/step")
