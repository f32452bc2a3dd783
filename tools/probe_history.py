"""K8a/K8b throughput: HistoryRing.push_async_step (AsyncSimulator::step on
the device ring) at N = 2^28, PEs of 2^20 points, q = 2; wall time per call
(includes the per-call table upload and the host synchronisation) and the
16 B/point HBM rate it implies.

    python tools/probe_history.py [log2N]"""
import sys
import time

import numpy as np

from paper_1510_08982_b200 import heat as H


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    N = 1 << lg
    u0 = np.zeros(N)
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    ring = H.HistoryRing(2, u0)
    p, part, model = H.SolverParams.from_r(0.4), H.PartitionSpec(N, 1 << 20), H.DelayModel.uniform(2, 1)
    rng = H.SplitMix64(1)
    for _ in range(3):
        ring.push_async_step(p, bc, part, model, rng)
    steps = 20
    t0 = time.perf_counter()
    for _ in range(steps):
        ring.push_async_step(p, bc, part, model, rng)
    dt = (time.perf_counter() - t0) / steps
    print(f"N=2^{lg} step={dt * 1e6:.1f} us  {N / dt / 1e9:.1f} GLUPS  {16 * N / dt / 1e9:.0f} GB/s")
    ring.close()


if __name__ == "__main__":
    main()
