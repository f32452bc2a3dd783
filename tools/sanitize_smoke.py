"""Small instances of every kernel family through the public API: a one-shot
smoke of all paths, and the driver for compute-sanitizer where a pool allows
it (this round's pool does not: it refuses runs under compute-sanitizer):

    python tools/sanitize_smoke.py [big]

K1 (one-shot sync, f64 and f32), K9 (small async_run), K3 (async_run, barrier /
flags / global rings), K5 (wide PEs), K6 (ensemble), K7 (small sync), the simulator, slab
plans.  `big` adds the streamed sync_run (N = 2^24, slow under memcheck)."""
import sys

import numpy as np

from paper_1510_08982_b200 import heat as H


def field(n, seed=1):
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1, 1, n)
    return u


def main():
    p = H.SolverParams.from_r(0.35)
    u = field(3000)
    bc = H.BoundaryCondition.dirichlet(float(u[0]), float(u[-1]))
    H.sync_final(u, p, bc, 100)                                   # K1 (N > 16384? no: K7)
    u = field(40000)
    bcd = H.BoundaryCondition.dirichlet(float(u[0]), float(u[-1]))
    H.sync_final(u, p, bcd, 100)                                  # K1 one-shot
    H.sync_run_f32(H.TemperatureField(u), p, bcd, 70, 70)          # K1 f32
    H.sync_final(u, p, H.BoundaryCondition.periodic(), 70)        # K1 periodic
    u = field(1024)
    bc = H.BoundaryCondition.dirichlet(float(u[0]), float(u[-1]))
    H.sync_run(H.TemperatureField(u), p, bc, 150, 50)             # K7 with trajectory
    H.async_run(H.TemperatureField(u), p, bc, H.PartitionSpec(1024, 128),
                H.DelayModel.uniform(2, 1), 150, 50)               # K9 (PEs of 8k points)
    u1 = field(1000)
    bc1 = H.BoundaryCondition.dirichlet(float(u1[0]), float(u1[-1]))
    H.async_run(H.TemperatureField(u1), p, bc1, H.PartitionSpec(1000, 125),
                H.DelayModel.uniform(2, 1), 150, 50)               # K3 barrier, segments
    H.async_final(u, p, bc, H.PartitionSpec(1024, 1), H.DelayModel.uniform(3, 2), 60)  # K3 global
    H.exec_run(H.TemperatureField(u), p, bc, H.PartitionSpec(1024, 128),
               H.ExecConfig(8, 200, H.ExecMode.BarrierFree, True, 4))  # K3 flags
    u = field(3 * 4096)
    bc = H.BoundaryCondition.dirichlet(float(u[0]), float(u[-1]))
    H.async_final(u, p, bc, H.PartitionSpec(3 * 4096, 4096), H.DelayModel.uniform(3, 4), 150)  # K5
    sim = H.AsyncSimulator(H.TemperatureField(u), p, bc, H.PartitionSpec(3 * 4096, 4096),
                           H.DelayModel.geometric(4, 0.6, 5))
    sim.step(10)
    sim.step(70)
    sim.close()
    cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1),
                           H.BoundaryCondition.periodic(), H.PartitionSpec(100, 1),
                           H.DelayModel.uniform(5, 0), 300, 100)
    H.ensemble_run(cfg, 4, 7)                                      # K6
    plan = H.Plan(20000, 0, 0, 2)                                  # slab plan
    plan.upload(np.zeros(20000))
    plan.sync_advance(0.3, H.BoundaryCondition.dirichlet(0.0, 0.0), 40)
    plan.close()
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        u = field(1 << 24)
        u[0] = u[-1] = 0.0
        H.sync_final(u, p, H.BoundaryCondition.dirichlet(0.0, 0.0), 100)  # streamed
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
