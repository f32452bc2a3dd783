"""Time the paper's ensembles (acceptance.cpp criteria 2-3: M = 50, N = 100,
one point per PE, q = 5, 2e5 steps) through heat.ensemble_run on the GPU."""
import time

from paper_1510_08982_b200 import heat as H


def main():
    for M in (50, 300):
        for name, bc in (("dirichlet", H.BoundaryCondition.dirichlet(1.0, 0.0)),
                         ("periodic", H.BoundaryCondition.periodic())):
            cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1), bc,
                                   H.PartitionSpec(100, 1), H.DelayModel.uniform(5, 0), 200000,
                                   1000)
            H.ensemble_run(cfg, 2, 1)
            t = time.perf_counter()
            res = H.ensemble_run(cfg, M, 1000)
            dt = time.perf_counter() - t
            print(f"M={M} {name}: {dt:.3f} s  ({dt / 2e5 * 1e6:.3f} us/step, "
                  f"{M * 100 * 2e5 / dt / 1e9:.2f} GLUPS) spread={H.terminal_spread(res)}")


if __name__ == "__main__":
    main()
