"""One K6 launch of the paper's ensemble (M = 50, N = 100, one point per PE,
q = 5, 2e5 steps, Dirichlet(1, 0)), for ncu."""
import sys

from paper_1510_08982_b200 import heat as H

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1),
                       H.BoundaryCondition.dirichlet(1.0, 0.0), H.PartitionSpec(100, 1),
                       H.DelayModel.uniform(5, 0), steps, 1000)
H.ensemble_run(cfg, 50, 1000)
