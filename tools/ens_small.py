from paper_1510_08982_b200 import heat as H
cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.checked(0.5, 0.01, 0.1), H.BoundaryCondition.periodic(),
                       H.PartitionSpec(100, 1), H.DelayModel.uniform(5, 0), 20000, 1000)
H.ensemble_run(cfg, 50, 1000)
