"""exec_run(BarrierFree) delay statistics at the measure() shapes."""
from paper_1510_08982_b200 import heat as H
for N, P in ((1000, 4), (1000, 10), (1000, 20), (10000, 10)):
    res = H.exec_run(H.cosine_init(N), H.SolverParams.from_r(0.5), H.BoundaryCondition.dirichlet(1.0, 0.0),
                     H.PartitionSpec(N, N // P), H.ExecConfig(P, 2000, H.ExecMode.BarrierFree))
    st = res.stats
    print(N, P, "reads", st.reads, "waits", st.waits, "max_delay", st.max_delay,
          "hist", st.delay_histogram[:8], f"{res.duration_ns / 2000:.1f} ns/step")
