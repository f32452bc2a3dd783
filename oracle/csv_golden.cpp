// TEST INFRASTRUCTURE ONLY: writes the reference's own CSV output
// (proj/src/csv.cpp: emit_trajectory_csv, emit_ensemble_csv, emit_bench_csv)
// for fixed small inputs, as golden fixtures for paper_1510_08982_b200/csvio.py
// (tests/golden/gen_csv_golden.py runs it; tests/test_csvio.py compares).
//   usage: csv_golden <out dir>
#include <string>
#include <vector>

#include "heat/analysis.hpp"
#include "heat/async_exec.hpp"
#include "heat/async_sim.hpp"
#include "heat/csv.hpp"
#include "heat/sync_solver.hpp"

using namespace heat;

int main(int argc, char** argv) {
    if (argc != 2) return 2;
    const std::string dir = argv[1];
    // sync trajectory: cosine IC, r = 0.3, Dirichlet(1, 0), 25 steps every 5
    const Trajectory ts = sync_run(cosine_init(13), SolverParams::from_r(0.3),
                                   BoundaryCondition::dirichlet(1.0, 0.0), 25, 5);
    emit_trajectory_csv(ts, dir + "/traj_sync.csv");
    // async trajectory: periodic, 3 PEs of 8, uniform q = 3 seed 77, 40 steps every 7
    const Trajectory ta = async_run(cosine_init(24), SolverParams::from_r(0.45),
                                    BoundaryCondition::periodic(), PartitionSpec(24, 8),
                                    DelayModel::uniform(3, 77), 40, 7);
    emit_trajectory_csv(ta, dir + "/traj_async.csv");
    // ensemble: 3 members of 16 points in 4 PEs, uniform q = 2, 30 steps every 10
    EnsembleConfig cfg{cosine_init(16), SolverParams::from_r(0.4),
                       BoundaryCondition::dirichlet(1.0, 0.0), PartitionSpec(16, 4),
                       DelayModel::uniform(2, 0), 30, 10};
    const EnsembleResult er = ensemble_run(cfg, 3, 5);
    emit_ensemble_csv(er, dir + "/ens_runs.csv", dir + "/ens_stats.csv");
    // bench rows
    std::vector<BenchRow> rows(2);
    rows[0].n_points = 1000;
    rows[0].mode = ExecMode::Barriered;
    rows[0].reps = 5;
    rows[0].median_ns = 123456;
    rows[0].min_ns = 120000;
    rows[1].n_points = 1000;
    rows[1].mode = ExecMode::BarrierFree;
    rows[1].reps = 5;
    rows[1].median_ns = 9876;
    rows[1].min_ns = 9000;
    emit_bench_csv(rows, dir + "/bench.csv");
    return 0;
}
