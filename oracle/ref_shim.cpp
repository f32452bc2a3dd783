// ref_shim.cpp -- extern "C" face over the REFERENCE library built from
// /root/reference/proj/src (core, sync_solver, async_sim, async_exec).
//
// TEST INFRASTRUCTURE ONLY (see oracle/heat_oracle.c header).  This file is
// our own code; it is compiled together with the reference's unmodified
// sources by oracle/Makefile into oracle/_ref/libheat_ref.so.  It lets the
// Python tests and bench.py's reference arm drive the reference through its
// own public API (heat::sync_run, heat::async_run, heat::exec_run, ...).
//
// Status codes mirror the exception taxonomy of SURVEY.md §8b:
//   0 ok, 1 std::domain_error, 2 std::invalid_argument, 3 std::logic_error,
//   4 heat::DivergenceError, 9 anything else.
#include <cstdint>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "heat/analysis.hpp"
#include "heat/async_exec.hpp"
#include "heat/async_sim.hpp"
#include "heat/core.hpp"
#include "heat/rng.hpp"
#include "heat/sync_solver.hpp"

namespace {

int classify() {
    try {
        throw;
    } catch (const heat::DivergenceError&) {
        return 4;
    } catch (const std::domain_error&) {
        return 1;
    } catch (const std::invalid_argument&) {
        return 2;
    } catch (const std::logic_error&) {
        return 3;
    } catch (...) {
        return 9;
    }
}

heat::BoundaryCondition make_bc(int bc, double c1, double c2) {
    return bc == 0 ? heat::BoundaryCondition::dirichlet(c1, c2)
                   : heat::BoundaryCondition::periodic();
}

heat::DelayModel make_model(int law, std::size_t q, std::size_t d, double p,
                            std::uint64_t seed) {
    if (law == 0) return heat::DelayModel::uniform(q, seed);
    if (law == 1) return heat::DelayModel::fixed(q, d, seed);
    return heat::DelayModel::geometric(q, p, seed);
}

void copy_traj(const heat::Trajectory& t, double* final_out, double* snaps,
               std::size_t* steps, std::size_t cap, std::size_t* n_snap) {
    const std::size_t n = t.final().size();
    if (final_out) std::memcpy(final_out, t.final().values().data(), n * sizeof(double));
    for (std::size_t j = 0; j < t.snapshots.size() && j < cap; ++j) {
        if (snaps) std::memcpy(snaps + j * n, t.snapshots[j].values().data(), n * sizeof(double));
        if (steps) steps[j] = t.steps[j];
    }
    if (n_snap) *n_snap = t.snapshots.size();
}

// Inverse of SplitMix64's finaliser: the class keeps its state private, so
// the state after a call is recovered from one more next() = mix(s + gamma).
std::uint64_t unxorshift(std::uint64_t y, int s) {
    std::uint64_t x = y;
    for (int i = 0; i < 64 / s + 1; ++i) x = y ^ (x >> s);
    return x;
}
std::uint64_t inverse_odd(std::uint64_t m) {
    std::uint64_t x = m;
    for (int i = 0; i < 6; ++i) x *= 2 - m * x;
    return x;
}
std::uint64_t state_of(heat::SplitMix64& rng) {
    std::uint64_t z = unxorshift(rng.next(), 31);
    z = unxorshift(z * inverse_odd(0x94d049bb133111ebULL), 27);
    z = unxorshift(z * inverse_odd(0xbf58476d1ce4e5b9ULL), 30);
    return z - 0x9e3779b97f4a7c15ULL;
}

}  // namespace

extern "C" {

void ref_set_strict(int on) { heat::set_strict_finite_checks(on != 0); }

// heat::SolverParams::r() for checked(alpha, dt, dx) (core.cpp:13-19, core.hpp:27)
int ref_params_checked_r(double alpha, double dt, double dx, double* r) {
    try {
        *r = heat::SolverParams::checked(alpha, dt, dx).r();
        return 0;
    } catch (...) {
        return classify();
    }
}

int ref_sync_step(const double* u, std::size_t n, double r, int bc, double c1, double c2,
                  double* out) {
    try {
        heat::TemperatureField f(std::vector<double>(u, u + n));
        heat::TemperatureField o =
            heat::sync_step(f, heat::SolverParams::from_r(r, true), make_bc(bc, c1, c2));
        std::memcpy(out, o.values().data(), n * sizeof(double));
        return 0;
    } catch (...) {
        return classify();
    }
}

int ref_sync_run(const double* u0, std::size_t n, double r, int bc, double c1, double c2,
                 std::size_t k_end, std::size_t stride, double* final_out, double* snaps,
                 std::size_t* steps, std::size_t cap, std::size_t* n_snap) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        heat::Trajectory t = heat::sync_run(f, heat::SolverParams::from_r(r, true),
                                            make_bc(bc, c1, c2), k_end, stride);
        copy_traj(t, final_out, snaps, steps, cap, n_snap);
        return 0;
    } catch (...) {
        return classify();
    }
}

int ref_sync_run_f32(const double* u0, std::size_t n, double r, int bc, double c1,
                     double c2, std::size_t k_end, double* final_out) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        heat::Trajectory t = heat::sync_run_f32(f, heat::SolverParams::from_r(r, true),
                                                make_bc(bc, c1, c2), k_end, k_end ? k_end : 1);
        copy_traj(t, final_out, nullptr, nullptr, 0, nullptr);
        return 0;
    } catch (...) {
        return classify();
    }
}

int ref_async_run(const double* u0, std::size_t n, double r, int bc, double c1, double c2,
                  std::size_t per_pe, int law, std::size_t q, std::size_t fixed_d, double p,
                  std::uint64_t seed, std::size_t k_end, std::size_t stride, double* final_out,
                  double* snaps, std::size_t* steps, std::size_t cap, std::size_t* n_snap) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        heat::Trajectory t = heat::async_run(
            f, heat::SolverParams::from_r(r, true), make_bc(bc, c1, c2),
            heat::PartitionSpec(n, per_pe), make_model(law, q, fixed_d, p, seed), k_end, stride);
        copy_traj(t, final_out, snaps, steps, cap, n_snap);
        return 0;
    } catch (...) {
        return classify();
    }
}

// heat::async_step (async_sim.cpp:107-116) on a HistoryRing rebuilt at step
// `step` from `count` snapshots (row d = u(step - d)); *rng in/out is the
// SplitMix64 state, read back after the call (also after a throw).
int ref_async_step(const double* snaps, std::size_t count, std::size_t depth, std::size_t step,
                   std::size_t n, double r, int bc, double c1, double c2, std::size_t part_total,
                   std::size_t per_pe, int law, std::size_t q, std::size_t fixed_d, double p,
                   std::uint64_t* rng_state, double* out) {
    heat::SplitMix64 rng(*rng_state);
    int st = 0;
    try {
        auto row = [&](std::size_t d) { return std::vector<double>(snaps + d * n, snaps + (d + 1) * n); };
        heat::HistoryRing ring(depth, row(count - 1));
        for (std::size_t j = 0; j + count - 1 < step; ++j) ring.push(row(count - 1));
        for (std::size_t d = count - 1; d-- > 0;) ring.push(row(d));
        heat::DelayModel m = make_model(law, q, fixed_d, p, 0);
        heat::TemperatureField f = heat::async_step(ring, heat::SolverParams::from_r(r, true),
                                                    make_bc(bc, c1, c2),
                                                    heat::PartitionSpec(part_total, per_pe), m, rng);
        std::memcpy(out, f.values().data(), n * sizeof(double));
    } catch (...) {
        st = classify();
    }
    *rng_state = state_of(rng);
    return st;
}

// sample_delay stream (async_sim.cpp:57-73) for golden vectors.
int ref_delay_stream(int law, std::size_t q, std::size_t fixed_d, double p, std::uint64_t seed,
                     std::size_t k, std::size_t count, std::uint64_t* out) {
    try {
        heat::DelayModel m = make_model(law, q, fixed_d, p, seed);
        heat::SplitMix64 rng(m.seed);
        for (std::size_t i = 0; i < count; ++i) out[i] = heat::sample_delay(rng, m, k);
        return 0;
    } catch (...) {
        return classify();
    }
}

// exec_run (async_exec.cpp:263-279).  lag_out (6 + 64 words) filled when record_lag:
// reads, min, max, overflow, mean bits, histogram size, histogram[...]
int ref_exec_run(const double* u0, std::size_t n, double r, int bc, double c1, double c2,
                 std::size_t per_pe, std::size_t workers, std::size_t k_end, int mode,
                 int record_lag, double* final_out, std::uint64_t* duration_ns,
                 std::uint64_t* lag_out) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        heat::ExecConfig cfg{workers, k_end,
                             mode == 0 ? heat::ExecMode::Barriered : heat::ExecMode::BarrierFree,
                             record_lag != 0};
        heat::ExecResult res = heat::exec_run(f, heat::SolverParams::from_r(r, true),
                                              make_bc(bc, c1, c2), heat::PartitionSpec(n, per_pe),
                                              cfg);
        std::memcpy(final_out, res.field.values().data(), n * sizeof(double));
        if (duration_ns) *duration_ns = std::uint64_t(res.duration.count());
        if (lag_out && res.lag) {
            const heat::LagStats& l = *res.lag;
            lag_out[0] = l.reads;
            lag_out[1] = l.min_lag;
            lag_out[2] = l.max_lag;
            lag_out[3] = l.overflow;
            double m = l.mean();
            std::memcpy(&lag_out[4], &m, sizeof m);
            lag_out[5] = l.histogram.size();
            for (std::size_t i = 0; i < l.histogram.size() && i < 64; ++i) lag_out[6 + i] = l.histogram[i];
        }
        return 0;
    } catch (...) {
        return classify();
    }
}

// exec_run repeated `reps` times on ONE TemperatureField (built once from the
// caller's buffer), each call's own duration (thread spawn..join,
// async_exec.cpp:101-106 / 227-231) into durations_ns[rep]; the last call's
// field goes to final_out (may be null).  The bench's CPU baseline at
// N = 2^30: it saves the shim's per-call 8 GiB field copies, not the
// reference's own (prepare_initial, the result field).
int ref_exec_run_reps(const double* u0, std::size_t n, double r, int bc, double c1, double c2,
                      std::size_t per_pe, std::size_t workers, std::size_t k_end, int mode,
                      std::size_t reps, std::uint64_t* durations_ns, double* final_out) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        heat::ExecConfig cfg{workers, k_end,
                             mode == 0 ? heat::ExecMode::Barriered : heat::ExecMode::BarrierFree,
                             false};
        const auto params = heat::SolverParams::from_r(r, true);
        const auto bcv = make_bc(bc, c1, c2);
        const heat::PartitionSpec part(n, per_pe);
        for (std::size_t i = 0; i < reps; ++i) {
            heat::ExecResult res = heat::exec_run(f, params, bcv, part, cfg);
            durations_ns[i] = std::uint64_t(res.duration.count());
            if (final_out && i + 1 == reps)
                std::memcpy(final_out, res.field.values().data(), n * sizeof(double));
        }
        return 0;
    } catch (...) {
        return classify();
    }
}

// detail::sync_step_into loop (sync_solver.hpp:26-39) in place on caller buffers:
// the single-core CPU baseline.  `a` holds u(0) (already prepared) and receives
// u(k); `b` is scratch of the same size.  Returns elapsed ns of the loop.
std::uint64_t ref_sync_step_into_loop(double* a, double* b, std::size_t n, double r, int bc,
                                      double c1, double c2, std::size_t k) {
    // wrap caller memory in vectors would copy; the inline template takes
    // std::vector, so we keep two persistent vectors per call.
    std::vector<double> cur(a, a + n), next(n);
    (void)b;
    auto bcv = make_bc(bc, c1, c2);
    auto t0 = std::chrono::steady_clock::now();
    for (std::size_t s = 0; s < k; ++s) {
        heat::detail::sync_step_into(cur, next, r, bcv);
        cur.swap(next);
    }
    auto t1 = std::chrono::steady_clock::now();
    std::memcpy(a, cur.data(), n * sizeof(double));
    return std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
}

int ref_prepare_initial(const double* u0, std::size_t n, int bc, double c1, double c2,
                        double* out) {
    try {
        heat::TemperatureField f(std::vector<double>(u0, u0 + n));
        std::vector<double> v = heat::detail::prepare_initial(f, make_bc(bc, c1, c2));
        std::memcpy(out, v.data(), n * sizeof(double));
        return 0;
    } catch (...) {
        return classify();
    }
}

int ref_cosine_init(std::size_t n, double* out) {
    try {
        heat::TemperatureField f = heat::cosine_init(n);
        std::memcpy(out, f.values().data(), n * sizeof(double));
        return 0;
    } catch (...) {
        return classify();
    }
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// ensemble_run (analysis.cpp:51-104): norms[runs][S], terminals[runs][n],
// mean/std[S]; steps_out[S]; returns S through n_steps.
int ref_ensemble_run(const double* u0, std::size_t n, double r, int bc, double c1, double c2,
                     std::size_t per_pe, int law, std::size_t q, std::size_t fixed_d, double p,
                     std::size_t k_end, std::size_t stride, std::size_t runs,
                     std::uint64_t base_seed, std::size_t* steps_out, std::size_t* n_steps,
                     double* norms, double* terminals, double* mean, double* stdv,
                     double* spread2) {
    try {
        heat::EnsembleConfig cfg{heat::TemperatureField(std::vector<double>(u0, u0 + n)),
                                 heat::SolverParams::from_r(r, true),
                                 make_bc(bc, c1, c2),
                                 heat::PartitionSpec(n, per_pe),
                                 make_model(law, q, fixed_d, p, 0),
                                 k_end,
                                 stride};
        heat::EnsembleResult res = heat::ensemble_run(cfg, runs, base_seed);
        const std::size_t S = res.steps.size();
        *n_steps = S;
        for (std::size_t s = 0; s < S; ++s) {
            steps_out[s] = res.steps[s];
            mean[s] = res.mean_series[s];
            stdv[s] = res.std_series[s];
        }
        for (std::size_t j = 0; j < runs; ++j) {
            for (std::size_t s = 0; s < S; ++s) norms[j * S + s] = res.norm_series[j][s];
            if (terminals)
                std::memcpy(terminals + j * n, res.terminal_fields[j].values().data(),
                            n * sizeof(double));
        }
        if (spread2 && runs >= 2) {
            heat::SpreadStats sp = heat::terminal_spread(res);
            spread2[0] = sp.std_terminal_mean_temp;
            spread2[1] = sp.std_terminal_norm;
        }
        return 0;
    } catch (...) {
        return classify();
    }
}

}  // extern "C"
