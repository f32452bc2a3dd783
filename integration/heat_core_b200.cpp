// heat_core_b200.cpp -- the reference-side binding: namespace heat's hot-path
// entry points implemented on the B200 library through its C-ABI
// (include/heat_b200.h).  Compiled against the reference's own headers
// (proj/include/heat/*.hpp, unmodified), it replaces these definitions of
// the reference library when linked in front of it:
//
//   heat::sync_step     sync_solver.hpp:60-62   -> heat_sync_step
//   heat::sync_run      sync_solver.hpp:64-67   -> heat_sync_run
//   heat::sync_run_f32  sync_solver.hpp:69-73   -> heat_sync_run_f32
//   heat::async_run     async_sim.hpp:97-101    -> heat_async_run
//   heat::async_step    async_sim.hpp:68-71     -> heat_history_create + heat_async_step
//   heat::exec_run      async_exec.hpp:68-70    -> heat_exec_run
//   heat::ensemble_run  analysis.hpp:36-52      -> heat_ensemble_run
//
//   heat::AsyncSimulator::step  async_sim.cpp:136-140  -> the device async_step
//
// Everything else (CSV, the CLI) keeps running on the reference's CPU code.  oracle/Makefile target `acceptance-b200` links
// the reference's acceptance suite (proj/tests/acceptance.cpp) this way.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "heat/analysis.hpp"
#include "heat/async_exec.hpp"
#include "heat/async_sim.hpp"
#include "heat/core.hpp"
#include "heat/sync_solver.hpp"
#include "heat_b200.h"

namespace heat {

namespace {

void throw_on(int st) {
    if (st == HEAT_OK) return;
    const char* m = heat_last_error();
    switch (st) {
        case HEAT_EDOMAIN: throw std::domain_error(m);
        case HEAT_EINVAL: throw std::invalid_argument(m);
        case HEAT_ELOGIC: throw std::logic_error(m);
        case HEAT_EDIVERGE: throw DivergenceError(m);
        default: throw std::runtime_error(m);
    }
}

int bc_kind(const BoundaryCondition& bc) {
    return bc.is_dirichlet() ? HEAT_BC_DIRICHLET : HEAT_BC_PERIODIC;
}

// The strict-check switch lives in the reference (sync_solver.cpp:9-20);
// mirror it into the library before every call.
void sync_strict() { heat_set_strict_finite_checks(strict_finite_checks() ? 1 : 0); }

using RunFn = int (*)(const double*, size_t, double, int, double, double, size_t, size_t, double*,
                      double*, size_t*, size_t, size_t*);

Trajectory run_traj(RunFn fn, const TemperatureField& u0, const SolverParams& params,
                    const BoundaryCondition& bc, std::size_t k_end, std::size_t stride) {
    sync_strict();
    const std::size_t n = u0.size();
    const std::size_t cap = heat_trajectory_length(n, k_end, stride);
    std::vector<double> snaps(cap * n);
    std::vector<std::size_t> steps(cap);
    std::size_t count = 0;
    throw_on(fn(u0.values().data(), n, params.r(), bc_kind(bc), bc.c1, bc.c2, k_end, stride,
                nullptr, snaps.data(), steps.data(), cap, &count));
    Trajectory t{{}, {}, params, bc};
    t.snapshots.reserve(count);
    for (std::size_t j = 0; j < count; ++j) {
        t.snapshots.emplace_back(
            std::vector<double>(snaps.begin() + j * n, snaps.begin() + (j + 1) * n));
        t.steps.push_back(steps[j]);
    }
    return t;
}

int law_of(const DelayModel& m) {
    return m.distribution == DelayModel::Distribution::Uniform ? HEAT_DELAY_UNIFORM
           : m.distribution == DelayModel::Distribution::Fixed ? HEAT_DELAY_FIXED
                                                               : HEAT_DELAY_GEOMETRIC;
}

// SplitMix64 (rng.hpp:16-41) keeps its state private.  One next() returns
// mix(s + gamma), and mix is a bijection (xorshifts and odd multipliers), so
// the position s is recovered from that draw; the caller then owes the stream
// one draw fewer.
std::uint64_t unxorshift(std::uint64_t y, int s) {
    std::uint64_t x = y;
    for (int i = 0; i < 64 / s + 1; ++i) x = y ^ (x >> s);
    return x;
}
std::uint64_t inverse_odd(std::uint64_t m) {  // m^-1 mod 2^64 (Newton)
    std::uint64_t x = m;
    for (int i = 0; i < 6; ++i) x *= 2 - m * x;
    return x;
}
constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
std::uint64_t take_position(SplitMix64& rng) {
    std::uint64_t z = unxorshift(rng.next(), 31);
    z = unxorshift(z * inverse_odd(0x94d049bb133111ebULL), 27);
    z = unxorshift(z * inverse_odd(0xbf58476d1ce4e5b9ULL), 30);
    return z - kGamma;
}

}  // namespace

TemperatureField sync_step(const TemperatureField& u, const SolverParams& params,
                           const BoundaryCondition& bc) {
    sync_strict();
    std::vector<double> out(u.size());
    throw_on(heat_sync_step(u.values().data(), u.size(), params.r(), bc_kind(bc), bc.c1, bc.c2,
                            out.data()));
    return TemperatureField(std::move(out));
}

Trajectory sync_run(const TemperatureField& u0, const SolverParams& params,
                    const BoundaryCondition& bc, std::size_t k_end, std::size_t stride) {
    return run_traj(heat_sync_run, u0, params, bc, k_end, stride);
}

Trajectory sync_run_f32(const TemperatureField& u0, const SolverParams& params,
                        const BoundaryCondition& bc, std::size_t k_end, std::size_t stride) {
    return run_traj(heat_sync_run_f32, u0, params, bc, k_end, stride);
}

Trajectory async_run(const TemperatureField& u0, const SolverParams& params,
                     const BoundaryCondition& bc, const PartitionSpec& part,
                     const DelayModel& model, std::size_t k_end, std::size_t stride) {
    sync_strict();
    if (part.total() != u0.size())  // AsyncSimulator ctor, async_sim.cpp:131-132
        throw std::invalid_argument("AsyncSimulator: partition inconsistent with grid");
    const std::size_t n = u0.size();
    const std::size_t cap = heat_trajectory_length(n, k_end, stride);
    std::vector<double> snaps(cap * n);
    std::vector<std::size_t> steps(cap);
    std::size_t count = 0;
    const int law = law_of(model);
    throw_on(heat_async_run(u0.values().data(), n, params.r(), bc_kind(bc), bc.c1, bc.c2,
                            part.per_pe(), model.q, law, model.fixed_delay, model.geometric_p,
                            model.seed, k_end, stride, nullptr, snaps.data(), steps.data(), cap,
                            &count));
    Trajectory t{{}, {}, params, bc};
    for (std::size_t j = 0; j < count; ++j) {
        t.snapshots.emplace_back(
            std::vector<double>(snaps.begin() + j * n, snaps.begin() + (j + 1) * n));
        t.steps.push_back(steps[j]);
    }
    return t;
}

namespace {
// The device step over a host ring into `out` (no TemperatureField: the
// simulator's step does not validate, async_sim.cpp:136-140).
void async_step_device(const HistoryRing& hist, const SolverParams& params,
                       const BoundaryCondition& bc, const PartitionSpec& part,
                       const DelayModel& model, SplitMix64& rng, std::vector<double>& out) {
    const std::size_t n = hist.grid_size(), k = hist.current_step();
    const std::size_t held = std::min(hist.depth(), k + 1);
    std::vector<double> rows(held * n);
    for (std::size_t d = 0; d < held; ++d)
        std::memcpy(rows.data() + d * n, hist.snapshot(d).data(), n * sizeof(double));
    heat_history* h = nullptr;
    throw_on(heat_history_create(&h, hist.depth(), n, k, rows.data(), held, -1));
    const bool draws = part.total() / part.per_pe() > 1;
    const std::uint64_t s0 = draws ? take_position(rng) : 0;
    std::uint64_t s = s0;
    out.resize(n);
    const int st = heat_async_step(h, params.r(), bc_kind(bc), bc.c1, bc.c2, part.total(),
                                   part.per_pe(), model.q, law_of(model), model.fixed_delay,
                                   model.geometric_p, &s, out.data(), 0);
    heat_history_destroy(h);
    if (draws) {  // s = s0 + m*gamma for the m draws consumed; one is already taken
        const std::uint64_t m = (s - s0) * inverse_odd(kGamma);
        for (std::uint64_t j = 1; j < m; ++j) rng.next();
    }
    throw_on(st);
}
}  // namespace

// AsyncSimulator::step (async_sim.cpp:136-140) with the step on the device:
// the simulator's own ring and SplitMix64 stream go through the same device
// async_step as heat::async_step, then the push.  (The class's members are
// laid out in the reference header; step() is the only out-of-line member
// that computes, so it is the one substituted.)
void AsyncSimulator::step() {
    sync_strict();
    async_step_device(ring_, params_, bc_, part_, model_, rng_, scratch_);
    ring_.push(scratch_);
    scratch_.resize(ring_.grid_size());
}

// async_step over the caller's (host) ring: the held snapshots go to a device
// ring at the same step, K8a/K8b compute the step, and the caller's stream is
// left where the reference would leave it (D draws, or through the failing
// draw on a logic_error).  A one-PE partition draws nothing and is not touched.
TemperatureField async_step(const HistoryRing& hist, const SolverParams& params,
                            const BoundaryCondition& bc, const PartitionSpec& part,
                            const DelayModel& model, SplitMix64& rng) {
    sync_strict();
    if (part.total() != hist.grid_size())  // async_sim.cpp:113-114
        throw std::invalid_argument("async_step: partition inconsistent with grid");
    std::vector<double> out;
    async_step_device(hist, params, bc, part, model, rng, out);
    return TemperatureField(std::move(out));
}

EnsembleResult ensemble_run(const EnsembleConfig& cfg, std::size_t runs,
                            std::uint64_t base_seed) {
    sync_strict();
    if (cfg.part.total() != cfg.u0.size())  // AsyncSimulator ctor, async_sim.cpp:131-132
        throw std::invalid_argument("AsyncSimulator: partition inconsistent with grid");
    const std::size_t n = cfg.u0.size();
    const std::size_t stride = cfg.stride == 0 ? detail::default_stride(n) : cfg.stride;
    const std::size_t cap = 2 + cfg.k_end / stride;
    std::vector<std::size_t> steps(cap);
    std::size_t S = 0;
    std::vector<double> norms(std::max<std::size_t>(1, runs) * cap), terms(runs * n), mean(cap),
        stdv(cap);
    const DelayModel& m = cfg.model;
    throw_on(heat_ensemble_run(cfg.u0.values().data(), n, cfg.params.r(), bc_kind(cfg.bc),
                               cfg.bc.c1, cfg.bc.c2, cfg.part.per_pe(), m.q, law_of(m),
                               m.fixed_delay, m.geometric_p, cfg.k_end, stride, runs, base_seed, steps.data(), cap, &S,
                               norms.data(), terms.data(), mean.data(), stdv.data()));
    EnsembleResult res;
    res.steps.assign(steps.begin(), steps.begin() + S);
    res.norm_series.resize(runs);
    for (std::size_t j = 0; j < runs; ++j) {
        res.norm_series[j].assign(norms.begin() + j * S, norms.begin() + (j + 1) * S);
        res.terminal_fields.emplace_back(
            std::vector<double>(terms.begin() + j * n, terms.begin() + (j + 1) * n));
        res.seeds.push_back(base_seed + j);
    }
    res.mean_series.assign(mean.begin(), mean.begin() + S);
    res.std_series.assign(stdv.begin(), stdv.begin() + S);
    return res;
}

ExecResult exec_run(const TemperatureField& u0, const SolverParams& params,
                    const BoundaryCondition& bc, const PartitionSpec& part,
                    const ExecConfig& cfg) {
    sync_strict();
    std::vector<double> out(u0.size());
    std::uint64_t ns = 0;
    heat_lag_stats lag{};
    throw_on(heat_exec_run(u0.values().data(), u0.size(), params.r(), bc_kind(bc), bc.c1, bc.c2,
                           part.per_pe(), cfg.workers, cfg.k_end,
                           cfg.mode == ExecMode::Barriered ? HEAT_EXEC_BARRIERED
                                                           : HEAT_EXEC_BARRIER_FREE,
                           cfg.record_lag ? 1 : 0, 0, out.data(), &ns, &lag, nullptr));
    ExecResult res{TemperatureField(std::move(out)), std::vector<std::size_t>(cfg.workers, cfg.k_end),
                   std::chrono::nanoseconds(ns), false, std::nullopt};
    // run_barriered never reports lag; run_barrier_free reports the merged
    // (possibly empty, P = 1) statistics when asked (async_exec.cpp:250-256).
    if (cfg.record_lag && cfg.mode == ExecMode::BarrierFree) {
        LagStats l;
        if (lag.reads) {
            l.reads = lag.reads;
            l.min_lag = lag.min_lag;
            l.max_lag = lag.max_lag;
            l.overflow = lag.overflow;
            l.histogram.assign(lag.histogram, lag.histogram + 64);
        }
        res.lag = l;
    }
    return res;
}

}  // namespace heat
