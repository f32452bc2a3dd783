// binding_check.cpp -- TEST INFRASTRUCTURE (see heat_oracle.c's header).
//
// Drives heat::async_step (async_sim.hpp:68-71) and heat::AsyncSimulator
// (async_sim.hpp:73-90) through the reference's own types on seeded random
// rings / simulators and prints one line per case: the exception
// class (or "ok"), the FNV-1a-64 of the result's bytes, and the caller's
// stream position after the call (its next draw).  oracle/Makefile links it
// twice: against the reference library (binding_check_ref) and with
// integration/heat_core_b200.cpp in front of it (binding_check_b200, the GPU
// ring + kernels K8a/K8b).  tests/test_gpu_history.py requires the two
// outputs to be identical.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "heat/async_sim.hpp"
#include "heat/core.hpp"
#include "heat/rng.hpp"
#include "heat/sync_solver.hpp"

namespace {

std::uint64_t fnv(const std::vector<double>& v) {
    std::uint64_t h = 1469598103934665603ULL;
    for (double x : v) {
        unsigned char b[8];
        std::memcpy(b, &x, 8);
        for (unsigned char c : b) h = (h ^ c) * 1099511628211ULL;
    }
    return h;
}

std::vector<double> field(heat::SplitMix64& g, std::size_t n) {
    std::vector<double> v(n);
    for (auto& x : v) x = g.next_double() * 4.0 - 2.0;
    return v;
}

}  // namespace

int main() {
    heat::SplitMix64 gen(20261018);
    for (int c = 0; c < 200; ++c) {
        const std::size_t n = 3 + gen.next_bounded(90);
        std::vector<std::size_t> divs;
        for (std::size_t d = 1; d <= n; ++d)
            if (n % d == 0) divs.push_back(d);
        const std::size_t per_pe = divs[gen.next_bounded(divs.size() - 1)];
        const std::size_t q = 1 + gen.next_bounded(6);
        const std::size_t depth = gen.next_bounded(3) ? q : 1 + gen.next_bounded(q - 1);
        const std::size_t steps = gen.next_bounded(10);
        const int law = int(gen.next_bounded(2));
        const double r = 0.5 * (gen.next_double() * 0.999 + 0.001);
        const bool periodic = gen.next() & 1;
        heat::HistoryRing ring(depth, field(gen, n));
        for (std::size_t k = 0; k < steps; ++k) ring.push(field(gen, n));
        heat::DelayModel m = law == 0   ? heat::DelayModel::uniform(q, 0)
                             : law == 1 ? heat::DelayModel::fixed(q, gen.next_bounded(q - 1), 0)
                                        : heat::DelayModel::geometric(q, 0.05 + 0.9 * gen.next_double(), 0);
        const auto bc = periodic ? heat::BoundaryCondition::periodic()
                                 : heat::BoundaryCondition::dirichlet(gen.next_double(), gen.next_double());
        heat::SplitMix64 rng(gen.next());
        const char* what = "ok";
        std::uint64_t h = 0;
        try {
            heat::TemperatureField f = heat::async_step(ring, heat::SolverParams::from_r(r), bc,
                                                        heat::PartitionSpec(n, per_pe), m, rng);
            h = fnv(f.values());
        } catch (const std::logic_error&) {  // domain_error / invalid_argument derive from it
            what = "logic_error";
        } catch (const std::exception& e) {
            what = "other";
            std::fprintf(stderr, "case %d: %s\n", c, e.what());
        }
        std::printf("%d %s %016llx %016llx\n", c, what, (unsigned long long)h,
                    (unsigned long long)rng.next());
    }
    // heat::AsyncSimulator (async_sim.hpp:73-90): seeded simulators stepped a
    // random number of times; the field after every few steps and the step index
    for (int c = 0; c < 60; ++c) {
        const std::size_t n = 3 + gen.next_bounded(70);
        std::vector<std::size_t> divs;
        for (std::size_t d = 1; d <= n; ++d)
            if (n % d == 0) divs.push_back(d);
        const std::size_t per_pe = divs[gen.next_bounded(divs.size() - 1)];  // bound inclusive
        const std::size_t q = 1 + gen.next_bounded(5);
        const int law = int(gen.next_bounded(3));
        const double r = 0.5 * (gen.next_double() * 0.999 + 0.001);
        const bool periodic = gen.next() & 1;
        std::vector<double> u0 = field(gen, n);
        const auto bc = periodic ? heat::BoundaryCondition::periodic()
                                 : heat::BoundaryCondition::dirichlet(u0[0], u0[n - 1]);
        const std::uint64_t seed = gen.next();
        const std::size_t fixed_d = gen.next_bounded(q - 1);
        const double gp = 0.05 + 0.9 * gen.next_double();
        heat::DelayModel m = law == 0   ? heat::DelayModel::uniform(q, seed)
                             : law == 1 ? heat::DelayModel::fixed(q, fixed_d, seed)
                                        : heat::DelayModel::geometric(q, gp, seed);
        const std::size_t steps = 1 + gen.next_bounded(40);
        const char* what = "ok";
        std::uint64_t h = 0;
        std::size_t idx = 0;
        try {
            heat::AsyncSimulator sim(heat::TemperatureField(u0), heat::SolverParams::from_r(r), bc,
                                     heat::PartitionSpec(n, per_pe), m);
            for (std::size_t k = 0; k < steps; ++k) {
                sim.step();
                if (k % 7 == 0) h ^= fnv(sim.current()) + k;
            }
            h ^= fnv(sim.current());
            idx = sim.step_index();
        } catch (const std::logic_error& e) {
            what = "logic_error";
            std::fprintf(stderr, "sim case %d: %s\n", c, e.what());
        } catch (const std::exception& e) {
            what = "other";
            std::fprintf(stderr, "sim case %d: %s\n", c, e.what());
        }
        std::printf("sim %d %s %016llx %zu\n", c, what, (unsigned long long)h, idx);
    }
    return 0;
}
