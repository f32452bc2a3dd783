// ensemble.cu -- K6: GPU ensemble driver (SURVEY.md §8f "next" #1).
//
// Replaces ensemble_run / run_member (analysis.cpp:16-104): M seeded members
// of the deterministic asynchronous scheme (AsyncSimulator, async_sim.cpp:
// 77-140) with seeds base_seed + j, each recording l2_norm (core.cpp:50-56)
// at the recorded steps; the host then forms the mean / population-std
// series in the reference's order (analysis.cpp:88-103).
//
// Mapping: one CTA per member; thread t owns points t, t+T, ...; the member's
// history of the last q steps lives in shared memory as q+1 full-field slots
// (the slot written at step k is never one a read at step k can ask for), and
// the members advance with one block barrier per step.  Every cross-PE read
// uses the delay the reference draws for it: draw number k*D + off(i, side) of
// the member's SplitMix64 stream in counter form (any partition, n = 1 too).
// The paper's experiments (Fig. 3/6: N = 100, one point per PE, q = 5,
// 2e5 steps, 50-300 members) are latency-bound per member and embarrassingly
// parallel across members -- 148 SMs run them side by side.
#include <algorithm>
#include <cmath>
#include <vector>

#include "async_pe.cuh"
#include "runtime.cuh"

namespace hb {
namespace {

struct EnsembleArgs {
    const double* u0;   // prepared initial field [n]
    int n;
    double r, c, c1, c2;
    int dirichlet;
    int q;              // delays in {0..q-1}; q+1 history slots
    int law;            // uniform, fixed or geometric
    int fixed_d;
    const uint64_t* gthr;  // geometric law: the q-1 delay thresholds (geometric_thresholds)
    unsigned long long base_seed;
    ModQ modq;          // x mod q (uniform law, steps k >= q-1)
    long long D;        // cross-PE reads per step
    const int* offL;    // [n] draw rank of point i's left read (-1: same PE or pinned)
    const int* offR;    // [n] ... right read
    long long k_end;
    long long stride;   // recording stride (norms at 0, stride, 2*stride, ..., k_end)
    int n_rec;          // number of recorded steps
    double* norms;      // [runs][n_rec]
    double* terminals;  // [runs][n] (may be null)
    unsigned int* flag; // [0] non-finite
    double* rows;       // one-member async_run: [n_rec][n] trajectory rows (may be null)
};

// l2_norm (core.cpp:50-56): sequential sum of squares, then sqrt -- one
// thread, the reference's summation order.
__device__ double seq_l2(const double* v, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(v[i], v[i]));
    return sqrt(s);
}

constexpr unsigned long long kGamma = 0x9e3779b97f4a7c15ULL;  // rng.hpp:21

// PT points per thread (t, t+T, ...); LAW 0 uniform, 1 fixed, 2 geometric.  The member is
// latency-bound (one warp per scheduler), so the step is written for a short
// dependent chain: per-point constants hoisted, SplitMix64 counters carried
// incrementally (draw k*D + off of the member's stream is mix(z) with
// z = seed + (k*D + off + 1)*gamma, advanced by D*gamma per step), the next
// step's delays drawn before the barrier, and the steady state (k >= q-1:
// bound = q-1, modulus q) free of branches.
template <int PT, int LAW>
__global__ void __launch_bounds__(1024) ensemble_kernel(const EnsembleArgs a) {
    extern __shared__ __align__(16) double hist[];  // [(q+1)][n], then the q-1 thresholds
    const int n = a.n, q = a.q, Q = a.q + 1, T = blockDim.x, t = threadIdx.x;
    const unsigned long long seed = a.base_seed + blockIdx.x;
    using A = Arith<double>;
    uint64_t* gthr = reinterpret_cast<uint64_t*>(hist + (size_t)Q * n);
    if (LAW == 2)
        for (int j = t; j < q - 1; j += T) gthr[j] = a.gthr[j];
    for (int i = t; i < n; i += T) hist[i] = a.u0[i];  // slot 0 = step 0
    __syncthreads();
    if (t == 0 && a.norms) a.norms[(size_t)blockIdx.x * a.n_rec] = seq_l2(hist, n);
    if (a.rows)
        for (int i = t; i < n; i += T) a.rows[i] = hist[i];

    int ci[PT], li[PT], ri[PT], offL[PT], offR[PT], dL[PT], dR[PT];
    bool live[PT], pin[PT];
    double pinv[PT];
    unsigned long long zL[PT], zR[PT];
    const unsigned long long zstep = (unsigned long long)a.D * kGamma;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
        const int i = t + j * T;
        live[j] = i < n;
        ci[j] = live[j] ? i : 0;
        // pinned ends take no draws (async_sim.cpp:92-95)
        pin[j] = a.dirichlet && (ci[j] == 0 || ci[j] == n - 1);
        pinv[j] = ci[j] == 0 ? a.c1 : a.c2;
        li[j] = ci[j] == 0 ? n - 1 : ci[j] - 1;
        ri[j] = ci[j] == n - 1 ? 0 : ci[j] + 1;
        offL[j] = live[j] ? a.offL[ci[j]] : -1;
        offR[j] = live[j] ? a.offR[ci[j]] : -1;
        zL[j] = seed + ((unsigned long long)(offL[j] < 0 ? 0 : offL[j]) + 1) * kGamma;
        zR[j] = seed + ((unsigned long long)(offR[j] < 0 ? 0 : offR[j]) + 1) * kGamma;
    }
    // delays of step kk for any kk (bound = min(kk, q-1)); advances z to kk+1
    auto draw_generic = [&](long long kk) {
        const long long bound = kk < q - 1 ? kk : q - 1;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            if (LAW == 0) {
                dL[j] = offL[j] < 0 || bound == 0
                            ? 0 : int(splitmix_mix(zL[j]) % (unsigned long long)(bound + 1));
                dR[j] = offR[j] < 0 || bound == 0
                            ? 0 : int(splitmix_mix(zR[j]) % (unsigned long long)(bound + 1));
            } else if (LAW == 1) {
                const int d = a.fixed_d < bound ? a.fixed_d : int(bound);
                dL[j] = offL[j] < 0 ? 0 : d;
                dR[j] = offR[j] < 0 ? 0 : d;
            } else {
                dL[j] = offL[j] < 0 ? 0 : geometric_delay(splitmix_mix(zL[j]), gthr, int(bound));
                dR[j] = offR[j] < 0 ? 0 : geometric_delay(splitmix_mix(zR[j]), gthr, int(bound));
            }
            zL[j] += zstep;
            zR[j] += zstep;
        }
    };
    // delays of a step kk >= q-1 (modulus q; a fixed d < q is never clamped)
    auto draw_steady = [&]() {
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            if (LAW == 0) {
                const int xl = int(modq(splitmix_mix(zL[j]), a.modq));
                const int xr = int(modq(splitmix_mix(zR[j]), a.modq));
                dL[j] = offL[j] < 0 ? 0 : xl;
                dR[j] = offR[j] < 0 ? 0 : xr;
                zL[j] += zstep;
                zR[j] += zstep;
            } else if (LAW == 1) {
                dL[j] = offL[j] < 0 ? 0 : a.fixed_d;
                dR[j] = offR[j] < 0 ? 0 : a.fixed_d;
            } else {
                const int xl = geometric_delay(splitmix_mix(zL[j]), gthr, q - 1);
                const int xr = geometric_delay(splitmix_mix(zR[j]), gthr, q - 1);
                dL[j] = offL[j] < 0 ? 0 : xl;
                dR[j] = offR[j] < 0 ? 0 : xr;
                zL[j] += zstep;
                zR[j] += zstep;
            }
        }
    };
    int slot = 0;  // k mod Q, a wrapped counter
    long long next_rec = a.stride;
    int rec = 1;
    // step k: read slots of steps k-d, write slot k+1; left before right is
    // the reference's draw order (async_sim.cpp:98-99), encoded in off*
    auto compute = [&](int nslot) {
        const double* cur = hist + slot * n;
        double* out = hist + nslot * n;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            const int sl = slot - dL[j] < 0 ? slot - dL[j] + Q : slot - dL[j];
            const int sr = slot - dR[j] < 0 ? slot - dR[j] + Q : slot - dR[j];
            const double left = hist[sl * n + li[j]];
            const double right = hist[sr * n + ri[j]];
            const double v = stencil_p(A::mul(a.r, right), A::mul(a.c, cur[ci[j]]), A::mul(a.r, left));
            if (live[j]) out[ci[j]] = pin[j] ? pinv[j] : v;
        }
    };
    auto finish = [&](long long k, int nslot) {
        slot = nslot;
        __syncthreads();
        if (k + 1 == next_rec || (k + 1 == a.k_end && next_rec != k + 1)) {
            if (t == 0 && a.norms)
                a.norms[(size_t)blockIdx.x * a.n_rec + rec] = seq_l2(hist + slot * n, n);
            if (a.rows)
                for (int i = t; i < n; i += T) a.rows[(size_t)rec * n + i] = hist[slot * n + i];
            ++rec;
            if (k + 1 == next_rec) next_rec += a.stride;
        }
    };
    draw_generic(0);
    long long k = 0;
    const long long k_gen = a.k_end < (long long)q - 2 ? a.k_end : (long long)(q > 2 ? q - 2 : 0);
    for (; k < k_gen; ++k) {  // the next step still has bound < q-1
        const int nslot = slot + 1 == Q ? 0 : slot + 1;
        compute(nslot);
        draw_generic(k + 1);
        finish(k, nslot);
    }
    for (; k < a.k_end; ++k) {
        const int nslot = slot + 1 == Q ? 0 : slot + 1;
        compute(nslot);
        draw_steady();  // next step's delays overlap this step's loads and the barrier
        finish(k, nslot);
    }
    const double* fin = hist + slot * n;  // slot == k_end mod Q
    bool bad = false;
    for (int i = t; i < n; i += T) {
        bad |= !isfinite(fin[i]);
        if (a.terminals) a.terminals[(size_t)blockIdx.x * n + i] = fin[i];
    }
    if (bad) atomicOr(a.flag, 1u);
}

using EnsembleKernel = void (*)(const EnsembleArgs);
EnsembleKernel pick_kernel(int pt, int law) {
    const EnsembleKernel k[3][3] = {
        {ensemble_kernel<1, 0>, ensemble_kernel<1, 1>, ensemble_kernel<1, 2>},
        {ensemble_kernel<2, 0>, ensemble_kernel<2, 1>, ensemble_kernel<2, 2>},
        {ensemble_kernel<4, 0>, ensemble_kernel<4, 1>, ensemble_kernel<4, 2>}};
    return k[pt == 1 ? 0 : pt == 2 ? 1 : 2][law];
}

// In-step draw rank of every read of async_step_into (async_sim.cpp:86-101),
// per point: ascending i, pinned ends skipped, left before right, only when
// the neighbour lies in another PE.
long long point_offsets(int n, int per_pe, bool dirichlet, std::vector<int>& offL,
                        std::vector<int>& offR) {
    offL.assign(n, -1);
    offR.assign(n, -1);
    long long cnt = 0;
    for (int i = 0; i < n; ++i) {
        if (dirichlet && (i == 0 || i == n - 1)) continue;
        const int li = i == 0 ? n - 1 : i - 1;
        const int ri = i == n - 1 ? 0 : i + 1;
        if (i / per_pe != li / per_pe) offL[i] = int(cnt++);
        if (i / per_pe != ri / per_pe) offR[i] = int(cnt++);
    }
    return cnt;
}

// mean / population std per recorded step, the reference's loop order
// (analysis.cpp:88-103)
void series_stats(const std::vector<double>& hn, size_t runs, size_t S, double* mean_series,
                  double* std_series) {
    for (size_t s = 0; s < S; ++s) {
        double mean = 0.0;
        for (size_t j = 0; j < runs; ++j) mean += hn[j * S + s];
        mean /= double(runs);
        double var = 0.0;
        for (size_t j = 0; j < runs; ++j) {
            const double dd = hn[j * S + s] - mean;
            var += dd * dd;
        }
        if (mean_series) mean_series[s] = mean;
        if (std_series) std_series[s] = std::sqrt(var / double(runs));
    }
}

// l2_norm of a device field in the reference's order (one thread); flag |= 1
// when the field holds a non-finite value (the terminal TemperatureField).
__global__ void member_norm_kernel(const double* __restrict__ v, long long n, double* out,
                                   unsigned int* flag) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (long long i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(v[i], v[i]));
        *out = sqrt(s);
    }
    if (flag) {
        bool bad = false;
        for (long long i = threadIdx.x; i < n; i += blockDim.x) bad |= !isfinite(v[i]);
        if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
    }
}

// run_member (analysis.cpp:16-38) for each member on a GPU AsyncSimulator
// handle: K3 for PEs <= 1024 points, K5 for wider ones.
int ensemble_via_simulators(const double* u0, size_t n, double r, int bc_kind, double c1,
                            double c2, size_t per_pe, size_t q, int law, size_t fixed_delay,
                            double geometric_p, const std::vector<size_t>& steps, size_t runs,
                            uint64_t base_seed, std::vector<double>& hn, double* terminals) {
    const size_t S = steps.size();
    double* dn = nullptr;
    unsigned int* dflag = nullptr;
    struct Bufs {
        double*& dn;
        unsigned int*& f;
        ~Bufs() {
            if (dn) cudaFree(dn);
            if (f) cudaFree(f);
        }
    } bufs{dn, dflag};
    HB_CUDA(cudaMalloc(&dn, S * sizeof(double)));
    HB_CUDA(cudaMalloc(&dflag, sizeof(unsigned int)));
    for (size_t j = 0; j < runs; ++j) {
        heat_async_sim* sim = nullptr;
        HB_TRY(heat_async_sim_create(&sim, u0, n, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay,
                                     geometric_p, base_seed + j));
        struct Guard {
            heat_async_sim* s;
            ~Guard() { heat_async_sim_destroy(s); }
        } guard{sim};
        size_t k = 0;
        const double* field = nullptr;
        cudaStream_t st = nullptr;
        for (size_t s = 0; s < S; ++s) {
            if (steps[s] > k) HB_TRY(heat_async_sim_step(sim, steps[s] - k));
            k = steps[s];
            async_sim_device_field(sim, &field, &st);
            const bool last = s + 1 == S;
            if (last) HB_CUDA(cudaMemsetAsync(dflag, 0, sizeof(unsigned int), st));
            member_norm_kernel<<<1, 256, 0, st>>>(field, (long long)n, dn + s,
                                                  last ? dflag : nullptr);
            HB_CUDA(cudaGetLastError());
            g_launches.fetch_add(1, std::memory_order_relaxed);
        }
        unsigned int bad = 0;
        HB_CUDA(cudaMemcpyAsync(hn.data() + j * S, dn, S * sizeof(double), cudaMemcpyDeviceToHost,
                                st));
        HB_CUDA(cudaMemcpyAsync(&bad, dflag, sizeof bad, cudaMemcpyDeviceToHost, st));
        if (terminals)
            HB_CUDA(cudaMemcpyAsync(terminals + j * n, field, n * sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        if (bad) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    return HEAT_OK;
}

}  // namespace
}  // namespace hb


namespace hb {
// async_run (async_sim.cpp:142-160) of a small field whose PEs K9 does not lay
// out (e.g. the paper's one point per PE): one K6 member with seed `seed`
// (member j of an ensemble draws from base_seed + j: the same stream), the
// trajectory rows written by the kernel.  K3 steps these at ~600 ns/step,
// K6 at ~230 (N = 100, q = 5; tools/probe_paper_member.py).  K6's step is
// one CTA barrier per step over all N points, K3's a warp per PE: K6 wins up
// to ~640 points (N = 600, PEs of 75: 585 vs 701 ns/step) and for PEs of
// fewer than 8 points at any N <= 1024 (N = 1024, PEs of 4: 919 vs 2159);
// K3 wins for N = 1000 with PEs of 10-125 (700-810 vs 920)
// (tools/probe_member_vs_k3.py).
bool async_member_eligible(size_t n, size_t per_pe, size_t q) {
    if (std::getenv("HEAT_NO_MEMBER_ASYNC")) return false;
    return n >= 3 && n <= 1024 && (n <= 640 || per_pe < 8) &&
           (q + 1) * n * sizeof(double) + q * 8 <= 200 * 1024;
}

int async_run_member(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                     size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                     uint64_t seed, size_t k_end, size_t stride, double* final_out,
                     double* snapshots, size_t* steps_out, size_t max_snapshots,
                     size_t* n_snapshots) {
    std::vector<size_t> steps{0};
    for (size_t k = stride; k < k_end; k += stride) steps.push_back(k);
    if (k_end > 0 && steps.back() != k_end) steps.push_back(k_end);
    const size_t S = steps.size();
    const bool want = snapshots != nullptr || steps_out != nullptr;
    std::vector<uint64_t> gthr;
    if (law == HEAT_DELAY_GEOMETRIC) HB_TRY(geometric_thresholds(geometric_p, q, gthr));
    const int PT = n <= 1024 ? 1 : n <= 2048 ? 2 : 4;
    const int T = int(((n + PT - 1) / PT + 31) / 32 * 32);
    const size_t smem = (q + 1) * n * sizeof(double) + gthr.size() * sizeof(uint64_t);

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const bool dir = bc_kind == HEAT_BC_DIRICHLET;
    std::vector<int> offL, offR;
    const long long D = point_offsets(int(n), int(per_pe), dir, offL, offR);
    auto a256 = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t o_u0 = 0, o_offL = o_u0 + a256(n * 8), o_offR = o_offL + a256(n * 4),
                 o_gthr = o_offR + a256(n * 4), o_term = o_gthr + a256(gthr.size() * 8 + 8),
                 o_rows = o_term + a256(n * 8), total = o_rows + a256(want ? S * n * 8 : 8);
    HB_TRY(ensure_scratch(*d, total));
    char* base = static_cast<char*>(d->scratch);
    cudaStream_t st = d->stream;
    HB_TRY(upload_prepared(*d, u0, n, bc_kind, c1, c2, reinterpret_cast<double*>(base + o_u0)));
    HB_CUDA(cudaMemcpyAsync(base + o_offL, offL.data(), n * 4, cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemcpyAsync(base + o_offR, offR.data(), n * 4, cudaMemcpyHostToDevice, st));
    if (!gthr.empty())
        HB_CUDA(cudaMemcpyAsync(base + o_gthr, gthr.data(), gthr.size() * 8, cudaMemcpyHostToDevice,
                                st));
    HB_CUDA(cudaMemsetAsync(d->flag, 0, 2 * sizeof(unsigned int), st));
    EnsembleArgs a{};
    a.u0 = reinterpret_cast<const double*>(base + o_u0);
    a.n = int(n);
    a.r = r;
    a.c = 1.0 - 2.0 * r;  // core.hpp:108
    a.c1 = c1;
    a.c2 = c2;
    a.dirichlet = dir;
    a.q = int(q);
    a.law = law;
    a.fixed_d = int(std::min<size_t>(fixed_delay, 1u << 30));
    a.gthr = reinterpret_cast<const uint64_t*>(base + o_gthr);
    a.base_seed = seed;
    a.modq = make_modq(unsigned(q));
    a.D = D;
    a.offL = reinterpret_cast<const int*>(base + o_offL);
    a.offR = reinterpret_cast<const int*>(base + o_offR);
    a.k_end = (long long)k_end;
    a.stride = (long long)stride;
    a.n_rec = int(S);
    a.norms = nullptr;
    a.terminals = reinterpret_cast<double*>(base + o_term);
    a.rows = want ? reinterpret_cast<double*>(base + o_rows) : nullptr;
    a.flag = d->flag;
    const EnsembleKernel kern = pick_kernel(PT, law);
    if (smem > 48 * 1024)
        HB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<1, T, smem, st>>>(a);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const size_t copy = std::min(S, max_snapshots);
    if (want && snapshots && copy)
        HB_CUDA(cudaMemcpyAsync(snapshots, a.rows, copy * n * 8, cudaMemcpyDeviceToHost, st));
    if (final_out)
        HB_CUDA(cudaMemcpyAsync(final_out, a.terminals, n * 8, cudaMemcpyDeviceToHost, st));
    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d->flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    if (steps_out)
        for (size_t j = 0; j < S && j < max_snapshots; ++j) steps_out[j] = steps[j];
    if (n_snapshots) *n_snapshots = want ? S : 0;
    return HEAT_OK;
}
}  // namespace hb

using namespace hb;

extern "C" int heat_ensemble_run(const double* u0, size_t n, double r, int bc_kind, double c1,
                                 double c2, size_t per_pe, size_t q, int law, size_t fixed_delay,
                                 double geometric_p, size_t k_end, size_t stride, size_t runs, uint64_t base_seed,
                                 size_t* steps_out, size_t max_steps, size_t* n_steps,
                                 double* norms, double* terminals, double* mean_series,
                                 double* std_series) {
    // EnsembleConfig holds a TemperatureField, PartitionSpec and DelayModel
    // (validated at construction); ensemble_run itself checks M.
    if (n < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u0) return fail(HEAT_EINVAL, "null field pointer");
    if (per_pe == 0 || n % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (law == HEAT_DELAY_FIXED && fixed_delay >= q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    if (law < 0 || law > 2) return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
    if (runs == 0) return fail(HEAT_EDOMAIN, "ensemble_run: M >= 1 required");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    if (stride == 0) stride = default_stride(n);

    // recorded steps (analysis.cpp:56-60)
    std::vector<size_t> steps{0};
    for (size_t k = stride; k < k_end; k += stride) steps.push_back(k);
    if (k_end > 0 && steps.back() != k_end) steps.push_back(k_end);
    const size_t S = steps.size();
    if (steps_out)
        for (size_t s = 0; s < S && s < max_steps; ++s) steps_out[s] = steps[s];
    if (n_steps) *n_steps = S;

    std::vector<uint64_t> gthr;
    if (law == HEAT_DELAY_GEOMETRIC) HB_TRY(geometric_thresholds(geometric_p, q, gthr));
    constexpr size_t kMaxPoints = 4096;
    const size_t smem = (q + 1) * n * sizeof(double) + gthr.size() * sizeof(uint64_t);
    std::vector<double> hn(runs * S);
    if (n > kMaxPoints || smem > 200 * 1024) {
        // the field or its history does not fit one CTA: members through
        // AsyncSimulator handles (K3 / K5) one after another
        HB_TRY(ensemble_via_simulators(u0, n, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay,
                                       geometric_p, steps, runs, base_seed, hn, terminals));
        if (norms) std::copy(hn.begin(), hn.end(), norms);
        series_stats(hn, runs, S, mean_series, std_series);
        return HEAT_OK;
    }
    const int PT = n <= 1024 ? 1 : n <= 2048 ? 2 : 4;
    const int T = int(((n + PT - 1) / PT + 31) / 32 * 32);

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const bool dir = bc_kind == HEAT_BC_DIRICHLET;
    std::vector<int> offL, offR;
    const long long D = point_offsets(int(n), int(per_pe), dir, offL, offR);
    // device scratch: u0 | offL | offR | thresholds | norms | terminals
    auto a256 = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t o_u0 = 0, o_offL = o_u0 + a256(n * 8), o_offR = o_offL + a256(n * 4),
                 o_gthr = o_offR + a256(n * 4), o_norms = o_gthr + a256(gthr.size() * 8 + 8),
                 o_term = o_norms + a256(runs * S * 8),
                 total = o_term + a256(terminals ? runs * n * 8 : 8);
    HB_TRY(ensure_scratch(*d, total));
    char* base = static_cast<char*>(d->scratch);
    cudaStream_t st = d->stream;
    HB_TRY(upload_prepared(*d, u0, n, bc_kind, c1, c2, reinterpret_cast<double*>(base + o_u0)));
    HB_CUDA(cudaMemcpyAsync(base + o_offL, offL.data(), n * 4, cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemcpyAsync(base + o_offR, offR.data(), n * 4, cudaMemcpyHostToDevice, st));
    if (!gthr.empty())
        HB_CUDA(cudaMemcpyAsync(base + o_gthr, gthr.data(), gthr.size() * 8, cudaMemcpyHostToDevice,
                                st));
    HB_CUDA(cudaMemsetAsync(d->flag, 0, 2 * sizeof(unsigned int), st));

    EnsembleArgs a{};
    a.u0 = reinterpret_cast<const double*>(base + o_u0);
    a.n = int(n);
    a.r = r;
    a.c = 1.0 - 2.0 * r;  // core.hpp:108
    a.c1 = c1;
    a.c2 = c2;
    a.dirichlet = dir;
    a.q = int(q);
    a.law = law;
    a.fixed_d = int(std::min<size_t>(fixed_delay, 1u << 30));
    a.gthr = reinterpret_cast<const uint64_t*>(base + o_gthr);
    a.base_seed = base_seed;
    a.modq = make_modq(unsigned(q));
    a.D = D;
    a.offL = reinterpret_cast<const int*>(base + o_offL);
    a.offR = reinterpret_cast<const int*>(base + o_offR);
    a.k_end = (long long)k_end;
    a.stride = (long long)stride;
    a.n_rec = int(S);
    a.norms = reinterpret_cast<double*>(base + o_norms);
    a.terminals = terminals ? reinterpret_cast<double*>(base + o_term) : nullptr;
    a.flag = d->flag;
    const EnsembleKernel kern = pick_kernel(PT, law);
    if (smem > 48 * 1024)
        HB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(runs), T, smem, st>>>(a);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);

    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(hn.data(), base + o_norms, runs * S * 8, cudaMemcpyDeviceToHost, st));
    if (terminals)
        HB_CUDA(cudaMemcpyAsync(terminals, base + o_term, runs * n * 8, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaMemcpyAsync(flags, d->flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    if (norms) std::copy(hn.begin(), hn.end(), norms);
    series_stats(hn, runs, S, mean_series, std_series);
    return HEAT_OK;
}
