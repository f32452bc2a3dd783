// history.cu -- HistoryRing (async_sim.hpp:31-57) in HBM and async_step
// (async_sim.hpp:68-71, async_sim.cpp:77-116) as two kernels over it.
//
// The reference keeps the last q full fields in a host ring and steps one
// field at a time, pulling each cross-PE neighbour from the snapshot its drawn
// delay selects.  Here the ring's snapshots are device buffers of N doubles
// (depth + 1 of them: the spare receives the next step, then rotates in on
// push, so a push moves no data).  One step is
//
//   K8a step_body_kernel   every point from the current snapshot: the
//                          synchronous update, Dirichlet ends pinned,
//                          periodic ends wrapped -- 16 B/point, HBM-bound;
//   K8b step_edges_kernel  one thread per PE: its first / last point again
//                          with the cross-PE neighbour read at the drawn
//                          depth (counter-form SplitMix64 draws in the
//                          reference's order, draw_offsets()).
//
// The caller's SplitMix64 state is advanced exactly as the reference's
// stream: by D draws for a completed step, and only through the failing draw
// when a delay reaches past the ring (HistoryRing::read's logic_error,
// async_sim.cpp:41-44).  Strict finite checks run after the step
// (async_sim.cpp:102-105): DivergenceError, the ring unchanged.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "runtime.cuh"

using namespace hb;

struct heat_history {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    size_t depth = 0, n = 0, step = 0, count = 0;
    std::vector<double*> buf;      // depth + 1 device fields (one allocation)
    std::vector<int> slot;         // slot[d] = buffer holding u(step - d), d < count
    int spare = 0;                 // buffer the next step is written into
    double* base = nullptr;
    // per-call scratch: snapshot table, draw offsets, geometric delays, flags
    const double** tab = nullptr;  // device [depth]
    int* offs = nullptr;           // device [2P]: offL then offR
    size_t offs_cap = 0;
    size_t offs_key_pe = 0;
    int offs_key_bc = -1;
    int D = 0;
    uint64_t* gthr = nullptr;      // geometric law: delay thresholds of (gthr_p, gthr_q)
    double gthr_p = -1.0;
    size_t gthr_q = 0;
    unsigned long long* flags = nullptr;  // [0] first failing draw, [1] non-finite
};

namespace {

constexpr unsigned long long kNoFail = ~0ull;

// K8a: the synchronous step from `cur` into `out` (sync_step_into,
// sync_solver.hpp:26-39): two points per thread, 16-B loads.
__global__ void step_body_kernel(const double* __restrict__ cur, double* __restrict__ out,
                                 long long n, double r, double c, int dirichlet, double c1,
                                 double c2) {
    using A = Arith<double>;
    const long long pairs = (n + 1) / 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < pairs;
         t += (long long)gridDim.x * blockDim.x) {
        const long long i = 2 * t;
        double s0, s1;
        if (i + 1 < n) {
            const double2 v = *reinterpret_cast<const double2*>(cur + i);
            s0 = v.x;
            s1 = v.y;
        } else {
            s0 = cur[i];
            s1 = cur[0];  // odd n: point i = n-1 alone, its right neighbour wraps
        }
        const double L = cur[i == 0 ? n - 1 : i - 1];
        const double R = i + 2 < n ? cur[i + 2] : cur[i + 2 - n];  // wraps to cur[0] / cur[1]
        // point i: (L, s0, s1); point i+1: (s0, s1, R)
        const double ps1 = A::mul(r, s1), ps0 = A::mul(r, s0);
        double o0 = stencil_p(ps1, A::mul(c, s0), A::mul(r, L));
        double o1 = stencil_p(A::mul(r, R), A::mul(c, s1), ps0);
        if (dirichlet) {
            if (i == 0) o0 = c1;
            if (i == n - 1) o0 = c2;
            if (i + 1 == n - 1) o1 = c2;
        }
        if (i + 1 < n) {
            *reinterpret_cast<double2*>(out + i) = make_double2(o0, o1);
        } else {
            out[i] = o0;
        }
    }
}

struct EdgeArgs {
    const double* cur;
    const double* const* tab;  // tab[d] = u(k - d)
    double* out;
    const int* offL;
    const int* offR;
    const uint64_t* gthr;       // geometric law: the q-1 delay thresholds
    unsigned long long* fail;   // lowest failing draw rank
    long long N, n, P;
    double r, c;
    uint64_t state;             // the caller's SplitMix64 state before the step
    long long bound;            // min(q - 1, k)
    long long count;            // snapshots held: a delay >= count is a logic_error
    int law;
    long long fixed_d;
};

__device__ __forceinline__ double stale_read(const EdgeArgs& a, long long j, int off, bool& ok) {
    long long d;
    if (a.law == HEAT_DELAY_UNIFORM) {
        d = (long long)(splitmix_draw(a.state, uint64_t(off)) % uint64_t(a.bound + 1));
    } else if (a.law == HEAT_DELAY_FIXED) {
        d = a.fixed_d < a.bound ? a.fixed_d : a.bound;
    } else {
        d = geometric_delay(splitmix_draw(a.state, uint64_t(off)), a.gthr, int(a.bound));
    }
    if (d >= a.count) {
        atomicMin(a.fail, (unsigned long long)off);
        ok = false;
        return 0.0;
    }
    return a.tab[d][j];
}

// K8b: the PE-boundary points of every PE with their stale reads (async_step_into,
// async_sim.cpp:77-101).  Runs after K8a on the same stream and overwrites them.
__global__ void step_edges_kernel(EdgeArgs a) {
    using A = Arith<double>;
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= a.P) return;
    const long long first = p * a.n, last = first + a.n - 1;
    const int oL = a.offL[p], oR = a.offR[p];
    bool ok = true;
    if (oL >= 0) {  // first point: left neighbour in PE p-1 (or the wrap)
        const long long i = first;
        const long long li = i == 0 ? a.N - 1 : i - 1, ri = i == a.N - 1 ? 0 : i + 1;
        const double L = stale_read(a, li, oL, ok);
        const double R = (a.n == 1) ? stale_read(a, ri, oR, ok) : a.cur[ri];
        if (ok) a.out[i] = stencil_p(A::mul(a.r, R), A::mul(a.c, a.cur[i]), A::mul(a.r, L));
    }
    if (oR >= 0 && a.n >= 2) {  // last point: right neighbour in PE p+1 (or the wrap)
        const long long i = last;
        const long long li = i - 1, ri = i == a.N - 1 ? 0 : i + 1;
        const double R = stale_read(a, ri, oR, ok);
        if (ok) a.out[i] = stencil_p(A::mul(a.r, R), A::mul(a.c, a.cur[i]), A::mul(a.r, a.cur[li]));
    }
}

__global__ void nonfinite_kernel(const double* __restrict__ u, long long n,
                                 unsigned long long* flag) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        bad |= !isfinite(u[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1ull);
}

void history_free(heat_history* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->base) cudaFree(h->base);
    if (h->tab) cudaFree(h->tab);
    if (h->offs) cudaFree(h->offs);
    if (h->gthr) cudaFree(h->gthr);
    if (h->flags) cudaFree(h->flags);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

int check_depth(const heat_history* h, size_t d) {
    if (d >= h->depth || d > h->step || d >= h->count)
        return fail(HEAT_ELOGIC, "HistoryRing: read depth out of range");
    return HEAT_OK;
}

}  // namespace

extern "C" {

int heat_history_create(heat_history** out, size_t depth, size_t n, size_t step,
                        const double* snapshots, size_t count, int device) {
    if (!out) return fail(HEAT_EINVAL, "null history handle");
    *out = nullptr;
    if (depth == 0) return fail(HEAT_EDOMAIN, "HistoryRing: depth >= 1 required");
    if (n < 3) return fail(HEAT_EDOMAIN, "HistoryRing: N >= 3 required");
    if (!snapshots) return fail(HEAT_EINVAL, "null snapshot pointer");
    if (count != std::min(depth, step + 1))
        return fail(HEAT_ELOGIC, "HistoryRing: count must equal min(depth, step + 1)");
    DevCtx* ctx = nullptr;
    HB_TRY(dev_ctx(device, &ctx));  // device checks (sm_100); leaves `device` current
    const int sms = ctx->sms;
    device = ctx->device;
    auto* h = new heat_history();
    struct Guard {
        heat_history*& p;
        ~Guard() {
            if (p) history_free(p);
        }
    } guard{h};
    h->device = device;
    h->sms = sms;
    h->depth = depth;
    h->n = n;
    h->step = step;
    h->count = count;
    HB_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    const size_t pitch = (n + 31) / 32 * 32;
    if (cudaMalloc(&h->base, (depth + 1) * pitch * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(HEAT_ENOMEM, "HistoryRing: device allocation failed");
    }
    h->buf.resize(depth + 1);
    for (size_t b = 0; b <= depth; ++b) h->buf[b] = h->base + b * pitch;
    h->slot.assign(depth, -1);
    for (size_t d = 0; d < count; ++d) {
        h->slot[d] = int(d);
        HB_CUDA(cudaMemcpyAsync(h->buf[d], snapshots + d * n, n * sizeof(double),
                                cudaMemcpyHostToDevice, h->stream));
    }
    // the buffers not holding a snapshot: the first is the spare
    h->spare = int(count);
    HB_CUDA(cudaMalloc(&h->tab, depth * sizeof(double*)));
    HB_CUDA(cudaMalloc(&h->flags, 2 * sizeof(unsigned long long)));
    HB_CUDA(cudaStreamSynchronize(h->stream));
    *out = h;
    h = nullptr;
    return HEAT_OK;
}

int heat_history_destroy(heat_history* h) {
    history_free(h);
    return HEAT_OK;
}

int heat_history_info(const heat_history* h, size_t* depth, size_t* current_step,
                      size_t* grid_size) {
    if (!h) return fail(HEAT_EINVAL, "null history handle");
    if (depth) *depth = h->depth;
    if (current_step) *current_step = h->step;
    if (grid_size) *grid_size = h->n;
    return HEAT_OK;
}

// HistoryRing::push (async_sim.cpp:33-40) of a host state.
int heat_history_push(heat_history* h, const double* state, size_t n) {
    if (!h) return fail(HEAT_EINVAL, "null history handle");
    if (n != h->n) return fail(HEAT_ELOGIC, "HistoryRing: state size mismatch");
    if (!state) return fail(HEAT_EINVAL, "null state pointer");
    HB_CUDA(cudaSetDevice(h->device));
    const int b = h->spare;
    HB_CUDA(cudaMemcpyAsync(h->buf[b], state, n * sizeof(double), cudaMemcpyHostToDevice,
                            h->stream));
    HB_CUDA(cudaStreamSynchronize(h->stream));
    const int evicted = h->count == h->depth ? h->slot[h->depth - 1] : -1;
    for (size_t d = h->depth - 1; d > 0; --d) h->slot[d] = h->slot[d - 1];
    h->slot[0] = b;
    ++h->step;
    if (h->count < h->depth) ++h->count;
    h->spare = evicted >= 0 ? evicted : int(h->count);
    return HEAT_OK;
}

// HistoryRing::read / snapshot (async_sim.cpp:42-55).
int heat_history_read(const heat_history* h, size_t i, size_t d, double* value) {
    if (!h || !value) return fail(HEAT_EINVAL, "null history handle or output");
    HB_TRY(check_depth(h, d));
    if (i >= h->n) return fail(HEAT_EINVAL, "HistoryRing: point index out of range");
    HB_CUDA(cudaSetDevice(h->device));
    HB_CUDA(cudaMemcpyAsync(value, h->buf[h->slot[d]] + i, sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream));
    HB_CUDA(cudaStreamSynchronize(h->stream));
    return HEAT_OK;
}

int heat_history_snapshot(const heat_history* h, size_t d, double* out) {
    if (!h || !out) return fail(HEAT_EINVAL, "null history handle or output");
    HB_TRY(check_depth(h, d));
    HB_CUDA(cudaSetDevice(h->device));
    HB_CUDA(cudaMemcpyAsync(out, h->buf[h->slot[d]], h->n * sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream));
    HB_CUDA(cudaStreamSynchronize(h->stream));
    return HEAT_OK;
}

// async_step (async_sim.cpp:107-116) over the device ring.  `out` (host, may be
// NULL) receives the new field; `push` != 0 also pushes it into the ring
// (AsyncSimulator::step, async_sim.cpp:136-140) without a host round trip.
int heat_async_step(heat_history* h, double r, int bc_kind, double c1, double c2,
                    size_t part_total, size_t per_pe, size_t q, int law, size_t fixed_delay,
                    double geometric_p, uint64_t* rng_state, double* out, int push) {
    if (!h || !rng_state) return fail(HEAT_EINVAL, "null history handle or rng state");
    // the caller's objects validate first: DelayModel and PartitionSpec ctors
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (law == HEAT_DELAY_FIXED && fixed_delay >= q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    if (part_total < 3) return fail(HEAT_EDOMAIN, "PartitionSpec: N >= 3 required");
    if (per_pe == 0 || part_total % per_pe != 0)
        return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (part_total != h->n)
        return fail(HEAT_EINVAL, "async_step: partition inconsistent with grid");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    if (law < 0 || law > 2) return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
    HB_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = h->stream;
    const size_t N = h->n, P = N / per_pe;
    const int dir = bc_kind == HEAT_BC_DIRICHLET;

    // draw ranks of the cross-PE reads, cached per (partition, bc)
    if (h->offs_key_pe != per_pe || h->offs_key_bc != bc_kind) {
        std::vector<int> offL, offR;
        h->D = draw_offsets(N, per_pe, dir, offL, offR);
        if (h->offs_cap < 2 * P) {
            if (h->offs) cudaFree(h->offs);
            h->offs = nullptr;
            h->offs_cap = 0;
            HB_CUDA(cudaMalloc(&h->offs, 2 * P * sizeof(int)));
            h->offs_cap = 2 * P;
        }
        offL.insert(offL.end(), offR.begin(), offR.end());
        HB_CUDA(cudaMemcpy(h->offs, offL.data(), 2 * P * sizeof(int), cudaMemcpyHostToDevice));
        h->offs_key_pe = per_pe;
        h->offs_key_bc = bc_kind;
    }
    const int D = h->D;
    const size_t k = h->step;
    const long long bound = (long long)std::min(q - 1, k);

    // geometric law: exact device delays from the thresholds (geometric_thresholds)
    if (law == HEAT_DELAY_GEOMETRIC && (h->gthr_p != geometric_p || h->gthr_q != q)) {
        std::vector<uint64_t> gthr;
        HB_TRY(geometric_thresholds(geometric_p, q, gthr));
        if (h->gthr) cudaFree(h->gthr);
        h->gthr = nullptr;
        h->gthr_q = 0;
        HB_CUDA(cudaMalloc(&h->gthr, std::max<size_t>(1, gthr.size()) * sizeof(uint64_t)));
        if (!gthr.empty())
            HB_CUDA(cudaMemcpy(h->gthr, gthr.data(), gthr.size() * sizeof(uint64_t),
                               cudaMemcpyHostToDevice));
        h->gthr_p = geometric_p;
        h->gthr_q = q;
    }

    std::vector<const double*> tab(h->depth, nullptr);
    for (size_t d = 0; d < h->count; ++d) tab[d] = h->buf[h->slot[d]];
    HB_CUDA(cudaMemcpyAsync(h->tab, tab.data(), h->depth * sizeof(double*),
                            cudaMemcpyHostToDevice, st));
    const unsigned long long init[2] = {kNoFail, 0};
    HB_CUDA(cudaMemcpyAsync(h->flags, init, sizeof init, cudaMemcpyHostToDevice, st));

    const double c = 1.0 - 2.0 * r;  // stencil, core.hpp:106-109
    double* cur = h->buf[h->slot[0]];
    double* nxt = h->buf[h->spare];
    const long long pairs = (long long)(N + 1) / 2;
    const int grid = int(std::min<long long>((pairs + 255) / 256, (long long)h->sms * 8));
    step_body_kernel<<<grid, 256, 0, st>>>(cur, nxt, (long long)N, r, c, dir, c1, c2);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (D > 0) {
        EdgeArgs a{};
        a.cur = cur;
        a.tab = h->tab;
        a.out = nxt;
        a.offL = h->offs;
        a.offR = h->offs + P;
        a.gthr = h->gthr;
        a.fail = h->flags;
        a.N = (long long)N;
        a.n = (long long)per_pe;
        a.P = (long long)P;
        a.r = r;
        a.c = c;
        a.state = *rng_state;
        a.bound = bound;
        a.count = (long long)h->count;
        a.law = law;
        a.fixed_d = (long long)fixed_delay;
        step_edges_kernel<<<int((P + 127) / 128), 128, 0, st>>>(a);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    const bool strict = g_strict.load();
    if (strict) {
        nonfinite_kernel<<<h->sms * 4, 256, 0, st>>>(nxt, (long long)N, h->flags + 1);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    unsigned long long flags[2];
    HB_CUDA(cudaMemcpyAsync(flags, h->flags, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (flags[0] != kNoFail) {  // the reference threw at that draw, after consuming it
        *rng_state += (flags[0] + 1) * 0x9e3779b97f4a7c15ULL;
        return fail(HEAT_ELOGIC, "HistoryRing: read depth out of range");
    }
    *rng_state += uint64_t(D) * 0x9e3779b97f4a7c15ULL;
    if (strict && flags[1])
        return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
    if (out) {
        HB_CUDA(cudaMemcpyAsync(out, nxt, N * sizeof(double), cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
    }
    if (push) {
        const int evicted = h->count == h->depth ? h->slot[h->depth - 1] : -1;
        for (size_t d = h->depth - 1; d > 0; --d) h->slot[d] = h->slot[d - 1];
        h->slot[0] = h->spare;
        ++h->step;
        if (h->count < h->depth) ++h->count;
        h->spare = evicted >= 0 ? evicted : int(h->count);
    }
    return HEAT_OK;
}

}  // extern "C"
