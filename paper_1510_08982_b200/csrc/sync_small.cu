// sync_small.cu -- K7: synchronous runs of small fields (N <= 16384, the
// paper's regime: cfg1 is N = 1024) in ONE CTA, the field resident in shared
// memory for the whole run.
//
// Replaces detail::sync_step_into iterated by run_impl (sync_solver.hpp:26-39,
// sync_solver.cpp:52-91) for small N, where K1's one launch per pass would be
// all launch latency.  Warp w owns the chunk [wC, (w+1)C) and keeps a window
// of 32 x V points -- the chunk plus a 64-point halo on each side -- in
// registers; it advances the window up to 64 steps with warp shuffles only
// (K1's step code), writes its exact chunk back to shared memory, and the
// CTA re-synchronises once per round, not once per step.  Dirichlet ends are
// re-pinned every step in the windows that hold them (reads beyond the field
// are zeros the pins cut off); periodic windows wrap.  Recorded steps end a
// round, and the kernel writes the trajectory rows itself.  Bit-identical to
// K1 and to the reference: the same stencil_p arithmetic on the same points.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "runtime.cuh"
#include "sync_tb.cuh"

namespace hb {
namespace {

struct SmallArgs {
    double* field;  // [n]: prepared initial field in, final field out
    int n;
    double r, c, c1, c2;
    int dirichlet;
    long long k_end;
    long long stride;  // 0: no trajectory
    double* snaps;     // [rows][n]: row 0 = step 0, row j = step j*stride, last row = k_end
    unsigned int* flag;
    int prep;  // validate the raw upload (flag[2], no steps) and snap the Dirichlet ends
};

constexpr int kSmallHalo = 64;  // steps per round = halo points per side

template <int V>
__global__ void __launch_bounds__(V <= 12 ? 1024 : 640, 1) sync_small_kernel(const SmallArgs a) {
    extern __shared__ double su[];
    constexpr int H = kSmallHalo, C = 32 * V - 2 * H;
    const int n = a.n, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    bool bad_in = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = a.field[i];
        bad_in |= !isfinite(v);
        su[i] = v;
    }
    if (a.prep) {
        // TemperatureField ctor (core.hpp:45-51) on the raw upload, then
        // prepare_initial's snap of the ends (the host checked |u - c| <= 1e-9)
        if (__syncthreads_or(bad_in)) {
            if (threadIdx.x == 0) atomicOr(a.flag + 2, 1u);
            return;
        }
        if (a.dirichlet && threadIdx.x == 0) {
            su[0] = a.c1;
            su[n - 1] = a.c2;
        }
    }
    __syncthreads();
    if (a.snaps)
        for (int i = threadIdx.x; i < n; i += blockDim.x) a.snaps[i] = su[i];
    const double r = a.r, c = a.c;
    const long long w0 = (long long)w * C - H;  // window start (unwrapped coordinates)
    const long long g0 = w0 + (long long)lane * V;
    const bool active = (long long)w * C < n;  // warp-uniform
    // windows holding a Dirichlet end re-pin it after every step
    const bool pinned = a.dirichlet && active && (w0 <= 0 || w0 + 32LL * V > n - 1);
    long long k = 0;
    long long next_rec = a.stride > 0 ? a.stride : a.k_end + 1;
    double u[V];
    while (k < a.k_end) {
        long long s = min((long long)H, a.k_end - k);
        s = min(s, next_rec - k);
        if (active) {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                long long g = g0 + i;
                if (a.dirichlet) {
                    u[i] = (g >= 0 && g < n) ? su[g] : 0.0;
                } else {
                    g %= n;
                    if (g < 0) g += n;
                    u[i] = su[g];
                }
            }
            if (pinned) {
                for (int t = 0; t < int(s); ++t) {
                    warp_step<double, V>(u, r, c);
                    pin_ends<double, V>(u, g0, 0, n - 1, a.c1, a.c2);
                }
            } else {
                warp_steps_pipelined<double, V>(u, r, c, int(s));
            }
        }
        __syncthreads();  // every window has been read before any chunk is written
        if (active) {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                const int idx = lane * V + i;
                const long long g = g0 + i;
                if (idx >= H && idx < H + C && g < n) su[g] = u[i];
            }
        }
        __syncthreads();
        k += s;
        if (a.snaps && (k == next_rec || k == a.k_end)) {
            const long long row = k % a.stride == 0 ? k / a.stride : k / a.stride + 1;
            for (int i = threadIdx.x; i < n; i += blockDim.x) a.snaps[row * n + i] = su[i];
            if (k == next_rec) next_rec += a.stride;
        }
    }
    bool bad = false;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bad |= !isfinite(su[i]);
        a.field[i] = su[i];
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flag, 1u);
}

}  // namespace

size_t sync_small_max_points() { return 16384; }

// Whole sync_run (or sync_step) of a small field on one CTA.  Validation as
// in sync_run_impl; trajectories are written by the kernel (0, stride,
// 2*stride, ..., k_end -- sync_solver.cpp:58-88).
int sync_run_small(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t k_end, size_t stride, double* final_out, double* snapshots,
                   size_t* steps_out, size_t max_snapshots, size_t* n_snapshots,
                   float* kernel_ms) {
    if (stride == 0) stride = default_stride(n);
    const bool want = snapshots != nullptr || steps_out != nullptr;
    const size_t rows = want ? 2 + k_end / stride : 0;  // upper bound (k_end not a multiple)
    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const size_t pitch = (n + 63) / 64 * 64;
    HB_TRY(ensure_buffers(*d, pitch * sizeof(double)));
    double* field = static_cast<double*>(d->buf[0]);
    cudaStream_t st = d->stream;
    // One round trip: the kernel validates the raw upload and snaps the ends
    // itself when the host-side end check (sync_solver.cpp:29-31) passes; when
    // it fails, upload_prepared reports the reference's errors in the
    // reference's order (a non-finite field before the end check).
    const bool ends_ok = bc_kind != HEAT_BC_DIRICHLET ||
                         (std::abs(u0[0] - c1) <= 1e-9 && std::abs(u0[n - 1] - c2) <= 1e-9);
    HB_CUDA(cudaMemsetAsync(d->flag, 0, 4 * sizeof(unsigned int), st));
    // pinned staging: [flags | input | final | trajectory rows]
    const size_t nb = n * sizeof(double);
    unsigned char* hs = host_stage(*d, 64 + 2 * nb + rows * nb);
    if (ends_ok) {
        const void* src = u0;
        if (hs) {
            std::memcpy(hs + 64, u0, nb);
            src = hs + 64;
        }
        HB_CUDA(cudaMemcpyAsync(field, src, nb, cudaMemcpyHostToDevice, st));
    } else {
        HB_TRY(upload_prepared(*d, u0, n, bc_kind, c1, c2, field));  // fails with the right error
    }
    if (want && d->snaps_bytes < rows * n * sizeof(double)) {
        if (d->snaps) cudaFree(d->snaps);
        d->snaps = nullptr;
        d->snaps_bytes = 0;
        HB_CUDA(cudaMalloc(&d->snaps, rows * n * sizeof(double)));
        d->snaps_bytes = rows * n * sizeof(double);
    }
    SmallArgs a{};
    a.field = field;
    a.n = int(n);
    a.r = r;
    a.c = 1.0 - 2.0 * r;  // core.hpp:108
    a.c1 = c1;
    a.c2 = c2;
    a.dirichlet = bc_kind == HEAT_BC_DIRICHLET;
    a.k_end = (long long)k_end;
    a.stride = want ? (long long)stride : 0;
    a.snaps = want ? static_cast<double*>(d->snaps) : nullptr;
    a.flag = d->flag;
    a.prep = 1;
    const int smem = int(n * sizeof(double));
    const int kMaxSmem = int(sync_small_max_points() * sizeof(double));
    // points per lane (measured, tools/probe_k3_pes.py): N <= 1024 8 (8 warps:
    // 113 ns/step at 1024; 12 gives 173), N <= 8192 12 (4096: 302 vs 355 at 8),
    // beyond 32.  HEAT_SMALL_V forces one for A/B.
    static const int forced_v = [] {
        const char* e = std::getenv("HEAT_SMALL_V");
        return e ? std::atoi(e) : 0;
    }();
    const int V = (forced_v == 8 && n <= 4096) || (forced_v == 12 && n <= 8192) ||
                          forced_v == 32
                      ? forced_v
                      : n <= 1024 ? 8 : n <= 8192 ? 12 : 32;
    if (V == 32 && n > 32 * 896) return fail(HEAT_ELOGIC, "K7: field too large");
    auto launch = [&](auto kern, int lanes) -> int {
        const int C = 32 * lanes - 2 * kSmallHalo;
        const int warps = int((n + C - 1) / C);
        int per_sm = 0;  // the limit is set once for the largest field this kernel takes
        HB_TRY(kernel_smem_config(reinterpret_cast<const void*>(kern), kMaxSmem,
                                  lanes <= 12 ? 1024 : 640, &per_sm));
        if (warps * 32 > (lanes <= 12 ? 1024 : 640)) return fail(HEAT_ELOGIC, "K7: too many warps");
        kern<<<1, warps * 32, smem, st>>>(a);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return HEAT_OK;
    };
    EventPair ev;
    if (kernel_ms) HB_TRY(ev.begin(st));
    if (V == 12)
        HB_TRY(launch(sync_small_kernel<12>, 12));
    else if (V == 8)
        HB_TRY(launch(sync_small_kernel<8>, 8));
    else
        HB_TRY(launch(sync_small_kernel<32>, 32));
    if (kernel_ms) HB_TRY(ev.end(st));
    // results and flags in one round trip
    size_t ns = 0;
    std::vector<size_t> ks;
    if (want) {
        // recorded steps: 0, stride, 2*stride, ..., and k_end when not a multiple
        ks.push_back(0);
        for (size_t kk = stride; kk <= k_end; kk += stride) ks.push_back(kk);
        if (k_end % stride) ks.push_back(k_end);
        ns = ks.size();
        const size_t copy = std::min(ns, max_snapshots);
        if (snapshots && copy)  // rows are contiguous on both sides: one copy
            HB_CUDA(cudaMemcpyAsync(hs ? static_cast<void*>(hs + 64 + 2 * nb) : snapshots, d->snaps,
                                    copy * nb, cudaMemcpyDeviceToHost, st));
    }
    if (final_out)
        HB_CUDA(cudaMemcpyAsync(hs ? static_cast<void*>(hs + 64 + nb) : final_out, field, nb,
                                cudaMemcpyDeviceToHost, st));
    unsigned int flags[4] = {0, 0, 0, 0};
    HB_CUDA(cudaMemcpyAsync(hs ? static_cast<void*>(hs) : flags, d->flag, sizeof flags,
                            cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (hs) {
        std::memcpy(flags, hs, sizeof flags);
        if (final_out) std::memcpy(final_out, hs + 64 + nb, nb);
        if (want && snapshots)
            std::memcpy(snapshots, hs + 64 + 2 * nb, std::min(ns, max_snapshots) * nb);
    }
    if (kernel_ms) HB_TRY(ev.elapsed(kernel_ms));
    if (flags[2]) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    if (steps_out)
        for (size_t j = 0; j < ns && j < max_snapshots; ++j) steps_out[j] = ks[j];
    if (n_snapshots) *n_snapshots = ns;
    return HEAT_OK;
}

}  // namespace hb
