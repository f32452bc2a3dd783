// sync_small.cu -- K7 and K7c: synchronous runs of small fields (N <= 16384,
// the paper's regime: cfg1 is N = 1024), the field resident in shared memory
// for the whole run.  K7 (below) is one CTA; K7c (further down) spreads the
// same windows over a thread-block cluster for N = 8m <= 8192 and is what
// sync_run uses there; exec_run(Barriered) keeps K7.
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
#include "small_cluster.cuh"

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


// ---- K7c: the same run spread over a thread-block cluster -----------------
// For N a multiple of 8 (<= 8192): windows of 32 x 8 points (128 exact + a
// 64-point halo per side), at most 4 warps per CTA so that each warp has an
// SM sub-partition to itself (the step is latency-bound: FP64 8 cycles,
// SHFL 30), the CTAs of one cluster each holding a full double-buffered copy
// of the field (small_cluster.cuh: st.async round writes, one mbarrier wait
// per round).  N and the window starts are multiples of 8, so a Dirichlet end
// is always a lane's first or last point: two selects inside the pipelined
// step re-pin it, and every warp runs the same pipelined code.  Trajectory
// rows are written from the exact lanes' registers at the recorded step, so
// records do not end rounds; with zero-copy I/O (mapped pinned staging) a
// call is one launch and one synchronize.
struct SmallClArgs {
    const double* in;  // [n] raw initial field (mapped host or device)
    double* field;     // [n] final field out
    int n;
    double r, c, c1, c2;
    int dirichlet;
    long long k_end;
    long long stride;  // 0: no trajectory
    double* snaps;     // [rows][n]
    unsigned int* flag;
    int ncta;
};

constexpr int kClMaxN = 8192;

template <int V, bool PIN>
__device__ __forceinline__ void cl_steps(double (&u)[V], double r, double c, double c1, double c2,
                                         bool pinF, bool pinL, int nsteps) {
    double pF = __dmul_rn(r, u[0]);
    double pLs = __dmul_rn(r, u[V - 1]);
    double pL = __shfl_up_sync(0xffffffffu, pLs, 1);
    double pR = __shfl_down_sync(0xffffffffu, pF, 1);
#pragma unroll 4
    for (int t = 0; t < nsteps; ++t) {
        const double p1 = __dmul_rn(r, u[1]);
        const double pVm2 = __dmul_rn(r, u[V - 2]);
        double nF = stencil_p(p1, __dmul_rn(c, u[0]), pL);
        double nL = stencil_p(pR, __dmul_rn(c, u[V - 1]), pVm2);
        if (PIN) {
            if (pinF) nF = c1;
            if (pinL) nL = c2;
        }
        const double pF2 = __dmul_rn(r, nF);
        const double pLs2 = __dmul_rn(r, nL);
        pL = __shfl_up_sync(0xffffffffu, pLs2, 1);
        pR = __shfl_down_sync(0xffffffffu, pF2, 1);
        double pm1 = pF, p0 = p1;
#pragma unroll
        for (int i = 1; i <= V - 2; ++i) {
            double pn;
            if (i + 1 == V - 1)
                pn = pLs;
            else if (i + 1 == V - 2)
                pn = pVm2;
            else
                pn = __dmul_rn(r, u[i + 1]);
            u[i] = stencil_p(pn, __dmul_rn(c, u[i]), pm1);
            pm1 = p0;
            p0 = pn;
        }
        u[0] = nF;
        u[V - 1] = nL;
        pF = pF2;
        pLs = pLs2;
    }
}

// V points per lane, 8 halo lanes per side: windows of 32V points (16V
// exact), rounds of 8V steps.  Each warp has its own sub-partition, so the
// step time is the per-warp time: fewer points per lane (more warps, more
// CTAs) is faster per step until the per-round cost dominates.
// HL halo lanes per side (H = HL*V points = steps per round): more halo
// lanes mean longer rounds (fewer exchanges per step) but fewer exact points
// per window, i.e. more windows, CTAs and SMs for the same field.
template <int V, bool CL, int HL = 8>
__global__ void __launch_bounds__(512, 1) sync_small_cl_kernel(const SmallClArgs a) {
    extern __shared__ double smem[];
    __shared__ __align__(8) unsigned long long sbar[2];
    constexpr int H = HL * V, C = 32 * V - 2 * H;
    const int N = a.n, Np = (N + 1) & ~1;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = CL ? int(small_ctarank()) : 0;
    const int gw = rank * int(blockDim.x >> 5) + w;
    double* su = smem;  // [2][Np]
    // the input may sit in mapped host memory: issue every load before any use
    bool bad_in = false;
    {
        const double2* in2 = reinterpret_cast<const double2*>(a.in);
        const int n2 = N / 2;
        for (int base = 0; base < n2; base += 8 * int(blockDim.x)) {
            double2 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = base + int(threadIdx.x) + j * int(blockDim.x);
                x[j] = i < n2 ? in2[i] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = base + int(threadIdx.x) + j * int(blockDim.x);
                if (i < n2) {
                    bad_in |= !isfinite(x[j].x) || !isfinite(x[j].y);
                    *reinterpret_cast<double2*>(&su[2 * i]) = x[j];
                }
            }
        }
    }
    // TemperatureField ctor (core.hpp:45-51) on the raw upload, then
    // prepare_initial's snap of the ends (the host checked |u - c| <= 1e-9)
    if (__syncthreads_or(bad_in)) {
        if (threadIdx.x == 0 && rank == 0) a.flag[2] = 1u;
        return;
    }
    if (a.dirichlet && threadIdx.x == 0) {
        su[0] = a.c1;
        su[N - 1] = a.c2;
    }
    __syncthreads();
    if (a.snaps && rank == 0)
        for (int i = threadIdx.x; i < N; i += blockDim.x) a.snaps[i] = su[i];
    const double r = a.r, c = a.c, c1 = a.c1, c2 = a.c2;
    const long long w0 = (long long)gw * C - H;
    const long long g0 = w0 + (long long)lane * V;
    const bool active = (long long)gw * C < N;  // warp-uniform
    const bool lreal = !a.dirichlet || (g0 >= 0 && g0 < N);
    const int wg0 = int(((g0 % N) + N) % N);
    const bool pinF = a.dirichlet && g0 == 0;
    const bool pinL = a.dirichlet && g0 + V - 1 == N - 1;
    const bool pinned = __any_sync(0xffffffffu, pinF || pinL);  // warp-uniform
    const bool lexact = active && lane >= H / V && lane < (H + C) / V && g0 < N;
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&sbar[0]));
    uint32_t incoming = 0;  // CL: bytes of halo groups the other CTAs send per round
    uint32_t send = 0;      // CL: CTAs that need my exact group (bit c)
    if (CL) {
        const HaloGeo geo{N, C, H, int(blockDim.x >> 5), a.ncta, !a.dirichlet};
        int cnt = 0;
        for (int base = 0; base < N; base += V * int(blockDim.x)) {
            const int g = base + V * int(threadIdx.x);
            cnt += __syncthreads_count(g < N && geo.needs(rank, g));
        }
        incoming = uint32_t(cnt * V * 8);
        if (lexact)
            for (int cc = 0; cc < a.ncta; ++cc)
                if (geo.needs(cc, int(g0))) send |= 1u << cc;
        if (threadIdx.x == 0) small_bars_init(bar0);
        small_cluster_sync();  // every CTA's barriers exist before the first st.async
    }
    int par = 0;
    uint32_t phases = 0;
    long long k = 0;
    long long next_rec = a.stride > 0 ? min(a.stride, a.k_end) : a.k_end + 1;
    double u[V];
    while (k < a.k_end) {
        const long long s = min((long long)H, a.k_end - k);
        const double* cu = su + par * Np;
        double* nu = su + (par ^ 1) * Np;
        const uint32_t nbar = bar0 + 8u * uint32_t(par ^ 1);
        if (CL && threadIdx.x == 0) small_bar_expect(nbar, incoming);
        if (active) {
#pragma unroll
            for (int i = 0; i < V; i += 2) {
                const double2 x = lreal ? *reinterpret_cast<const double2*>(&cu[wg0 + i])
                                        : make_double2(0.0, 0.0);
                u[i] = x.x;
                u[i + 1] = x.y;
            }
            for (int t0 = 0, len = 0; t0 < int(s); t0 += len) {
                const long long kb = k + t0;
                len = int(min(s - t0, next_rec - kb));
                if (pinned)
                    cl_steps<V, true>(u, r, c, c1, c2, pinF, pinL, len);
                else
                    cl_steps<V, false>(u, r, c, c1, c2, pinF, pinL, len);
                if (kb + len == next_rec) {  // a trajectory row: my exact chunk
                    if (lexact) {
                        double* row = a.snaps + ((next_rec + a.stride - 1) / a.stride) * N + g0;
#pragma unroll
                        for (int i = 0; i < V; i += 2)
                            *reinterpret_cast<double2*>(row + i) = make_double2(u[i], u[i + 1]);
                    }
                    next_rec = next_rec + a.stride > a.k_end && next_rec < a.k_end
                                   ? a.k_end
                                   : next_rec + a.stride;
                }
            }
            if (lexact) {
#pragma unroll
                for (int i = 0; i < V; i += 2)
                    *reinterpret_cast<double2*>(&nu[g0 + i]) = make_double2(u[i], u[i + 1]);
                if (CL) put_mask<V>(&nu[g0], u, nbar, send);
            }
        }
        __syncthreads();
        if (CL) {
            const int b = par ^ 1;
            mbar_wait_parity(nbar, (phases >> b) & 1u);
            phases ^= 1u << b;
        }
        par ^= 1;
        k += s;
    }
    // each CTA writes the points it owns (its copy of the rest is stale)
    su += par * Np;
    const int lo = rank * int(blockDim.x >> 5) * C, hi = min(lo + int(blockDim.x >> 5) * C, N);
    bool bad = false;
    for (int i = lo + int(threadIdx.x); i < hi; i += blockDim.x) {
        bad |= !isfinite(su[i]);
        a.field[i] = su[i];
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) a.flag[0] = 1u;
}

}  // namespace

size_t sync_small_max_points() { return 16384; }


// K7c host side: zero-copy I/O through the mapped pinned staging when it is
// large enough (device buffers and copies otherwise), one launch.
static int sync_run_small_cl(const double* u0, size_t n, double r, int bc_kind, double c1,
                             double c2, size_t k_end, size_t stride, double* final_out,
                             double* snapshots, size_t* steps_out, size_t max_snapshots,
                             size_t* n_snapshots, float* kernel_ms) {
    const bool want = snapshots != nullptr || steps_out != nullptr;
    const size_t rows = want ? 2 + k_end / stride : 0;
    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const size_t pitch = (n + 63) / 64 * 64;
    HB_TRY(ensure_buffers(*d, pitch * sizeof(double)));
    double* field = static_cast<double*>(d->buf[0]);
    cudaStream_t st = d->stream;
    const bool ends_ok = bc_kind != HEAT_BC_DIRICHLET ||
                         (std::abs(u0[0] - c1) <= 1e-9 && std::abs(u0[n - 1] - c2) <= 1e-9);
    if (!ends_ok) HB_TRY(upload_prepared(*d, u0, n, bc_kind, c1, c2, field));  // the right error
    const size_t nb = n * sizeof(double);
    const size_t o_rows = 64 + 2 * nb;  // [flags 64 | input | final | rows]
    unsigned char* hs = host_stage(*d, o_rows + rows * nb);
    SmallClArgs a{};
    if (hs) {
        std::memset(hs, 0, 64);
        std::memcpy(hs + 64, u0, nb);
        a.in = reinterpret_cast<const double*>(hs + 64);
        a.field = reinterpret_cast<double*>(hs + 64 + nb);
        a.flag = reinterpret_cast<unsigned int*>(hs);
        a.snaps = want ? reinterpret_cast<double*>(hs + o_rows) : nullptr;
    } else {
        HB_CUDA(cudaMemsetAsync(d->flag, 0, 4 * sizeof(unsigned int), st));
        HB_CUDA(cudaMemcpyAsync(field, u0, nb, cudaMemcpyHostToDevice, st));
        if (want && d->snaps_bytes < rows * nb) {
            if (d->snaps) cudaFree(d->snaps);
            d->snaps = nullptr;
            d->snaps_bytes = 0;
            HB_CUDA(cudaMalloc(&d->snaps, rows * nb));
            d->snaps_bytes = rows * nb;
        }
        a.in = field;
        a.field = field;
        a.flag = d->flag;
        a.snaps = want ? static_cast<double*>(d->snaps) : nullptr;
    }
    a.n = int(n);
    a.r = r;
    a.c = 1.0 - 2.0 * r;  // core.hpp:108
    a.c1 = c1;
    a.c2 = c2;
    a.dirichlet = bc_kind == HEAT_BC_DIRICHLET;
    a.k_end = (long long)k_end;
    a.stride = want ? (long long)stride : 0;
    // points per lane: HEAT_K7C_V in {4, 8} forces one (N must be a multiple)
    static const int forced_v = [] {
        const char* e = std::getenv("HEAT_K7C_V");
        return e ? std::atoi(e) : 0;
    }();
    const int V = forced_v == 4 || forced_v == 8 ? forced_v : 8;
    // halo lanes per side: HEAT_K7C_HL in {8, 10, 12} (V = 8 only)
    static const int forced_hl = [] {
        const char* e = std::getenv("HEAT_K7C_HL");
        return e ? std::atoi(e) : 0;
    }();
    // default: 10 halo lanes (80-step rounds) while that keeps one window per
    // SM sub-partition (<= 32 windows: N <= 3072; cfg1 50.3 ns/step against
    // 53.3 with 8, 50.9 with 12), else 8
    const int HL = V != 8                                      ? 8
                   : forced_hl == 8 || forced_hl == 10 || forced_hl == 12 ? forced_hl
                   : (n + 95) / 96 <= 32                        ? 10
                                                                : 8;
    if (n % size_t(V)) return fail(HEAT_ELOGIC, "K7c: N is not a multiple of the lane width");
    const int Cw = (32 - 2 * HL) * V;  // exact points per window
    const int warps = int((n + Cw - 1) / Cw);
    // more than four windows: a cluster, one warp per SM sub-partition
    static const bool no_cluster = std::getenv("HEAT_K7_NO_CLUSTER") != nullptr;
    const int ncta = no_cluster ? 1 : std::min(8, (warps + 3) / 4);
    const int wpc = (warps + ncta - 1) / ncta;
    if (wpc > 16) return fail(HEAT_ELOGIC, "K7c: too many warps per CTA");
    a.ncta = ncta;
    const int smem = int(2 * ((n + 1) & ~size_t(1)) * sizeof(double));
    auto pick = [&](auto k1, auto kc) {
        return ncta > 1 ? reinterpret_cast<const void*>(kc) : reinterpret_cast<const void*>(k1);
    };
    const void* fn =
        V == 4     ? pick(sync_small_cl_kernel<4, false>, sync_small_cl_kernel<4, true>)
        : HL == 10 ? pick(sync_small_cl_kernel<8, false, 10>, sync_small_cl_kernel<8, true, 10>)
        : HL == 12 ? pick(sync_small_cl_kernel<8, false, 12>, sync_small_cl_kernel<8, true, 12>)
                   : pick(sync_small_cl_kernel<8, false>, sync_small_cl_kernel<8, true>);
    int per_sm = 0;
    HB_TRY(kernel_smem_config(fn, int(2 * kClMaxN * sizeof(double)), wpc * 32, &per_sm));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(ncta));
    cfg.blockDim = dim3(unsigned(wpc * 32));
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(ncta);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ncta > 1 ? 1 : 0;
    void* params[] = {&a};
    EventPair ev;
    if (kernel_ms) HB_TRY(ev.begin(st));
    HB_CUDA(cudaLaunchKernelExC(&cfg, fn, params));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (kernel_ms) HB_TRY(ev.end(st));
    size_t ns = 0;
    std::vector<size_t> ks;
    if (want) {
        ks.push_back(0);
        for (size_t kk = stride; kk <= k_end; kk += stride) ks.push_back(kk);
        if (k_end % stride) ks.push_back(k_end);
        ns = ks.size();
    }
    const size_t copy = std::min(ns, max_snapshots);
    unsigned int flags[4] = {0, 0, 0, 0};
    if (hs) {
        HB_CUDA(cudaStreamSynchronize(st));
        std::memcpy(flags, hs, sizeof flags);
        if (final_out) std::memcpy(final_out, hs + 64 + nb, nb);
        if (snapshots && copy) std::memcpy(snapshots, hs + o_rows, copy * nb);
    } else {
        if (snapshots && copy)
            HB_CUDA(cudaMemcpyAsync(snapshots, d->snaps, copy * nb, cudaMemcpyDeviceToHost, st));
        if (final_out) HB_CUDA(cudaMemcpyAsync(final_out, field, nb, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaMemcpyAsync(flags, d->flag, sizeof flags, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
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

// Whole sync_run (or sync_step) of a small field on one CTA.  Validation as
// in sync_run_impl; trajectories are written by the kernel (0, stride,
// 2*stride, ..., k_end -- sync_solver.cpp:58-88).
int sync_run_small(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t k_end, size_t stride, double* final_out, double* snapshots,
                   size_t* steps_out, size_t max_snapshots, size_t* n_snapshots,
                   float* kernel_ms, bool one_cta) {
    if (stride == 0) stride = default_stride(n);
    // N a multiple of 8 up to 8192: K7c (cluster, zero-copy).  HEAT_NO_K7C=1: K7.
    static const bool no_k7c = std::getenv("HEAT_NO_K7C") != nullptr;
    // (one CTA holds at most 16 windows: HEAT_K7_NO_CLUSTER=1 beyond 2048 points takes K7)
    static const bool no_cluster = std::getenv("HEAT_K7_NO_CLUSTER") != nullptr;
    if (!no_k7c && !one_cta && n % 8 == 0 && n <= size_t(kClMaxN) && (!no_cluster || n <= 2048))
        return sync_run_small_cl(u0, n, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                                 steps_out, max_snapshots, n_snapshots, kernel_ms);
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
