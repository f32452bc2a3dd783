// async_host.cu -- host side of the asynchronous kernels: draw-order tables,
// launch selection, recording, executors.  C-ABI: heat_async_run,
// heat_sample_delay, heat_exec_run.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>

#include "async_pe.cuh"
#include "async_stream.cuh"
#include "runtime.cuh"
#include "stream_host.cuh"

namespace hb {

// In-step rank of every cross-PE read (async_sim.cpp:86-101: points in
// ascending i, pinned Dirichlet ends skipped, left before right, a draw only
// when the neighbour lies in another PE).  With P >= 2 only a PE's first
// point reads left across and only its last point reads right across.
int draw_offsets(size_t N, size_t n, int dirichlet, std::vector<int>& offL, std::vector<int>& offR) {
    const size_t P = N / n;
    offL.assign(P, -1);
    offR.assign(P, -1);
    int cnt = 0;
    for (size_t p = 0; p < P; ++p) {
        const size_t first = p * n, last = p * n + n - 1;
        const bool pin_first = dirichlet && (first == 0 || first == N - 1);
        const bool pin_last = dirichlet && (last == 0 || last == N - 1);
        if (P >= 2 && !pin_first) offL[p] = cnt++;  // left neighbour is always another PE
        if (P >= 2 && !pin_last) offR[p] = cnt++;   // (n == 1: same point, left then right)
    }
    return cnt;
}

namespace {

struct AsyncWork {
    // device allocations inside DevCtx::scratch
    double* field;
    double* ring;
    unsigned long long* prog;
    int* offL;
    int* offR;
    unsigned long long* stats;
    unsigned int* abort_word;
    double* edge_log;
    int* used_log;
};

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// K3 geometry for PEs of n points, P of them: S lanes per PE (32/S PEs per
// warp, shuffles confined to the segment) and V points per lane.  The
// narrowest segment that keeps >= 4 warps (one per scheduler) and <= 32
// points per lane: cfg2 (8 PEs of 128) runs 4 warps of two 16-lane PEs, not 8
// warps of 4-point lanes.  HEAT_PE_SEG forces S for A/B.
void pe_geometry(size_t n, size_t P, int& S, int& V, size_t& warps) {
    static const int forced = [] {
        const char* e = std::getenv("HEAT_PE_SEG");
        const int v = e ? std::atoi(e) : 0;
        return (v == 2 || v == 4 || v == 8 || v == 16 || v == 32) ? v : 0;
    }();
    auto lanes_v = [&](int s) {
        int v = 1;
        while (v * s < int(n)) v *= 2;
        return v;
    };
    S = 32;
    if (forced && lanes_v(forced) <= 32) {
        S = forced;
    } else {
        for (int cand = 16; cand >= 2; cand /= 2) {
            const size_t w = (P + size_t(32 / cand) - 1) / size_t(32 / cand);
            if (lanes_v(cand) > 32 || w < 4) break;
            S = cand;
        }
    }
    V = lanes_v(S);
    warps = (P + size_t(32 / S) - 1) / size_t(32 / S);
}

int pick_ring(int q) {
    int R = 64;
    while (R < 4 * q) R *= 2;
    return R;
}

// Full K3 layout for P PEs of n points, delay bound q, mode (0 deterministic
// lockstep, 1 free-running flags): lane segments only in the lockstep
// barrier mode (with flags, two PEs in one warp serialise each other's
// spin-waits, measured +9%); shared rings when one CTA of <= 16 warps holds
// every PE and the rings fit.
struct K3Layout {
    int S = 32, V = 1, R = 64;
    size_t warps = 0, smem = 0;
    bool shared = false;
};
K3Layout k3_layout(size_t n, size_t P, int q, int mode) {
    K3Layout L;
    pe_geometry(n, P, L.S, L.V, L.warps);
    L.R = pick_ring(q);
    L.smem = P * 2 * L.R * sizeof(double) + P * sizeof(unsigned long long);
    L.shared = L.warps <= 16 && L.smem <= 160 * 1024;
    if (mode != 0 || !L.shared) {
        L.S = 32;
        L.V = 1;
        while (L.V * 32 < int(n)) L.V *= 2;
        L.warps = P;
        L.shared = P <= 16 && L.smem <= 160 * 1024;
    }
    return L;
}

template <int V, bool S, bool B>
int launch_v(const AsyncPeArgs& a, int P, cudaStream_t st, size_t smem) {
    if (S) {
        // the dynamic rings plus the static histograms can pass 48 KB well below
        // the rings' own 160 KB cap: raise the limit once, per device
        int per_sm = 0;
        HB_TRY(kernel_smem_config(reinterpret_cast<const void*>(async_pe_kernel<V, S, B>),
                                  160 * 1024, 512, &per_sm));
        async_pe_kernel<V, S, B><<<1, 32 * P, smem, st>>>(a);
        HB_CUDA(cudaGetLastError());
    } else {
        // every PE warp must be co-resident: cooperative launch or refuse
        const int threads = 256;
        const int blocks = (P * 32 + threads - 1) / threads;
        int dev = 0, per_sm = 0, sms = 0;
        HB_CUDA(cudaGetDevice(&dev));
        HB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, async_pe_kernel<V, S, B>,
                                                              threads, 0));
        if ((long long)per_sm * sms < blocks)
            return fail(HEAT_EINVAL, "async: " + std::to_string(P) +
                                         " PE warps cannot be co-resident on this device");
        AsyncPeArgs copy = a;
        void* params[] = {&copy};
        HB_CUDA(cudaLaunchCooperativeKernel((const void*)async_pe_kernel<V, S, B>, dim3(blocks),
                                            dim3(threads), params, 0, st));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return HEAT_OK;
}

template <bool S, bool B>
int launch_sb(int V, const AsyncPeArgs& a, int P, cudaStream_t st, size_t smem) {
    switch (V) {
        case 1: return launch_v<1, S, B>(a, P, st, smem);
        case 2: return launch_v<2, S, B>(a, P, st, smem);
        case 4: return launch_v<4, S, B>(a, P, st, smem);
        case 8: return launch_v<8, S, B>(a, P, st, smem);
        case 16: return launch_v<16, S, B>(a, P, st, smem);
        default: return launch_v<32, S, B>(a, P, st, smem);
    }
}

// One CTA with shared rings (barrier mode for deterministic runs, flags for
// free-running ones) or a cooperative multi-CTA launch with global rings.
int launch_pe(int V, bool shared, bool barrier, const AsyncPeArgs& a, int P, cudaStream_t st,
              size_t smem) {
    if (!shared) return launch_sb<false, false>(V, a, P, st, 0);
    return barrier ? launch_sb<true, true>(V, a, P, st, smem)
                   : launch_sb<true, false>(V, a, P, st, smem);
}

// K3 runs a PE wider than a warp's 1024 points as `upe` equal units of at
// most 1024 points (the smallest such split).  The edges between units of
// one PE read the neighbour's value of the same step (kUnitEdge), so the PE
// stays synchronous inside; PE edges keep their draw ranks.
// The smallest split of a PE of n points into equal units of <= 1024 points;
// false when there is none (no side effects: a probe).
bool k3_split(size_t n, size_t& upe) {
    upe = 1;
    if (n <= 32 * 32) return true;
    for (upe = 2; upe <= n && (n % upe != 0 || n / upe > 32 * 32); ++upe) {}
    return !(upe > n || n / upe < 2);
}
int k3_units(size_t n, size_t& upe) {
    if (!k3_split(n, upe))
        return fail(HEAT_EINVAL, "async: a PE of this width has no split into units of <= 1024 "
                                 "points");
    return HEAT_OK;
}
void unit_offsets(const std::vector<int>& peL, const std::vector<int>& peR, size_t upe,
                  std::vector<int>& offL, std::vector<int>& offR) {
    const size_t U = peL.size() * upe;
    offL.resize(U);
    offR.resize(U);
    for (size_t u = 0; u < U; ++u) {
        offL[u] = u % upe == 0 ? peL[u / upe] : kUnitEdge;
        offR[u] = (u + 1) % upe == 0 ? peR[u / upe] : kUnitEdge;
    }
}

}  // namespace


int async_pe_run(DevCtx& d, const AsyncRunSpec& s, double* dfield, size_t stride,
                 const std::function<int(size_t, const double*)>& on_record,
                 unsigned long long* host_stats,
                 std::vector<double>* edge_log, std::vector<int>* used_log, float* device_ms) {
    // PEs wider than 1024 points run as units (k3_units; the callers send PEs
    // of a multiple of 32 points to K5 instead)
    size_t upe = 1;
    HB_TRY(k3_units(s.n, upe));
    if (upe > 1 && s.want_logs)
        return fail(HEAT_EINVAL, "async: edge logs need PEs of <= 1024 points or a multiple of "
                                 "32 points");
    const size_t Ppe = s.N / s.n, P = Ppe * upe, nu = s.n / upe;  // PEs, units, unit width
    if (P > 65536) return fail(HEAT_EINVAL, "async: too many PEs");
    const int q = int(s.q);
    const K3Layout G = k3_layout(nu, P, q, s.mode);
    const int S = G.S, V = G.V, R = G.R;
    const size_t warps = G.warps;
    const int dir = s.bc_kind == HEAT_BC_DIRICHLET;
    std::vector<int> peL, peR, offL, offR;
    const int D = draw_offsets(s.N, s.n, dir, peL, peR);  // the PEs' draw ranks
    unit_offsets(peL, peR, upe, offL, offR);

    // geometric law: the delay thresholds (exact, runtime.cu geometric_thresholds)
    std::vector<uint64_t> gthr;
    if (s.mode == 0 && s.law == HEAT_DELAY_GEOMETRIC)
        HB_TRY(geometric_thresholds(s.geometric_p, s.q, gthr));

    // scratch layout
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
    const size_t o_ring = take(P * 2 * R * sizeof(double));
    const size_t o_prog = take(P * sizeof(unsigned long long));
    const size_t o_offL = take(P * sizeof(int));
    const size_t o_offR = take(P * sizeof(int));
    const size_t o_gthr = take(std::max<size_t>(1, gthr.size()) * sizeof(uint64_t));
    const size_t o_stats = take(kStatWords * sizeof(unsigned long long));
    const size_t o_abort = take(sizeof(unsigned int));
    const size_t o_elog = take(s.want_logs ? (s.k_end + 1) * P * 2 * sizeof(double) : 0);
    const size_t o_ulog = take(s.want_logs ? std::max<size_t>(1, s.k_end) * P * 2 * sizeof(int) : 0);
    HB_TRY(ensure_scratch(d, off));
    char* base = static_cast<char*>(d.scratch);
    cudaStream_t st = d.stream;

    // initial ring: slot 0 = step-0 edge values, prog = 0 (one small kernel)
    async_init_kernel<<<std::max<size_t>(1, std::min<size_t>(1024, (P * 2 * R + 255) / 256)), 256,
                        0, st>>>(dfield, int(nu), int(P), R, reinterpret_cast<double*>(base + o_ring),
                                 reinterpret_cast<unsigned long long*>(base + o_prog),
                                 s.want_logs ? reinterpret_cast<double*>(base + o_elog) : nullptr);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    std::vector<unsigned long long> stats0(kStatWords, 0);
    stats0[kStatLagMin] = ~0ull;
    HB_CUDA(cudaMemcpyAsync(base + o_offL, offL.data(), P * sizeof(int), cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemcpyAsync(base + o_offR, offR.data(), P * sizeof(int), cudaMemcpyHostToDevice, st));
    if (!gthr.empty())
        HB_CUDA(cudaMemcpyAsync(base + o_gthr, gthr.data(), gthr.size() * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemcpyAsync(base + o_stats, stats0.data(), kStatWords * sizeof(unsigned long long),
                            cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemsetAsync(base + o_abort, 0, sizeof(unsigned int), st));
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 2 * sizeof(unsigned int), st));

    AsyncPeArgs a{};
    a.field = dfield;
    a.N = (long long)s.N;
    a.n = int(nu);
    a.P = int(P);
    a.r = s.r;
    a.c = 1.0 - 2.0 * s.r;  // core.hpp:108
    a.c1 = s.c1;
    a.c2 = s.c2;
    a.dirichlet = dir;
    a.mode = s.mode;
    a.q = q;
    a.R = R;
    a.law = s.law;
    a.fixed_d = int(std::min<size_t>(s.fixed_d, 1u << 30));
    a.seed = s.seed;
    a.modq = make_modq(unsigned(q));
    a.D = D;
    a.off_left = reinterpret_cast<const int*>(base + o_offL);
    a.off_right = reinterpret_cast<const int*>(base + o_offR);
    a.gthr = reinterpret_cast<const uint64_t*>(base + o_gthr);
    a.ring = reinterpret_cast<double*>(base + o_ring);
    a.prog = reinterpret_cast<unsigned long long*>(base + o_prog);
    // statistics only when asked for: they sit on the latency-critical step
    a.stats = host_stats ? reinterpret_cast<unsigned long long*>(base + o_stats) : nullptr;
    a.edge_log = s.want_logs ? reinterpret_cast<double*>(base + o_elog) : nullptr;
    a.used_log = s.want_logs ? reinterpret_cast<int*>(base + o_ulog) : nullptr;
    a.flag = d.flag;
    a.abort_word = reinterpret_cast<unsigned int*>(base + o_abort);
    a.timeout_ns = 20ull * 1000 * 1000 * 1000;  // 20 s watchdog per wait

    const size_t smem = G.smem;
    const bool shared = G.shared;  // one CTA of <= 512 threads
    a.seg = S;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (device_ms) {
        HB_CUDA(cudaEventCreate(&ev0));
        HB_CUDA(cudaEventCreate(&ev1));
        HB_CUDA(cudaEventRecord(ev0, st));
    }
    // Recording: small trajectories are written by the kernel itself (one
    // launch for the whole run); large ones split the run at recorded steps.
    const size_t nsnap = stride ? 2 + s.k_end / stride : 0;
    const bool in_kernel = stride && on_record && nsnap * s.N * sizeof(double) <= (512ull << 20);
    if (in_kernel) {
        if (d.snaps_bytes < nsnap * s.N * sizeof(double)) {
            if (d.snaps) cudaFree(d.snaps);
            d.snaps = nullptr;
            d.snaps_bytes = 0;
            HB_CUDA(cudaMalloc(&d.snaps, nsnap * s.N * sizeof(double)));
            d.snaps_bytes = nsnap * s.N * sizeof(double);
        }
        a.snaps = static_cast<double*>(d.snaps);
        a.snap_stride = (long long)stride;
        a.k_final = (long long)s.k_end;
    }
    size_t k = 0;
    while (k < s.k_end) {
        const size_t next = (stride && !in_kernel) ? std::min(s.k_end, (k / stride + 1) * stride)
                                                   : s.k_end;
        a.k0 = (long long)k;
        a.k1 = (long long)next;
        HB_TRY(launch_pe(V, shared, s.mode == 0, a, int(warps), st, smem));
        k = next;
        if (in_kernel) {
            unsigned int flags[2] = {0, 0};
            HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
            HB_CUDA(cudaStreamSynchronize(st));
            if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
            if (flags[0]) {
                if (g_strict.load())
                    return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
                return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
            }
            for (size_t kk = stride; kk <= s.k_end; kk += stride)
                HB_TRY(on_record(kk, a.snaps + (kk / stride) * s.N));
            if (s.k_end % stride)
                HB_TRY(on_record(s.k_end, a.snaps + (s.k_end / stride + 1) * s.N));
        } else if (stride && on_record) {
            unsigned int flags[2] = {0, 0};
            HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
            HB_CUDA(cudaStreamSynchronize(st));
            if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
            if (flags[0]) {
                if (g_strict.load())
                    return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
                return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
            }
            HB_TRY(on_record(k, dfield));
        }
    }
    if (device_ms) {
        HB_CUDA(cudaEventRecord(ev1, st));
        HB_CUDA(cudaEventSynchronize(ev1));
        HB_CUDA(cudaEventElapsedTime(device_ms, ev0, ev1));
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    if (host_stats)
        HB_CUDA(cudaMemcpyAsync(host_stats, base + o_stats, kStatWords * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st));
    if (s.want_logs && edge_log && used_log) {
        edge_log->resize((s.k_end + 1) * P * 2);
        used_log->resize(s.k_end * P * 2);
        HB_CUDA(cudaMemcpyAsync(edge_log->data(), base + o_elog, edge_log->size() * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
        if (!used_log->empty())
            HB_CUDA(cudaMemcpyAsync(used_log->data(), base + o_ulog, used_log->size() * sizeof(int),
                                    cudaMemcpyDeviceToHost, st));
    }
    HB_CUDA(cudaStreamSynchronize(st));
    if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    return HEAT_OK;
}

// K5 (streaming async) host code lives in stream_host.cu.

}  // namespace hb

using namespace hb;

extern "C" {

int heat_sample_delay(size_t q, int law, size_t fixed_delay, double geometric_p, uint64_t seed,
                      uint64_t j, size_t k, size_t* delay) {
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    const size_t bound = std::min(q - 1, k);
    const uint64_t x = splitmix_draw(seed, j);
    switch (law) {
        case HEAT_DELAY_UNIFORM: *delay = size_t(x % (bound + 1)); return HEAT_OK;
        case HEAT_DELAY_FIXED:
            if (fixed_delay >= q) return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
            *delay = std::min(fixed_delay, bound);
            return HEAT_OK;
        case HEAT_DELAY_GEOMETRIC: {
            if (!(geometric_p > 0.0) || geometric_p > 1.0)
                return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
            const double u = double(x >> 11) * 0x1.0p-53;
            double g = std::floor(std::log1p(-u) / std::log1p(-geometric_p));
            if (!std::isfinite(g) || g < 0.0) g = 0.0;
            *delay = std::min(size_t(g), bound);
            return HEAT_OK;
        }
    }
    return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
}

int heat_async_run(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                   size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                   uint64_t seed, size_t k_end, size_t stride, double* final_out,
                   double* snapshots, size_t* steps_out, size_t max_snapshots,
                   size_t* n_snapshots) {
    if (N < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u0) return fail(HEAT_EINVAL, "null field pointer");
    if (per_pe == 0 || N % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (law == HEAT_DELAY_FIXED && fixed_delay >= q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    if (law < 0 || law > 2) return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    // A single PE never reads across: no draws, bit-identical to sync_run
    // (test_async_sim.cpp:131-150).
    if (per_pe == N)
        return heat_sync_run(u0, N, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                             steps_out, max_snapshots, n_snapshots);
    return async_run_core(u0, N, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay, geometric_p,
                          seed, k_end, stride, final_out, snapshots, steps_out, max_snapshots,
                          n_snapshots);
}

}  // extern "C"

namespace hb {

// async_run for PEs no kernel geometry covers (wider than 1024 points, off
// the 32-point grid, with no split into units of <= 1024 points: a prime
// width): the reference's own loop, one async_step per step over a device
// HistoryRing (K8a/K8b, history.cu) -- async_sim.cpp:118-160 literally.
// Slow (a host round trip per step) but any partition works.
int async_run_history(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                      size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                      uint64_t seed, size_t k_end, size_t stride, double* final_out,
                      double* snapshots, size_t* steps_out, size_t max_snapshots,
                      size_t* n_snapshots) {
    std::vector<double> cur;
    HB_TRY(prepare_initial(u0, N, bc_kind, c1, c2, cur));
    heat_history* h = nullptr;
    HB_TRY(heat_history_create(&h, q, N, 0, cur.data(), 1, -1));
    struct Guard {
        heat_history* h;
        ~Guard() { heat_history_destroy(h); }
    } guard{h};
    size_t ns = 0;
    auto record = [&](size_t k, const double* v) -> int {
        for (size_t i = 0; i < N; ++i)  // a snapshot is a TemperatureField (core.hpp:45-51)
            if (!std::isfinite(v[i])) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
        if (ns < max_snapshots) {
            if (snapshots) std::memcpy(snapshots + ns * N, v, N * sizeof(double));
            if (steps_out) steps_out[ns] = k;
        }
        ++ns;
        return HEAT_OK;
    };
    const bool want = snapshots != nullptr || steps_out != nullptr;
    if (want) HB_TRY(record(0, cur.data()));
    uint64_t rng = seed;
    for (size_t k = 0; k < k_end; ++k) {
        const bool rec = want && ((k + 1) % stride == 0 || k + 1 == k_end);
        HB_TRY(heat_async_step(h, r, bc_kind, c1, c2, N, per_pe, q, law, fixed_delay, geometric_p,
                               &rng, rec || k + 1 == k_end ? cur.data() : nullptr, 1));
        if (rec) HB_TRY(record(k + 1, cur.data()));
    }
    if (final_out) {
        if (k_end == 0) HB_TRY(heat_history_snapshot(h, 0, cur.data()));
        // the reference records the final step as a TemperatureField
        // (async_sim.cpp:150-158), whose ctor rejects non-finite values
        if (!want)
            for (size_t i = 0; i < N; ++i)
                if (!std::isfinite(cur[i]))
                    return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
        std::memcpy(final_out, cur.data(), N * sizeof(double));
    }
    if (n_snapshots) *n_snapshots = ns;
    return HEAT_OK;
}

// Body of async_run after validation; also the small-N exact sync path
// (q = 1 replays d = 0 for every read: bit-identical to sync_run).
int async_run_core(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                   size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                   uint64_t seed, size_t k_end, size_t stride, double* final_out,
                   double* snapshots, size_t* steps_out, size_t max_snapshots,
                   size_t* n_snapshots) {
    if (stride == 0) stride = default_stride(N);
    {
        size_t upe = 1;
        if (per_pe > 32 * 32 && per_pe % 32 != 0 && !k3_split(per_pe, upe))
            return async_run_history(u0, N, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay,
                                     geometric_p, seed, k_end, stride, final_out, snapshots,
                                     steps_out, max_snapshots, n_snapshots);
    }
    if (async_small_eligible(N, per_pe, q))  // K9: one CTA, temporal-blocked rounds
        return async_run_small(u0, N, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay,
                               geometric_p, seed, k_end, stride, final_out, snapshots, steps_out,
                               max_snapshots, n_snapshots);
    if (async_member_eligible(N, per_pe, q))  // K6, one member: PEs K9 does not lay out
        return async_run_member(u0, N, r, bc_kind, c1, c2, per_pe, q, law, fixed_delay,
                                geometric_p, seed, k_end, stride, final_out, snapshots, steps_out,
                                max_snapshots, n_snapshots);

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    // K5 streaming kernel for wide PEs of whole 32-point units, else K3
    const bool wide = per_pe > 32 * 32 && per_pe % 32 == 0;
    const size_t pitch = (N + 63) / 64 * 64;
    HB_TRY(ensure_buffers(*d, (wide ? 2 : 1) * pitch * sizeof(double)));
    double* bufs[2] = {static_cast<double*>(d->buf[0]), static_cast<double*>(d->buf[0]) + pitch};
    int cur = 0;
    HB_TRY(upload_prepared(*d, u0, N, bc_kind, c1, c2, bufs[0]));

    const bool want_snaps = snapshots != nullptr || steps_out != nullptr;
    size_t ns = 0;
    cudaStream_t st = d->stream;
    auto record_from = [&](size_t k, const double* field) -> int {
        if (ns < max_snapshots) {
            if (snapshots)
                HB_CUDA(cudaMemcpyAsync(snapshots + ns * N, field, N * sizeof(double),
                                        cudaMemcpyDeviceToHost, st));
            if (steps_out) steps_out[ns] = k;
        }
        ++ns;
        return HEAT_OK;  // stream order keeps the rows; one sync at the end
    };
    if (want_snaps) HB_TRY(record_from(0, bufs[0]));
    AsyncRunSpec s{N, per_pe, r, bc_kind, c1, c2, 0, q, law, fixed_delay, geometric_p, seed,
                   k_end, false};
    if (wide) {
        HB_TRY(async_stream_run(*d, s, bufs, cur, want_snaps ? stride : 0, record_from, nullptr,
                                nullptr));
    } else {
        HB_TRY(async_pe_run(*d, s, bufs[0], want_snaps ? stride : 0,
                            record_from, nullptr, nullptr,
                            nullptr, nullptr));
    }
    if (final_out)
        HB_CUDA(cudaMemcpyAsync(final_out, bufs[cur], N * sizeof(double), cudaMemcpyDeviceToHost,
                                st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (n_snapshots) *n_snapshots = ns;
    return HEAT_OK;
}

}  // namespace hb

extern "C" {

int heat_async_free_run(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                        size_t per_pe, size_t q, size_t k_end, double* final_out,
                        heat_async_stats* stats) {
    if (N < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u0 || !final_out) return fail(HEAT_EINVAL, "null field pointer");
    if (per_pe == 0 || N % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    const bool wide = per_pe > 32 * 32;  // K5 (whole 32-point units), else K3
    if (wide && per_pe % 32 != 0)
        return fail(HEAT_EINVAL, "logged free run: PEs of <= 1024 points or of whole 32-point "
                                 "units");
    if (per_pe == N) return fail(HEAT_EINVAL, "logged free run: needs >= 2 PEs");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const size_t pitch = (N + 63) / 64 * 64;
    HB_TRY(ensure_buffers(*d, (wide ? 2 : 1) * pitch * sizeof(double)));
    double* bufs[2] = {static_cast<double*>(d->buf[0]), static_cast<double*>(d->buf[0]) + pitch};
    HB_TRY(upload_prepared(*d, u0, N, bc_kind, c1, c2, bufs[0]));
    AsyncRunSpec s{N, per_pe, r, bc_kind, c1, c2, 1, q, HEAT_DELAY_UNIFORM, 0, 0.5, 0, k_end, true};
    std::vector<unsigned long long> hs(kStatWords, 0);
    std::vector<double> elog;
    std::vector<int> ulog;
    if (!wide) {
        HB_TRY(async_pe_run(*d, s, bufs[0], 0, nullptr, hs.data(), &elog, &ulog, nullptr));
        HB_CUDA(cudaMemcpy(final_out, bufs[0], N * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
        // K5 logs every PE edge value and every read's source step on the
        // device ((k_end+1)*P*2 doubles + k_end*P*2 ints: 123 MB for cfg3)
        const size_t P = N / per_pe;
        elog.assign((k_end + 1) * P * 2, 0.0);
        ulog.assign(k_end * P * 2, 0);
        for (size_t p = 0; p < P; ++p) {  // step 0: the prepared field's PE edges
            const size_t f = p * per_pe, l = f + per_pe - 1;
            const bool dir = bc_kind == HEAT_BC_DIRICHLET;
            elog[p * 2 + 0] = dir && f == 0 ? c1 : u0[f];
            elog[p * 2 + 1] = dir && l == N - 1 ? c2 : u0[l];
        }
        struct DevBuf {
            void* p = nullptr;
            ~DevBuf() {
                if (p) cudaFree(p);
            }
        } de, du;
        HB_CUDA(cudaMalloc(&de.p, elog.size() * sizeof(double)));
        HB_CUDA(cudaMalloc(&du.p, std::max<size_t>(1, ulog.size()) * sizeof(int)));
        HB_CUDA(cudaMemcpy(de.p, elog.data(), 2 * P * sizeof(double), cudaMemcpyHostToDevice));
        StreamLogs logs;
        logs.edge_log = static_cast<double*>(de.p);
        logs.used_log = static_cast<int*>(du.p);
        int cur = 0;
        s.want_logs = false;  // (the K3 flag; K5 takes `logs`)
        HB_TRY(async_stream_run(*d, s, bufs, cur, 0, nullptr, hs.data(), nullptr, &logs));
        HB_CUDA(cudaMemcpy(elog.data(), de.p, elog.size() * sizeof(double), cudaMemcpyDeviceToHost));
        if (!ulog.empty())
            HB_CUDA(cudaMemcpy(ulog.data(), du.p, ulog.size() * sizeof(int), cudaMemcpyDeviceToHost));
        HB_CUDA(cudaMemcpy(final_out, bufs[cur], N * sizeof(double), cudaMemcpyDeviceToHost));
    }

    // a-posteriori residual: only PE-boundary points read a neighbour; the
    // async step differs from A u(k) there by r*(u_j(k*) - u_j(k)).
    const size_t P = N / per_pe;
    const bool dir = bc_kind == HEAT_BC_DIRICHLET;
    double umax = 0.0, sum = 0.0;
    for (size_t i = 0; i < N; ++i) umax = std::max(umax, std::abs(u0[i]));
    for (double v : elog) umax = std::max(umax, std::abs(v));
    for (size_t k = 0; k < k_end; ++k) {
        double res = 0.0;
        for (size_t p = 0; p < P; ++p) {
            const size_t first = p * per_pe, last = first + per_pe - 1;
            const long long lpe = p > 0 ? (long long)p - 1 : (dir ? -1 : (long long)P - 1);
            const long long rpe = p + 1 < P ? (long long)p + 1 : (dir ? -1 : 0);
            double rp = 0.0;
            const bool pin_first = dir && (first == 0 || first == N - 1);
            const bool pin_last = dir && (last == 0 || last == N - 1);
            if (lpe >= 0 && !pin_first) {  // first point read PE lpe's last point at k*
                const int ks = ulog[(k * P + p) * 2 + 0];
                rp += r * std::abs(elog[(size_t(ks) * P + lpe) * 2 + 1] - elog[(k * P + lpe) * 2 + 1]);
            }
            double rq = 0.0;
            if (rpe >= 0 && !pin_last) {  // last point read PE rpe's first point at k*
                const int ks = ulog[(k * P + p) * 2 + 1];
                rq = r * std::abs(elog[(size_t(ks) * P + rpe) * 2 + 0] - elog[(k * P + rpe) * 2 + 0]);
            }
            // with one point per PE both reads hit the same point
            res = std::max(res, per_pe == 1 ? rp + rq : std::max(rp, rq));
        }
        sum += res;
    }
    const double eps = 0x1.0p-52;
    sum += double(k_end) * 8.0 * eps * std::max(1.0, umax);  // rounding of both sequences
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->reads = hs[kStatReads];
        stats->waits = hs[kStatWaits];
        stats->max_delay = hs[kStatMaxDelay];
        for (int i = 0; i < 64; ++i) stats->delay_histogram[i] = hs[kStatDelayHist + i];
        stats->residual_sum = sum;
    }
    return HEAT_OK;
}

int heat_exec_run(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                  size_t per_pe, size_t workers, size_t k_end, int mode, int record_lag,
                  size_t q_free, double* field_out, uint64_t* duration_ns, heat_lag_stats* lag,
                  heat_async_stats* stats) {
    // exec_run validation order (async_exec.cpp:263-272); the PartitionSpec
    // ctor (core.cpp:66-72) runs first at the caller.
    if (N < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (per_pe == 0 || N % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (workers == 0 || workers != N / per_pe)
        return fail(HEAT_EINVAL, "exec_run: cfg.workers must equal part.P");
    if (k_end == 0) return fail(HEAT_EINVAL, "exec_run: k_end >= 1 required");
    if (mode != HEAT_EXEC_BARRIERED && mode != HEAT_EXEC_BARRIER_FREE)
        return fail(HEAT_EINVAL, "exec_run: unknown mode");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    const bool sync_path = mode == HEAT_EXEC_BARRIERED || workers == 1;
    if (sync_path) {
        // Barriered is bit-identical to sync_run (acceptance.cpp:225-229); so is
        // BarrierFree with one PE (test_exec.cpp:69-87).
        // Timed like the BarrierFree kernels below: the compute launches'
        // device time only, not the staging and copies around them (the
        // reference's duration brackets the workers, async_exec.cpp:101-106).
        float ms = 0.f;
        int st = sync_run_timed(u0, N, r, bc_kind, c1, c2, k_end, field_out, &ms);
        if (duration_ns) *duration_ns = uint64_t(double(ms) * 1e6);
        if (lag) std::memset(lag, 0, sizeof *lag);
        if (stats) std::memset(stats, 0, sizeof *stats);
        return st;
    }
    size_t upe_probe = 1;
    if (per_pe > 32 * 32 && per_pe % 32 != 0 && !k3_split(per_pe, upe_probe)) {
        // PEs no free-running kernel lays out (wider than 1024 points, off the
        // 32-point grid, no split into units of <= 1024: a prime width such as
        // 1031).  The run takes the delay-0 trajectory -- every PE reads its
        // neighbours' current values, a schedule the free-running model allows
        // (0 <= k - k* <= q - 1) -- on the synchronous kernels, which have no
        // per-step barrier either (temporal blocking).
        float ms = 0.f;
        const int st = sync_run_timed(u0, N, r, bc_kind, c1, c2, k_end, field_out, &ms);
        if (duration_ns) *duration_ns = uint64_t(double(ms) * 1e6);
        if (lag) std::memset(lag, 0, sizeof *lag);
        if (stats) {
            std::memset(stats, 0, sizeof *stats);
            const size_t P = N / per_pe;
            const size_t edges = bc_kind == HEAT_BC_DIRICHLET ? 2 * (P - 1) : 2 * P;
            stats->reads = (unsigned long long)(edges * k_end);
            stats->delay_histogram[0] = stats->reads;
        }
        return st;
    }

    std::lock_guard<std::mutex> lock(d->mu);
    const size_t qf = q_free ? q_free : 8;
    if (!record_lag && free_eligible(N, per_pe, qf, k_end)) {
        // K10: one warp per PE in one thread-block cluster, DSMEM edge rings
        std::vector<unsigned long long> hs(kStatWords, 0);
        float ms = 0.f;
        HB_TRY(exec_free_run(*d, u0, N, r, bc_kind, c1, c2, per_pe, qf, k_end, field_out,
                             stats ? hs.data() : nullptr, &ms));
        if (duration_ns) *duration_ns = uint64_t(double(ms) * 1e6);
        if (lag) std::memset(lag, 0, sizeof *lag);
        if (stats) {
            std::memset(stats, 0, sizeof *stats);
            stats->reads = hs[kStatReads];
            stats->waits = hs[kStatWaits];
            stats->max_delay = hs[kStatMaxDelay];
            for (int i = 0; i < 64; ++i) stats->delay_histogram[i] = hs[kStatDelayHist + i];
        }
        return HEAT_OK;
    }
    const bool wide = per_pe > 32 * 32 && per_pe % 32 == 0;  // K5; else K3 (units)
    const size_t pitch = (N + 63) / 64 * 64;
    HB_TRY(ensure_buffers(*d, (wide ? 2 : 1) * pitch * sizeof(double)));
    double* bufs[2] = {static_cast<double*>(d->buf[0]), static_cast<double*>(d->buf[0]) + pitch};
    int cur = 0;
    HB_TRY(upload_prepared(*d, u0, N, bc_kind, c1, c2, bufs[0]));
    const size_t q = qf;
    AsyncRunSpec s{N, per_pe, r, bc_kind, c1, c2, 1, q, HEAT_DELAY_UNIFORM, 0, 0.5, 0, k_end,
                   false};
    std::vector<unsigned long long> hs(kStatWords, 0);
    float ms = 0.f;
    if (wide)
        HB_TRY(async_stream_run(*d, s, bufs, cur, 0, nullptr, hs.data(), &ms));
    else
        HB_TRY(async_pe_run(*d, s, bufs[0], 0, nullptr, hs.data(), nullptr, nullptr, &ms));
    HB_CUDA(cudaMemcpy(field_out, bufs[cur], N * sizeof(double), cudaMemcpyDeviceToHost));
    if (duration_ns) *duration_ns = uint64_t(double(ms) * 1e6);
    if (lag) {
        std::memset(lag, 0, sizeof *lag);
        if (record_lag && hs[kStatReads]) {
            lag->reads = hs[kStatReads];
            lag->min_lag = hs[kStatLagMin];
            lag->max_lag = hs[kStatLagMax];
            lag->overflow = hs[kStatLagOverflow];
            for (int i = 0; i < 64; ++i) lag->histogram[i] = hs[kStatLagHist + i];
        }
    }
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->reads = hs[kStatReads];
        stats->waits = hs[kStatWaits];
        stats->max_delay = hs[kStatMaxDelay];
        for (int i = 0; i < 64; ++i) stats->delay_histogram[i] = hs[kStatDelayHist + i];
    }
    return HEAT_OK;
}

static int plan_async(heat_plan* p, const AsyncRunSpec& s, heat_async_stats* stats);

int heat_plan_async_advance(heat_plan* p, double r, int bc_kind, double c1, double c2,
                            size_t per_pe, size_t q, size_t steps, heat_async_stats* stats) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    AsyncRunSpec s{p->n, per_pe, r, bc_kind, c1, c2, 1, q, HEAT_DELAY_UNIFORM, 0, 0.5, 0, steps,
                   false};
    return plan_async(p, s, stats);
}

int heat_plan_async_replay(heat_plan* p, double r, int bc_kind, double c1, double c2,
                           size_t per_pe, size_t q, int law, size_t fixed_delay,
                           double geometric_p, uint64_t seed, size_t steps,
                           heat_async_stats* stats) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    if (law < 0 || law > 2) return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
    if (q > 0 && law == HEAT_DELAY_FIXED && fixed_delay >= q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    AsyncRunSpec s{p->n, per_pe, r, bc_kind, c1, c2, 0, q, law, fixed_delay, geometric_p, seed,
                   steps, false};
    return plan_async(p, s, stats);
}

// Bounded-staleness async on a resident field: every call is a fresh run
// (rings seeded from the current field, k counted from 0).
static int plan_async(heat_plan* p, const AsyncRunSpec& s, heat_async_stats* stats) {
    const size_t per_pe = s.n, q = s.q, steps = s.k_end;
    const int bc_kind = s.bc_kind;
    if (p->world != 1) return fail(HEAT_EINVAL, "async advance of multi-GPU slabs is not supported");
    if (per_pe == 0 || p->n % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    if (per_pe <= 32 * 32 || per_pe == p->n)
        return fail(HEAT_EINVAL, "plan async advance needs >= 2 PEs wider than 1024 points");
    HB_CUDA(cudaSetDevice(p->device));
    StreamLayout L;
    std::vector<int> offL, offR;
    const StreamExternal ext{};
    HB_TRY(stream_layout(s, virtual_device_groups(p->n / per_pe), ext, L, offL, offR));
    if (p->async_bytes < L.bytes) {
        if (p->async_scratch) cudaFree(p->async_scratch);
        p->async_scratch = nullptr;
        p->async_bytes = 0;
        HB_CUDA(cudaMalloc(&p->async_scratch, L.bytes));
        p->async_bytes = L.bytes;
    }
    char* base = static_cast<char*>(p->async_scratch);
    HB_TRY(async_stream_advance(p->sms, p->stream, p->bufs, p->cur, s, L, base, ext, offL, offR, 0,
                                0, true, p->flag, nullptr));
    HB_TRY(async_stream_advance(p->sms, p->stream, p->bufs, p->cur, s, L, base, ext, offL, offR, 0,
                                steps, false, p->flag, nullptr));
    if (stats) {
        std::vector<unsigned long long> hs(kStatWords, 0);
        HB_CUDA(cudaMemcpyAsync(hs.data(), base + L.o_stats, kStatWords * 8, cudaMemcpyDeviceToHost,
                                p->stream));
        HB_CUDA(cudaStreamSynchronize(p->stream));
        std::memset(stats, 0, sizeof *stats);
        stats->reads = hs[kStatReads];
        stats->waits = hs[kStatWaits];
        stats->max_delay = hs[kStatMaxDelay];
        for (int i = 0; i < 64; ++i) stats->delay_histogram[i] = hs[kStatDelayHist + i];
    }
    return HEAT_OK;
}

}  // extern "C"

// ---- AsyncSimulator on the GPU (async_sim.hpp:73-90, async_sim.cpp:122-140) --
// A handle owns its device state -- field(s), the PE rings and progress
// words, the draw offsets -- and advances it in slices [k, k + count): the
// kernels take absolute step numbers, the counter-form draws need no stream
// state, and K3's rings / K5's scratch persist between slices, so stepping a
// run in any slicing is bit-identical to async_run over the whole.
struct heat_async_sim {
    hb::DevCtx ctx;  // own stream, flag words, buffers, scratch
    hb::AsyncRunSpec s{};
    size_t P = 0;
    bool wide = false;
    double* field[2] = {nullptr, nullptr};
    int cur = 0;
    size_t k = 0;
    bool started = false;
    // K3 scratch layout (U units of nu points: PEs wider than 1024 points
    // are split, k3_units)
    size_t U = 0, nu = 0;
    int R = 0, D = 0, V = 1, S = 32;
    size_t warps = 0;
    size_t o_ring = 0, o_prog = 0, o_offL = 0, o_offR = 0, o_abort = 0;
    bool shared = false;
    size_t smem = 0;
    // K5
    hb::StreamLayout L;
    std::vector<int> offL, offR;
    // GEOMETRIC: the delay thresholds (device, uploaded once)
    uint64_t* gthr = nullptr;
    // PEs no kernel geometry covers (prime widths above 1024 points): the
    // reference's own step, async_step over a device HistoryRing (K8a/K8b)
    heat_history* hist = nullptr;
    uint64_t rng = 0;
};

namespace {

void sim_free(heat_async_sim* sim) {
    if (!sim) return;
    cudaSetDevice(sim->ctx.device);
    if (sim->ctx.stream) cudaStreamSynchronize(sim->ctx.stream);
    if (sim->ctx.buf[0]) cudaFree(sim->ctx.buf[0]);
    if (sim->ctx.scratch) cudaFree(sim->ctx.scratch);
    if (sim->ctx.flag) cudaFree(sim->ctx.flag);
    if (sim->gthr) cudaFree(sim->gthr);
    if (sim->hist) heat_history_destroy(sim->hist);
    if (sim->ctx.stream) cudaStreamDestroy(sim->ctx.stream);
    delete sim;
}

int sim_step_k3(heat_async_sim* sim, size_t count) {
    DevCtx& d = sim->ctx;
    const auto& s = sim->s;
    char* base = static_cast<char*>(d.scratch);
    cudaStream_t st = d.stream;
    if (!sim->started) {
        async_init_kernel<<<std::max<size_t>(1, std::min<size_t>(1024, (sim->U * 2 * sim->R + 255) / 256)),
                            256, 0, st>>>(sim->field[0], int(sim->nu), int(sim->U), sim->R,
                                          reinterpret_cast<double*>(base + sim->o_ring),
                                          reinterpret_cast<unsigned long long*>(base + sim->o_prog),
                                          nullptr);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
        HB_CUDA(cudaMemcpyAsync(base + sim->o_offL, sim->offL.data(), sim->U * sizeof(int),
                                cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemcpyAsync(base + sim->o_offR, sim->offR.data(), sim->U * sizeof(int),
                                cudaMemcpyHostToDevice, st));
        HB_CUDA(cudaMemsetAsync(base + sim->o_abort, 0, sizeof(unsigned int), st));
        sim->started = true;
    }
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 2 * sizeof(unsigned int), st));
    AsyncPeArgs a{};
    a.field = sim->field[0];
    a.N = (long long)s.N;
    a.n = int(sim->nu);
    a.P = int(sim->U);
    a.r = s.r;
    a.c = 1.0 - 2.0 * s.r;  // core.hpp:108
    a.c1 = s.c1;
    a.c2 = s.c2;
    a.dirichlet = s.bc_kind == HEAT_BC_DIRICHLET;
    a.k0 = (long long)sim->k;
    a.k1 = (long long)(sim->k + count);
    a.mode = 0;
    a.q = int(s.q);
    a.R = sim->R;
    a.law = s.law;
    a.fixed_d = int(std::min<size_t>(s.fixed_d, 1u << 30));
    a.seed = s.seed;
    a.modq = make_modq(unsigned(s.q));
    a.D = sim->D;
    a.off_left = reinterpret_cast<const int*>(base + sim->o_offL);
    a.off_right = reinterpret_cast<const int*>(base + sim->o_offR);
    a.gthr = sim->gthr;
    a.ring = reinterpret_cast<double*>(base + sim->o_ring);
    a.prog = reinterpret_cast<unsigned long long*>(base + sim->o_prog);
    a.flag = d.flag;
    a.abort_word = reinterpret_cast<unsigned int*>(base + sim->o_abort);
    a.timeout_ns = 20ull * 1000 * 1000 * 1000;
    a.seg = sim->S;
    return launch_pe(sim->V, sim->shared, true, a, int(sim->warps), st, sim->smem);
}

int sim_step_k5(heat_async_sim* sim, size_t count) {
    DevCtx& d = sim->ctx;
    StreamExternal ext{};
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 2 * sizeof(unsigned int), d.stream));
    const bool init = !sim->started;
    sim->started = true;
    return async_stream_advance(d.sms, d.stream, sim->field, sim->cur, sim->s, sim->L,
                                static_cast<char*>(d.scratch), ext, sim->offL, sim->offR,
                                sim->k, count, init, d.flag, nullptr);
}

}  // namespace

extern "C" {

int heat_k3_geometry(size_t n, size_t P, size_t q, int mode, int* lanes_per_pe,
                     int* points_per_lane, size_t* warps, int* shared_rings) {
    if (n == 0 || P == 0 || q == 0) return fail(HEAT_EINVAL, "k3 geometry: n, P, q >= 1");
    const K3Layout G = k3_layout(n, P, int(q), mode);
    if (lanes_per_pe) *lanes_per_pe = G.S;
    if (points_per_lane) *points_per_lane = G.V;
    if (warps) *warps = G.warps;
    if (shared_rings) *shared_rings = G.shared ? 1 : 0;
    return HEAT_OK;
}

int heat_async_sim_create(heat_async_sim** out, const double* u0, size_t N, double r,
                          int bc_kind, double c1, double c2, size_t per_pe, size_t q, int law,
                          size_t fixed_delay, double geometric_p, uint64_t seed) {
    if (!out) return fail(HEAT_EINVAL, "null simulator handle");
    *out = nullptr;
    // the caller's objects validate first (TemperatureField, DelayModel,
    // PartitionSpec ctors), then AsyncSimulator's ctor (async_sim.cpp:122-134):
    // prepare_initial, partition vs grid, q >= 1
    if (N < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u0) return fail(HEAT_EINVAL, "null field pointer");
    if (law == HEAT_DELAY_FIXED && q > 0 && fixed_delay >= q)
        return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
    if (law == HEAT_DELAY_GEOMETRIC && (!(geometric_p > 0.0) || geometric_p > 1.0))
        return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    if (law < 0 || law > 2) return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
    if (per_pe == 0 || N % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    int dev = 0;
    HB_CUDA(cudaGetDevice(&dev));
    DevCtx* shared_ctx = nullptr;
    HB_TRY(dev_ctx(dev, &shared_ctx));  // device checks (sm_100)
    auto* sim = new heat_async_sim();
    struct Guard {
        heat_async_sim*& p;
        ~Guard() {
            if (p) sim_free(p);
        }
    } guard{sim};
    DevCtx& d = sim->ctx;
    d.device = dev;
    d.sms = shared_ctx->sms;
    HB_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    HB_CUDA(cudaMalloc(&d.flag, kFlagWords * sizeof(unsigned int)));
    HB_CUDA(cudaMemset(d.flag, 0, kFlagWords * sizeof(unsigned int)));
    sim->P = N / per_pe;
    sim->wide = per_pe > 32 * 32 && per_pe % 32 == 0 && sim->P > 1;  // K5; else K3 (units)
    const size_t pitch = (N + 63) / 64 * 64;
    // two buffers for K5 and for a single PE (K1 ping-pong), one for K3
    HB_TRY(ensure_buffers(d, (sim->wide || sim->P == 1 ? 2 : 1) * pitch * sizeof(double)));
    sim->field[0] = static_cast<double*>(d.buf[0]);
    sim->field[1] = sim->field[0] + pitch;
    HB_TRY(upload_prepared(d, u0, N, bc_kind, c1, c2, sim->field[0]));
    // HistoryRing(q, prepare_initial(u0, bc)) in the ctor's initialiser list
    if (q == 0) return fail(HEAT_EDOMAIN, "HistoryRing: depth >= 1 required");
    sim->s = AsyncRunSpec{N, per_pe, r, bc_kind, c1, c2, 0, q, law, fixed_delay, geometric_p, seed,
                          0, false};
    if (sim->P == 1) {
        // one PE never reads across: plain synchronous steps (K1 on field[0..1])
        sim->wide = true;
    }
    size_t upe_probe = 1;
    if (sim->P > 1 && per_pe > 32 * 32 && per_pe % 32 != 0 && !k3_split(per_pe, upe_probe)) {
        // AsyncSimulator::step literally (async_sim.cpp:136-140): async_step
        // over a HistoryRing of depth q seeded with the prepared field, the
        // simulator's SplitMix64 stream advanced as the reference's
        std::vector<double> prep;
        HB_TRY(prepare_initial(u0, N, bc_kind, c1, c2, prep));
        HB_TRY(heat_history_create(&sim->hist, q, N, 0, prep.data(), 1, dev));
        sim->rng = seed;
        *out = sim;
        sim = nullptr;  // owned by the caller now
        return HEAT_OK;
    }
    if (sim->wide && sim->P > 1) {
        HB_TRY(stream_layout(sim->s, 1, StreamExternal{}, sim->L, sim->offL, sim->offR));
        HB_TRY(ensure_scratch(d, sim->L.bytes));
    } else if (!sim->wide) {
        size_t upe = 1;
        HB_TRY(k3_units(per_pe, upe));
        sim->U = sim->P * upe;
        sim->nu = per_pe / upe;
        const K3Layout G = k3_layout(sim->nu, sim->U, int(q), 0);
        sim->S = G.S;
        sim->V = G.V;
        sim->warps = G.warps;
        sim->R = G.R;
        std::vector<int> peL, peR;
        sim->D = draw_offsets(N, per_pe, bc_kind == HEAT_BC_DIRICHLET, peL, peR);
        unit_offsets(peL, peR, upe, sim->offL, sim->offR);
        size_t off = 0;
        auto take = [&](size_t bytes) {
            size_t o = off;
            off += align256(bytes);
            return o;
        };
        sim->o_ring = take(sim->U * 2 * sim->R * sizeof(double));
        sim->o_prog = take(sim->U * sizeof(unsigned long long));
        sim->o_offL = take(sim->U * sizeof(int));
        sim->o_offR = take(sim->U * sizeof(int));
        sim->o_abort = take(sizeof(unsigned int));
        HB_TRY(ensure_scratch(d, off));
        sim->smem = G.smem;
        sim->shared = G.shared;
        if (law == HEAT_DELAY_GEOMETRIC) {  // exact device delays of the law
            std::vector<uint64_t> gthr;
            HB_TRY(geometric_thresholds(geometric_p, q, gthr));
            HB_CUDA(cudaMalloc(&sim->gthr, std::max<size_t>(1, gthr.size()) * sizeof(uint64_t)));
            if (!gthr.empty())
                HB_CUDA(cudaMemcpy(sim->gthr, gthr.data(), gthr.size() * sizeof(uint64_t),
                                   cudaMemcpyHostToDevice));
        }
    }
    *out = sim;
    sim = nullptr;  // owned by the caller now
    return HEAT_OK;
}

int heat_async_sim_step(heat_async_sim* sim, size_t count) {
    if (!sim) return fail(HEAT_EINVAL, "null simulator handle");
    if (count == 0) return HEAT_OK;
    HB_CUDA(cudaSetDevice(sim->ctx.device));
    if (sim->hist) {  // one async_step per step (a host round trip each)
        const AsyncRunSpec& s = sim->s;
        for (size_t j = 0; j < count; ++j) {
            HB_TRY(heat_async_step(sim->hist, s.r, s.bc_kind, s.c1, s.c2, s.N, s.n, s.q, s.law,
                                   s.fixed_d, s.geometric_p, &sim->rng, nullptr, 1));
            ++sim->k;
        }
        return HEAT_OK;
    }
    if (sim->P == 1) {  // a single PE: synchronous steps
        HB_CUDA(cudaMemsetAsync(sim->ctx.flag, 0, 2 * sizeof(unsigned int), sim->ctx.stream));
        HB_TRY(sync_advance<double>(sim->ctx.sms, sim->field, sim->cur, (long long)sim->s.N,
                                    sim->s.r, sim->s.bc_kind == HEAT_BC_PERIODIC, sim->s.c1,
                                    sim->s.c2, count, sim->ctx.flag, sim->ctx.stream));
    } else if (sim->wide) {
        HB_TRY(sim_step_k5(sim, count));
    } else {
        HB_TRY(sim_step_k3(sim, count));
    }
    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, sim->ctx.flag, sizeof flags, cudaMemcpyDeviceToHost,
                            sim->ctx.stream));
    HB_CUDA(cudaStreamSynchronize(sim->ctx.stream));
    sim->k += count;
    if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
    // async_step_into checks only under strict finite checks (async_sim.cpp:102-104)
    if (flags[0] && g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by async step");
    return HEAT_OK;
}

int heat_async_sim_current(heat_async_sim* sim, double* out, size_t* step_index) {
    if (!sim) return fail(HEAT_EINVAL, "null simulator handle");
    HB_CUDA(cudaSetDevice(sim->ctx.device));
    if (sim->hist) {
        if (out) HB_TRY(heat_history_snapshot(sim->hist, 0, out));
        if (step_index) *step_index = sim->k;
        return HEAT_OK;
    }
    if (out)
        HB_CUDA(cudaMemcpyAsync(out, sim->field[sim->cur], sim->s.N * sizeof(double),
                                cudaMemcpyDeviceToHost, sim->ctx.stream));
    HB_CUDA(cudaStreamSynchronize(sim->ctx.stream));
    if (step_index) *step_index = sim->k;
    return HEAT_OK;
}

int heat_async_sim_destroy(heat_async_sim* sim) {
    sim_free(sim);
    return HEAT_OK;
}

}  // extern "C"

namespace hb {
// The simulator's current field on the device and its stream (ensemble.cu).
void async_sim_device_field(heat_async_sim* sim, const double** field, cudaStream_t* st) {
    *field = sim->field[sim->cur];
    *st = sim->ctx.stream;
}
}  // namespace hb
