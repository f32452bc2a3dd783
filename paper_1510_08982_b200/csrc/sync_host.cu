// sync_host.cu -- launch logic for K1 (sync_tb.cuh) and the synchronous
// C-ABI entry points: heat_sync_step / heat_sync_run / heat_sync_run_f32.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include <cudaTypedefs.h>

#include "runtime.cuh"
#include "sync_col.cuh"
#include "sync_cta.cuh"
#include "sync_tb.cuh"

namespace hb {

namespace {
constexpr int kV = 32;  // points per lane; also the maximum steps per pass

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 3-D view of a field as [chunk][128-B row][row elements] with 128B swizzle;
// the box is `box_chunks` whole V-point chunks.
template <typename Real, int V>
int make_chunk_map(CUtensorMap* m, const void* base, long long nchunks, int box_chunks) {
    using T = SyncTB<Real, V>;
    auto enc = tensor_map_encoder();
    if (!enc) return fail(HEAT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {cuuint64_t(T::kRowElems), cuuint64_t(T::kRowsPerChunk),
                                cuuint64_t(nchunks > 0 ? nchunks : 1)};
    const cuuint64_t strides[2] = {128, cuuint64_t(T::kChunkBytes)};
    const cuuint32_t box[3] = {cuuint32_t(T::kRowElems), cuuint32_t(T::kRowsPerChunk),
                               cuuint32_t(box_chunks)};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, sizeof(Real) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(HEAT_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return HEAT_OK;
}

// Compile-time variants of K1 (window buffers per warp x step-loop unroll);
// HEAT_SYNC_VARIANT selects one for A/B measurements, the default is the
// fastest measured on B200 (profiles/).
using SyncKernelFn = void (*)(CUtensorMap, CUtensorMap, SyncPassArgs);
using SyncKernelFn3 = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, SyncPassArgs);
struct SyncVariant {
    SyncKernelFn fn;
    int nbuf;
    int V;                    // points per lane
    int out;                  // exact points per tile
    int win_units, out_units; // tensor-map boxes (32-point units) of a window / its outputs
    int smem;                 // dynamic shared memory per CTA
    int halo;                 // halo points per side = max steps per pass
    bool dyn;                 // tiles dealt by an atomic counter
    int warps;                // warps per CTA
    int blocks_per_sm;        // filled by the occupancy query
    bool cta_tiles;           // one tile per CTA (K1c) instead of one per warp
    SyncKernelFn3 fn3 = nullptr;  // K1s (strips with a carried column): `out` is a chunk's
    int out1_units = 0;           // outputs; its later tiles store out1_units units
    const void* kernel() const {
        return fn3 ? reinterpret_cast<const void*>(fn3) : reinterpret_cast<const void*>(fn);
    }
};
template <typename Real, int V, int NBUF, int UNR, bool TMA_ST = true, int H = 32, bool DYN = false,
          int W = 4>
SyncVariant variant() {
    using T = SyncTB<Real, V, H, W>;
    return {sync_tb_kernel<Real, V, NBUF, UNR, TMA_ST, H, DYN, W>, NBUF, V, T::kOut, T::kWinUnits,
            T::kOutUnits, T::smem_bytes(NBUF), H, DYN, W, 0, false};
}
// K1c (sync_cta.cuh): G warps step one CTA-wide window, seams exchanged in
// shared memory; f64 only (48-point lanes)
template <typename Real, int V, int H, int G, int PU>
SyncVariant variant_cta() {
    using C = SyncCTA<Real, V, H, G>;
    return {sync_cta_kernel<Real, V, H, G, PU>, 2, V, C::kOut, C::kWinUnits, C::kOutUnits,
            C::smem_bytes(), H, true, G, 0, true};
}
// K1s (sync_col.cuh): chunks of CH tiles per warp, boundary column carried
template <typename Real, int V, int H, int CH, int PU, bool MID = false>
SyncVariant variant_col() {
    using K = SyncCol<Real, V, H, CH>;
    SyncVariant v{nullptr, 2, V, K::kChunkOut, SyncTB<Real, V, H>::kWinUnits, K::kOut0Units,
                  K::smem_bytes(), H, true, 4, 0, false};
    v.fn3 = sync_col_kernel<Real, V, H, CH, PU, MID>;
    v.out1_units = K::kOut1Units;
    return v;
}
template <typename Real, int CH, int PU, bool MID = false>
SyncVariant variant_col48() {
    if constexpr (sizeof(Real) == 8)
        return variant_col<Real, 48, 64, CH, PU, MID>();
    else
        return variant<Real, 64, 2, -4, true, 64, true>();  // = variant 15 for f32
}
// 24: K1s with 32-point lanes (3 CTAs of 4 warps per SM instead of 2)
template <typename Real, int CH, int PU>
SyncVariant variant_col32() {
    if constexpr (sizeof(Real) == 8) {
        SyncVariant v = variant_col<Real, 32, 64, CH, PU>();
        return v;
    } else {
        return variant<Real, 64, 2, -4, true, 64, true>();  // = variant 15 for f32
    }
}
template <typename Real, int PU>
SyncVariant variant_cta48() {
    if constexpr (sizeof(Real) == 8)
        return variant_cta<Real, 48, 64, 4, PU>();
    else
        return variant<Real, 64, 2, -4, true, 64, true>();  // = variant 15 for f32
}
// 48-point lanes exist for f64 only (48 f32 values are not whole 128-B rows);
// f32 takes 64-point lanes (256 B, two rows) with the same halo, buffers and deal
template <typename Real, int NBUF, bool TMA_ST = true, int H = 32, bool DYN = false, int UNR = 0>
SyncVariant variant48() {
    if constexpr (sizeof(Real) == 8)
        return variant<Real, 48, NBUF, UNR, TMA_ST, H, DYN>();
    else
        return variant<Real, 64, NBUF, UNR, TMA_ST, H, DYN>();
}
// 13: 48-point lanes, 64-point halo, 2 buffers, tiles dealt by an atomic counter:
// +6.2% over its static-deal twin 11 (3980 vs 3748 GLUPS on one box), which was +0.6% over
// 6 (48-point lanes, 32-point halo: 3874 GLUPS at 2^30; V = 32, variant 4: 3761).  Callers
// that cap the steps per pass below the default halo get kHalo32Variant.  tools/ab_sync.sh.
// 15: as 13 with the pipelined step loop unrolled x4 instead of x2: +0.45% (4017 vs 3998,
// twice, same box); unrolled x1 (14) loses 1.7%.
// 20: K1s (sync_col.cuh), chunks of 8 tiles with a carried boundary column:
// 4076 vs 4036 GLUPS for 15 on the same box, three times (95.3% of the stepped
// points exact against 91.7%; FP64 pipe 92.1% vs 93.4% active).  23: the same
// with the next tile's load issued half way through the steps (MID): 4077.8 vs
// 4076.0.  24: 32-point lanes, 3 CTAs per SM: 3956 vs 4073.
constexpr int kDefaultSyncVariant = 20;
constexpr int kHalo32Variant = 6;
constexpr int kSyncVariants = 25;

// The selected variant's table entry (no CUDA calls); `max_halo` (> 0) caps
// the halo, i.e. the steps per pass the caller will ask for.
template <typename Real>
SyncVariant& sync_variant_entry(int max_halo = 0) {
    // 0-5: V = 32 (buffers x step schedule); 6-8: wider lanes, same 32-point
    // halo (f64 only: an f32 lane of 48 points is not whole swizzle rows);
    // 9-10: register stores instead of the TMA store; 11-12: 64-point halo
    static SyncVariant table[kSyncVariants] = {
        variant<Real, kV, 2, 1>(),
        variant<Real, kV, 2, 2>(),
        variant<Real, kV, 1, 1>(),
        variant<Real, kV, 1, 2>(),
        variant<Real, kV, 2, 0>(),  // 4: pipelined steps, 2 buffers
        variant<Real, kV, 1, 0>(),  // 5: pipelined steps, 1 buffer
        variant48<Real, 2>(),        // 6: 48-point lanes, 2 buffers
        variant48<Real, 1>(),        // 7: 48-point lanes, 1 buffer
        variant<Real, 64, 1, 0>(),   // 8: 64-point lanes, 1 buffer
        variant48<Real, 2, false>(), // 9: 48-point lanes, 2 load buffers, register stores
        variant<Real, kV, 2, 0, false>(),  // 10: 32-point lanes, 2 load buffers, register stores
        variant48<Real, 2, true, 64>(),    // 11: 48-point lanes, 64-point halo (64 steps a pass)
        variant<Real, 64, 1, 0, true, 64>(),  // 12: 64-point lanes, 64-point halo, 1 buffer
        variant48<Real, 2, true, 64, true>(),  // 13: as 11, tiles dealt by an atomic counter
        variant48<Real, 2, true, 64, true, -1>(),  // 14: as 13, step loop not unrolled
        variant48<Real, 2, true, 64, true, -4>(),  // 15: as 13, step loop unrolled 4
        // 16: 64-point lanes (f64), 64-point halo, 2 buffers, atomic deal, unrolled 4,
        //     3 warps per CTA (2 x 3 x 32 KB of buffers per SM): 93.75% exact points
        variant<Real, 64, 2, -4, true, 64, true, (sizeof(Real) == 8 ? 3 : 4)>(),
        // 17: as 16, step loop unrolled 2
        variant<Real, 64, 2, 0, true, 64, true, (sizeof(Real) == 8 ? 3 : 4)>(),
        // 18: K1c, 4 warps x 48-point lanes in one CTA window, 64-point halo,
        //     atomic deal, step loop unrolled 4 (f32: variant 15's geometry)
        variant_cta48<Real, 4>(),
        // 19: as 18, step loop unrolled 2
        variant_cta48<Real, 2>(),
        // 20-22: K1s, 48x64 tiles in chunks with a carried boundary column (the
        //        chunk's later tiles need no left halo): chunks of 8 unrolled 4,
        //        of 16 unrolled 4, of 8 unrolled 3 (unrolled 2: -1.0%, 1: -4.2%)
        variant_col48<Real, 8, 4>(),
        variant_col48<Real, 16, 4>(),
        variant_col48<Real, 8, 3>(),
        variant_col48<Real, 8, 4, true>(),
        variant_col32<Real, 8, 4>(),
    };
    static const int idx = [] {
        const char* e = std::getenv("HEAT_SYNC_VARIANT");
        const int v = e ? std::atoi(e) : kDefaultSyncVariant;
        return (v >= 0 && v < kSyncVariants) ? v : kDefaultSyncVariant;
    }();
    if (max_halo > 0 && table[idx].halo > max_halo) {
        // f32 keeps 32-point lanes (48 f32 values are not whole swizzle rows)
        SyncVariant& h = table[sizeof(Real) == 8 ? kHalo32Variant : 4];
        if (h.halo <= max_halo) return h;
    }
    return table[idx];
}

template <typename Real>
int sync_variant(SyncVariant** out, int max_halo = 0) {
    SyncVariant& v = sync_variant_entry<Real>(max_halo);
    // per device (the current one): shared memory limit + occupancy
    HB_TRY(kernel_smem_config(v.kernel(), v.smem, v.warps * kWarp, &v.blocks_per_sm));
    *out = &v;
    return HEAT_OK;
}
}  // namespace

template <typename Real>
int sync_advance(int sms, Real* bufs[2], int& cur, long long n, double r, int periodic,
                 double c1, double c2, size_t steps, unsigned int* flag, cudaStream_t st) {
    SlabGeom g;
    g.len = n;
    g.out_lo = 0;
    g.out_hi = n;
    g.pin_lo = periodic ? -1 : 0;
    g.pin_hi = periodic ? -1 : n - 1;
    g.wrap = periodic;
    return sync_advance_slab<Real>(sms, bufs, cur, g, r, c1, c2, steps, flag, st);
}

// One K1 configuration (array, pins, coefficients, tensor maps of both
// ping-pong buffers) from which passes over any output range are launched.
template <typename Real>
struct SyncLauncher {
    using T = SyncTB<Real, kV>;
    SyncVariant* var = nullptr;
    int sms = 0;
    Real* bufs[2] = {nullptr, nullptr};
    CUtensorMap load_map[2], store_map[2], store_map1[2];
    SyncPassArgs a{};

    int init(int sms_, Real* b[2], const SlabGeom& g, double r, double c1, double c2,
             unsigned int* flag, int max_halo = 0) {
        HB_TRY(sync_variant<Real>(&var, max_halo));
        sms = sms_;
        bufs[0] = b[0];
        bufs[1] = b[1];
        a.len = g.len;
        a.pin_lo = g.pin_lo;
        a.pin_hi = g.pin_hi;
        a.wrap = g.wrap;
        a.r = r;
        if (sizeof(Real) == 8) {
            a.c = 1.0 - 2.0 * r;  // core.hpp:108: Real(1) - Real(2)*r, one rounding
        } else {
            const float rf = float(r);
            a.c = double(1.0f - 2.0f * rf);
        }
        a.c1 = c1;
        a.c2 = c2;
        a.nonfinite = flag;
        a.nchunks = g.len / kV;
        // tensor maps: [chunk][row][16 doubles] views of both ping-pong arrays,
        // 32-chunk boxes for window loads, 30-chunk boxes for output stores
        for (int i = 0; i < 2; ++i) {
            HB_TRY((make_chunk_map<Real, kV>(&load_map[i], bufs[i], a.nchunks, var->win_units)));
            HB_TRY((make_chunk_map<Real, kV>(&store_map[i], bufs[i], a.nchunks, var->out_units)));
            if (var->fn3)
                HB_TRY((make_chunk_map<Real, kV>(&store_map1[i], bufs[i], a.nchunks,
                                                 var->out1_units)));
        }
        return HEAT_OK;
    }

    // Advance outputs [out_lo, out_hi) by nsteps (<= V): reads bufs[src],
    // writes bufs[src ^ 1].
    // counter_slot: which of the context's tile counters (one per stream that
    // may run K1 concurrently) the launch uses.
    int pass(int src, long long out_lo, long long out_hi, int nsteps, bool check,
             cudaStream_t st, int counter_slot = 0) {
        if (out_lo % kV != 0) return fail(HEAT_ELOGIC, "sync pass: out_lo must be chunk aligned");
        if (out_hi <= out_lo) return HEAT_OK;
        if (nsteps > var->halo) return fail(HEAT_ELOGIC, "sync pass: more steps than the halo");
        long long tiles = (out_hi - out_lo + var->out - 1) / var->out;
        long long big = 0;
        if (var->fn3) {
            // K1s: chunks of CH tiles, then single tiles for the last ~4 per
            // resident warp (a single tile emits the first-tile count, out0)
            const long long out0 = (long long)var->out_units * 32;
            const long long resident = (long long)sms * var->blocks_per_sm * var->warps;
            const long long tail = std::min<long long>(out_hi - out_lo, 4 * resident * out0);
            big = (out_hi - out_lo - tail) / var->out;
            tiles = big + (out_hi - out_lo - big * var->out + out0 - 1) / out0;
        }
        const long long want = var->cta_tiles ? tiles : (tiles + var->warps - 1) / var->warps;
        const int grid = int(std::min<long long>(want, (long long)sms * var->blocks_per_sm));
        SyncPassArgs p = a;
        p.out_lo = out_lo;
        p.out_hi = out_hi;
        p.tiles = tiles;
        p.big_chunks = big;
        p.src = bufs[src];
        p.dst = bufs[src ^ 1];
        p.nsteps = nsteps;
        p.check_finite = check;
        if (var->dyn) {  // the stream owner's counter, zeroed in stream order
            p.counter = tile_counter_of(a.nonfinite) + counter_slot;
            HB_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(unsigned long long), st));
        }
        if (var->fn3)
            var->fn3<<<grid, var->warps * kWarp, var->smem, st>>>(load_map[src], store_map[src ^ 1],
                                                                 store_map1[src ^ 1], p);
        else
            var->fn<<<grid, var->warps * kWarp, var->smem, st>>>(load_map[src], store_map[src ^ 1], p);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return HEAT_OK;
    }
};

template <typename Real>
int sync_advance_slab(int sms, Real* bufs[2], int& cur, const SlabGeom& g, double r, double c1,
                      double c2, size_t steps, unsigned int* flag, cudaStream_t st,
                      int max_steps_per_pass) {
    if (steps == 0) return HEAT_OK;
    if (g.out_lo % kV != 0) return fail(HEAT_ELOGIC, "sync pass: out_lo must be chunk aligned");
    SyncLauncher<Real> L;
    HB_TRY(L.init(sms, bufs, g, r, c1, c2, flag, max_steps_per_pass));
    const int halo = L.var->halo;
    const int cap = max_steps_per_pass > 0 ? std::min(max_steps_per_pass, halo) : halo;
    while (steps > 0) {
        const int s = int(std::min<size_t>(steps, size_t(cap)));
        // With `rem` steps still to go after this pass, the final outputs need
        // this pass's values on [out_lo - rem, out_hi + rem): a slab whose
        // ghosts were refreshed for the whole advance (ghost width >= steps)
        // computes that shrinking light cone; a single domain clips it to
        // [0, len).  The finite check runs on the last pass only.
        const long long rem = (long long)(steps - size_t(s));
        const long long lo = g.out_lo - rem > 0 ? (g.out_lo - rem) / kV * kV : 0;
        const long long hi = std::min(g.len, g.out_hi + rem);
        HB_TRY(L.pass(cur, lo, hi, s, rem == 0, st));
        cur ^= 1;
        steps -= size_t(s);
    }
    return HEAT_OK;
}

int make_chunk_map_f64(CUtensorMap* m, const void* base, long long nchunks, int box_chunks) {
    return make_chunk_map<double, kV>(m, base, nchunks, box_chunks);
}

template int sync_advance<double>(int, double* [2], int&, long long, double, int, double, double,
                                  size_t, unsigned int*, cudaStream_t);
template int sync_advance<float>(int, float* [2], int&, long long, double, int, double, double,
                                 size_t, unsigned int*, cudaStream_t);
template int sync_advance_slab<double>(int, double* [2], int&, const SlabGeom&, double, double,
                                       double, size_t, unsigned int*, cudaStream_t, int);

namespace {

// Device-side TemperatureField validation (core.hpp:45-51): flag[2] |= 1 on a
// non-finite value.  Runs right after the upload so the host never walks the
// field (an O(N) host pass would dominate end-to-end time at N = 2^30).
// snap: also write the Dirichlet ends (each index is read, then written, by
// the one thread that owns it).
__global__ void validate_kernel(double* __restrict__ u, long long n, unsigned int* flag, int snap,
                                double c1, double c2) {
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        bad |= !isfinite(u[i]);
        if (snap && i == 0) u[0] = c1;
        if (snap && i == n - 1) u[n - 1] = c2;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag + 2, 1u);
}

__global__ void narrow_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = float(in[i]);
}

}  // namespace

// Upload u0 (caller's host buffer, pinned or pageable) into `dst` (double),
// validate it on the device and snap the Dirichlet ends
// (prepare_initial, sync_solver.cpp:25-37).  Leaves the stream synchronised.
int upload_prepared(DevCtx& d, const double* u0, size_t n, int bc_kind, double c1, double c2,
                    double* dst) {
    cudaStream_t st = d.stream;
    // The end check reads the host field; the device finite check still comes
    // first in the errors reported (the TemperatureField ctor precedes
    // prepare_initial), and the same kernel snaps the ends: one round trip.
    constexpr double kTol = 1e-9;  // kDirichletEndTol, sync_solver.hpp:44
    const bool dir = bc_kind == HEAT_BC_DIRICHLET;
    const bool ends_ok = !dir || (std::abs(u0[0] - c1) <= kTol && std::abs(u0[n - 1] - c2) <= kTol);
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 4 * sizeof(unsigned int), st));
    HB_CUDA(cudaMemcpyAsync(dst, u0, n * sizeof(double), cudaMemcpyHostToDevice, st));
    validate_kernel<<<d.sms * 4, 256, 0, st>>>(dst, (long long)n, d.flag, dir && ends_ok, c1, c2);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    unsigned int flags[4] = {0, 0, 0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (flags[2]) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    if (!ends_ok) return fail(HEAT_EINVAL, "Dirichlet BC inconsistent with initial end values");
    return HEAT_OK;
}

namespace {

// Validation + Dirichlet snap of one uploaded chunk [lo, hi) of the streamed
// sync_run: flag[2] |= 1 on a non-finite value (core.hpp:45-51), then the
// ends take c1 / c2 exactly (prepare_initial, sync_solver.cpp:25-37).
__global__ void prep_chunk_kernel(double* __restrict__ u, long long lo, long long hi, long long n,
                                  double c1, double c2, unsigned int* flag) {
    bool bad = false;
    for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
         i += (long long)gridDim.x * blockDim.x) {
        bad |= !isfinite(u[i]);
        if (i == 0) u[0] = c1;
        if (i == n - 1) u[n - 1] = c2;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag + 2, 1u);
}

constexpr size_t kStreamMinPoints = size_t(1) << 24;  // below: copies are cheap, one shot
constexpr int kStreamChunks = 16;
// above: copies are a small share (and the S x C pass events add up).  At
// cfg3 (157 passes) streaming hides both copies: 2.64 s against 2.94 s for
// the one-shot path with pinned buffers, 2.65 s against 3.79 s with pageable
// ones (tools/pageable_trace.py, HEAT_STREAM_TRACE=1)
constexpr size_t kStreamMaxPasses = 1024;
// HEAT_STREAM_MAX_PASSES overrides kStreamMaxPasses (A/B only)
static size_t stream_max_passes() {
    static const size_t v = [] {
        const char* e = std::getenv("HEAT_STREAM_MAX_PASSES");
        return e ? size_t(std::atoll(e)) : kStreamMaxPasses;
    }();
    return v;
}

}  // namespace

// Chunk boundaries of the streamed sync_run for N points and a "wave" (one
// tile per resident warp, in points).  Chunks of whole waves keep every
// launch free of a ragged last wave.  Large fields get graded chunks (4, 7,
// 12, 20, 32, 52 waves, <= 64-wave middle, the head mirrored at the end):
// the first pass starts after a short upload and the last download is short,
// while neighbouring chunks differ by less than the compute/copy time ratio
// (~1.8), so neither the compute nor the download stream starves.  Smaller
// fields: 16 equal chunks.  Every chunk but the last starts on a 32-point unit.
std::vector<long long> stream_chunk_plan(long long N, long long wave) {
    std::vector<long long> B{0};
    if (wave > 0 && N >= 128 * wave) {
        std::vector<long long> head;
        long long rem = N;
        for (long long w = 4; w < 64 && rem > 8 * w * wave; w = (w * 8 + 4) / 5) {
            head.push_back(w * wave);
            rem -= 2 * w * wave;
        }
        for (long long h : head) B.push_back(B.back() + h);
        const long long m = (rem + 64 * wave - 1) / (64 * wave);
        const long long each = (rem / m) / wave * wave;  // whole waves; the last absorbs the rest
        for (long long j = 0; j + 1 < m; ++j) B.push_back(B.back() + each);
        long long tail = 0;
        for (long long h : head) tail += h;
        B.push_back((N - tail) / kV * kV);  // chunk starts stay 32-aligned
        for (size_t j = head.size(); j-- > 1;) B.push_back(B.back() + head[j]);
        B.push_back(N);                     // the last chunk absorbs N mod 32
    } else {
        const long long cp = ((N + kStreamChunks - 1) / kStreamChunks + kV - 1) / kV * kV;
        for (long long b = cp; b < N; b += cp) B.push_back(b);
        B.push_back(N);
    }
    return B;
}

namespace {

// Streamed sync_run (large Dirichlet fields, final state only): the field is
// uploaded in C chunks on one copy stream, advanced chunk by chunk on the
// compute stream, and downloaded chunk by chunk on a second copy stream, so
// the 2 x 8N bytes of PCIe traffic overlap the temporal-blocked passes.
//
// Pass pi of chunk c advances outputs R(pi, c) = [B_c - (pi+1)*h,
// B_{c+1} - (pi+1)*h) (first range from 0, last to n), h = the kernel's halo
// (32 or 64 points): shifting each pass's ranges by h -- the reach of one
// pass of <= h steps --
// makes every input of R(pi, c) an output of passes already issued for
// chunks <= c, and chunk c's first pass needs only uploaded chunks <= c.
// Issued in chunk-major order on one stream, no launch overwrites values a
// later launch still reads: the pass-(pi+2) write of chunk c ends exactly
// where the pass-(pi+1) read of chunk c+1 begins.  Window reads beyond a
// range's last output are stale values that cannot reach an exact output
// within one pass.  The per-range kernels are the same K1 passes as the
// one-shot path, so results are bit-identical.
int sync_run_streamed(DevCtx& d, const double* u0, size_t n, double r, double c1, double c2,
                      size_t k_end, double* final_out) {
    using T = SyncTB<double, kV>;
    const long long N = (long long)n;
    const size_t pitch = (n + 63) / 64 * 64;
    HB_TRY(ensure_buffers(d, 2 * pitch * sizeof(double)));
    double* bufs[2] = {static_cast<double*>(d.buf[0]), static_cast<double*>(d.buf[0]) + pitch};
    cudaStream_t st = d.stream;
    SlabGeom g;
    g.len = N;
    g.out_lo = 0;
    g.out_hi = N;
    g.pin_lo = 0;
    g.pin_hi = N - 1;
    SyncLauncher<double> L;
    HB_TRY(L.init(d.sms, bufs, g, r, c1, c2, d.flag));
    const long long shift = L.var->halo;  // steps per pass = reach of one pass
    const long long S = ((long long)k_end + shift - 1) / shift;  // passes
    // Chunk boundaries.  A "wave" is one tile per resident warp; chunks of
    // whole waves keep every launch free of a ragged last wave.  Large fields
    // get graded chunks (4, 6, 10, 16, 26, 41 waves, <= 64-wave middle, the
    // head mirrored at the end): the first pass starts after a short upload
    // and the last download is short, while neighbouring chunks differ by
    // less than the compute/copy time ratio (~1.8), so neither the compute
    // nor the download stream starves.  Smaller fields: 16 equal chunks.
    // (K1s: a wave of single tiles too -- each launch deals its range's last
    // tiles one by one anyway -- so the chunk plan is the K1 one)
    const long long tile_out = L.var->fn3 ? (long long)L.var->out_units * kV : L.var->out;
    const long long wave = (long long)d.sms * L.var->blocks_per_sm *
                           (L.var->cta_tiles ? 1 : L.var->warps) * tile_out;
    const std::vector<long long> B = stream_chunk_plan(N, wave);
    const int C = int(B.size()) - 1;
    for (int c = 0; c < C; ++c)
        if (B[c + 1] - B[c] <= (S + 1) * shift || B[c] % kV)
            return fail(HEAT_ELOGIC, "streamed sync_run: chunk plan violates the shift bound");
    auto lo = [&](int c, long long pi) { return c == 0 ? 0 : B[c] - (pi + 1) * shift; };
    auto hi = [&](int c, long long pi) { return c == C - 1 ? N : B[c + 1] - (pi + 1) * shift; };

    // Chunks alternate between two compute streams.  Pass pi of chunk c needs
    // pass pi-1 of chunks c and c-1 only (its inputs end inside R(pi-1, c) and
    // begin inside R(pi-1, c-1)); every later pass of chunk c-1 touches its
    // buffers only below where chunk c's pass-pi ranges begin.  So chunk c's
    // early passes run beside chunk c-1's late ones, and each launch's last
    // tiles share the GPU with the other stream's work instead of idling it.
    cudaStream_t cs[2] = {st, d.stream2};
    std::vector<cudaEvent_t> ev(size_t(C) + 1 + size_t(S) * C, nullptr);  // up[c], ready, E(pi,c)
    struct Cleanup {
        std::vector<cudaEvent_t>& e;
        ~Cleanup() {
            for (auto x : e)
                if (x) cudaEventDestroy(x);
        }
    } cleanup{ev};
    for (auto& e : ev) HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t* up = ev.data();
    cudaEvent_t ready = ev[C];
    auto E = [&](long long pi, int c) { return ev[size_t(C) + 1 + size_t(pi) * C + c]; };

    // A PAGEABLE field (the drop-in caller's std::vector) would make every
    // copy block the host inside the driver's own staging, which serialises
    // the pipeline: it goes through rings of pinned slots instead (4 for the
    // uploads, 4 for the downloads), filled and drained by host threads while
    // the copy engines move the other slots.  Downloads run on their own host
    // thread, so a chunk's result leaves as soon as its last pass is done,
    // while later chunks are still being uploaded.
    const bool page_in = host_pageable(u0), page_out = host_pageable(final_out);
    // HEAT_STREAM_TRACE=1: host-side phase times on stderr (A/B only)
    static const bool trace = std::getenv("HEAT_STREAM_TRACE") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    auto secs = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double>(b - a).count();
    };
    unsigned char* slots[kRingSlots] = {};
    if (page_in || page_out) HB_TRY(host_ring(d, slots));
    const int ncpu = int(std::max(1u, std::thread::hardware_concurrency()));
    const int hthreads = std::min(8, std::max(1, page_in && page_out ? ncpu / 2 : ncpu));
    const long long slot_pts = (long long)(kRingSlotBytes / sizeof(double));
    constexpr int kHalf = kRingSlots / 2;
    struct Ring {  // one direction's slots: j in [base, base + kHalf)
        int base, next = 0;
        bool busy[kHalf] = {};
    };
    auto take_slot = [&](Ring& R, int* j) -> int {  // the next slot, once its last copy is done
        const int i = R.next;
        R.next = (R.next + 1) % kHalf;
        if (R.busy[i]) HB_CUDA(cudaEventSynchronize(d.ring_ev[R.base + i]));
        R.busy[i] = false;
        *j = R.base + i;
        return HEAT_OK;
    };
    Ring rin{0}, rout{kHalf};
    double t_copy_in = 0, t_copy_out = 0, t_drain_wait = 0, t_down_end = 0;

    // the flag reset precedes every upload and every kernel on either stream
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 4 * sizeof(unsigned int), st));
    HB_CUDA(cudaEventRecord(ready, st));
    HB_CUDA(cudaStreamWaitEvent(d.h2d, ready, 0));
    HB_CUDA(cudaStreamWaitEvent(cs[1], ready, 0));

    const int fin = int(S & 1);
    // downloads: chunk c's final range once E(S-1, c) is recorded (enq > c)
    std::atomic<int> enq{0};
    std::atomic<bool> abort_dl{false};
    auto download_all = [&]() -> int {
        struct Pending {
            int j;
            double* dst;
            size_t bytes;
        };
        std::vector<Pending> pend;  // slot downloads not yet copied out (FIFO)
        size_t head = 0;
        auto drain_one = [&]() -> int {
            const Pending pd = pend[head++];
            const auto w0 = clk::now();
            HB_CUDA(cudaEventSynchronize(d.ring_ev[pd.j]));
            const auto c0 = clk::now();
            t_drain_wait += secs(w0, c0);
            parallel_memcpy(pd.dst, slots[pd.j], pd.bytes, hthreads);
            t_copy_out += secs(c0, clk::now());
            rout.busy[pd.j - rout.base] = false;
            return HEAT_OK;
        };
        for (int c = 0; c < C; ++c) {
            while (enq.load(std::memory_order_acquire) <= c) {
                if (abort_dl.load()) return HEAT_OK;
                std::this_thread::yield();
            }
            const long long a0 = lo(c, S - 1), a1 = hi(c, S - 1);
            HB_CUDA(cudaStreamWaitEvent(d.d2h, E(S - 1, c), 0));
            if (!page_out) {
                HB_CUDA(cudaMemcpyAsync(final_out + a0, bufs[fin] + a0,
                                        (a1 - a0) * sizeof(double), cudaMemcpyDeviceToHost, d.d2h));
                continue;
            }
            for (long long o = a0; o < a1; o += slot_pts) {
                const long long cnt = std::min(slot_pts, a1 - o);
                // keep kHalf - 1 downloads in flight; copy out the oldest
                while (pend.size() - head >= size_t(kHalf - 1)) HB_TRY(drain_one());
                int j = 0;
                HB_TRY(take_slot(rout, &j));
                HB_CUDA(cudaMemcpyAsync(slots[j], bufs[fin] + o, size_t(cnt) * sizeof(double),
                                        cudaMemcpyDeviceToHost, d.d2h));
                HB_CUDA(cudaEventRecord(d.ring_ev[j], d.d2h));
                rout.busy[j - rout.base] = true;
                pend.push_back({j, final_out + o, size_t(cnt) * sizeof(double)});
            }
        }
        while (head < pend.size()) HB_TRY(drain_one());
        t_down_end = secs(t_start, clk::now());
        return HEAT_OK;
    };
    int dl_status = HEAT_OK;
    std::string dl_msg;
    std::thread downloader;
    if (page_out)
        downloader = std::thread([&] {
            cudaSetDevice(d.device);
            dl_status = download_all();
            if (dl_status != HEAT_OK) dl_msg = last_error_msg();
        });
    struct Joiner {
        std::thread& t;
        std::atomic<bool>& ab;
        ~Joiner() {
            if (t.joinable()) {
                ab.store(true);
                t.join();
            }
        }
    } joiner{downloader, abort_dl};

    for (int c = 0; c < C; ++c) {
        const long long a0 = B[c], a1 = B[c + 1];
        cudaStream_t s_c = cs[c & 1];
        if (!page_in) {
            HB_CUDA(cudaMemcpyAsync(bufs[0] + a0, u0 + a0, (a1 - a0) * sizeof(double),
                                    cudaMemcpyHostToDevice, d.h2d));
        } else {
            for (long long o = a0; o < a1; o += slot_pts) {
                const long long cnt = std::min(slot_pts, a1 - o);
                int j = 0;
                HB_TRY(take_slot(rin, &j));
                const auto c0 = clk::now();
                parallel_memcpy(slots[j], u0 + o, size_t(cnt) * sizeof(double), hthreads);
                t_copy_in += secs(c0, clk::now());
                HB_CUDA(cudaMemcpyAsync(bufs[0] + o, slots[j], size_t(cnt) * sizeof(double),
                                        cudaMemcpyHostToDevice, d.h2d));
                HB_CUDA(cudaEventRecord(d.ring_ev[j], d.h2d));
                rin.busy[j - rin.base] = true;
            }
        }
        HB_CUDA(cudaEventRecord(up[c], d.h2d));
        HB_CUDA(cudaStreamWaitEvent(s_c, up[c], 0));  // chunks <= c are in
        prep_chunk_kernel<<<d.sms * 2, 256, 0, s_c>>>(bufs[0], a0, a1, N, c1, c2, d.flag);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
        size_t left = k_end;
        for (long long pi = 0; pi < S; ++pi) {
            if (c > 0 && pi > 0) HB_CUDA(cudaStreamWaitEvent(s_c, E(pi - 1, c - 1), 0));
            const int s = int(std::min<size_t>(left, size_t(shift)));
            HB_TRY(L.pass(int(pi & 1), lo(c, pi), hi(c, pi), s, pi == S - 1, s_c, c & 1));
            HB_CUDA(cudaEventRecord(E(pi, c), s_c));
            left -= size_t(s);
        }
        enq.store(c + 1, std::memory_order_release);
    }
    const auto t_enq = clk::now();
    if (page_out) {
        downloader.join();
        if (dl_status != HEAT_OK) return fail(dl_status, dl_msg);
    } else {
        HB_TRY(download_all());  // pinned destination: the copies are only enqueued
    }
    if (trace)
        std::fprintf(stderr,
                     "[stream] chunks %d passes %lld: uploads+enqueue %.3f s (copy-in %.3f), "
                     "downloads done at %.3f s (drain waits %.3f, copy-out %.3f), end %.3f s\n",
                     C, S, secs(t_start, t_enq), t_copy_in, t_down_end, t_drain_wait, t_copy_out,
                     secs(t_start, clk::now()));
    HB_CUDA(cudaStreamWaitEvent(st, E(S - 1, C - 1), 0));  // both streams done
    if (C > 1) HB_CUDA(cudaStreamWaitEvent(st, E(S - 1, C - 2), 0));
    unsigned int flags[4] = {0, 0, 0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    HB_CUDA(cudaStreamSynchronize(d.d2h));
    if (flags[2]) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    return HEAT_OK;
}

constexpr size_t kOverlapSnapPoints = size_t(1) << 20;  // below: one stream is fine

// sync_run of a large f64 field with a recorded trajectory, snapshot
// downloads overlapped with the compute (streaming the
// trajectory).  A recorded step is copied device-to-device into one of two
// staging buffers (HBM speed) and downloaded from there on the copy stream
// while the next segment computes; events keep each staging buffer until its
// download has read it.  The host issues snapshot j's download only after
// enqueueing segment j+1, so even a pageable destination (whose copy blocks
// the host) overlaps the GPU's next segment.  Non-finite values are
// absorbing, so the finite check of the last pass decides the outcome.
int sync_run_overlapped(DevCtx& d, double** bufs, size_t n, double r, int periodic, double c1,
                        double c2, size_t k_end, size_t stride, double* final_out,
                        double* snapshots, size_t* steps_out, size_t max_snapshots,
                        size_t* n_snapshots) {
    cudaStream_t st = d.stream;
    const size_t pitch = (n + 63) / 64 * 64;
    if (d.snaps_bytes < 2 * pitch * sizeof(double)) {
        if (d.snaps) cudaFree(d.snaps);
        d.snaps = nullptr;
        d.snaps_bytes = 0;
        HB_CUDA(cudaMalloc(&d.snaps, 2 * pitch * sizeof(double)));
        d.snaps_bytes = 2 * pitch * sizeof(double);
    }
    double* stage[2] = {static_cast<double*>(d.snaps), static_cast<double*>(d.snaps) + pitch};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // ready[2], done[2]
    struct Cleanup {
        cudaEvent_t* e;
        ~Cleanup() {
            for (int i = 0; i < 4; ++i)
                if (e[i]) cudaEventDestroy(e[i]);
        }
    } cleanup{ev};
    for (auto& e : ev) HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bool done_recorded[2] = {false, false};
    long long pend_row = -1;
    int pend_slot = 0;
    auto issue_pending = [&]() -> int {  // the download of the staged snapshot
        if (pend_row < 0) return HEAT_OK;
        HB_CUDA(cudaStreamWaitEvent(d.d2h, ev[pend_slot], 0));
        HB_CUDA(cudaMemcpyAsync(snapshots + size_t(pend_row) * n, stage[pend_slot],
                                n * sizeof(double), cudaMemcpyDeviceToHost, d.d2h));
        HB_CUDA(cudaEventRecord(ev[2 + pend_slot], d.d2h));
        done_recorded[pend_slot] = true;
        pend_row = -1;
        return HEAT_OK;
    };
    size_t ns = 0;
    int cur = 0;
    auto stage_row = [&](size_t kk) -> int {  // snapshot of step kk into a staging buffer
        if (ns < max_snapshots) {
            const int slot = int(ns & 1);
            if (done_recorded[slot]) HB_CUDA(cudaStreamWaitEvent(st, ev[2 + slot], 0));
            HB_CUDA(cudaMemcpyAsync(stage[slot], bufs[cur], n * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st));
            HB_CUDA(cudaEventRecord(ev[slot], st));
            HB_TRY(issue_pending());  // the previous one, now that this segment is queued
            pend_row = (long long)ns;
            pend_slot = slot;
            if (steps_out) steps_out[ns] = kk;
        }
        ++ns;
        return HEAT_OK;
    };
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 2 * sizeof(unsigned int), st));
    HB_TRY(stage_row(0));
    size_t k = 0;
    while (k < k_end) {
        const size_t next = std::min(k_end, (k / stride + 1) * stride);
        HB_TRY(sync_advance<double>(d.sms, bufs, cur, (long long)n, r, periodic, c1, c2, next - k,
                                    d.flag, st));
        k = next;
        HB_TRY(stage_row(k));
    }
    HB_TRY(issue_pending());
    if (final_out)
        HB_CUDA(cudaMemcpyAsync(final_out, bufs[cur], n * sizeof(double), cudaMemcpyDeviceToHost,
                                st));
    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    HB_CUDA(cudaStreamSynchronize(d.d2h));
    if (flags[0]) {
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    if (n_snapshots) *n_snapshots = ns;
    return HEAT_OK;
}

// Shared body of sync_run / sync_run_f32 (sync_solver.cpp:52-91).  Snapshots
// and the final state are copied straight into the caller's buffers.
template <typename Real>
int sync_run_impl(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                  size_t k_end, size_t stride, double* final_out, double* snapshots,
                  size_t* steps_out, size_t max_snapshots, size_t* n_snapshots,
                  float* kernel_ms = nullptr, bool one_cta = false) {
    if (n < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u0) return fail(HEAT_EINVAL, "null field pointer");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    if (stride == 0) stride = default_stride(n);
    // Small f64 fields (the paper's regime): the whole run on one CTA (K7).
    if (sizeof(Real) == 8 && n <= sync_small_max_points() && !std::getenv("HEAT_NO_SMALL_SYNC"))
        return sync_run_small(reinterpret_cast<const double*>(u0), n, r, bc_kind, c1, c2, k_end,
                              stride, final_out, snapshots, steps_out, max_snapshots,
                              n_snapshots, kernel_ms, one_cta);

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const bool f32 = sizeof(Real) == 4;
    // Large Dirichlet runs that only want the final state: stream the copies
    // under the compute.  The host end check (sync_solver.cpp:29-31) runs
    // first; when it fails, the one-shot path reports the reference's errors
    // in the reference's order (a non-finite field before the end check).
    if (!f32 && final_out && !snapshots && !steps_out && bc_kind == HEAT_BC_DIRICHLET &&
        n >= kStreamMinPoints && k_end > 0 &&
        (k_end + sync_variant_entry<double>().halo - 1) / sync_variant_entry<double>().halo <=
            stream_max_passes() &&
        std::abs(u0[0] - c1) <= 1e-9 && std::abs(u0[n - 1] - c2) <= 1e-9 && !kernel_ms &&
        !std::getenv("HEAT_NO_STREAMED_SYNC"))
        return sync_run_streamed(*d, reinterpret_cast<const double*>(u0), n, r, c1, c2, k_end,
                                 final_out);
    const size_t pitch = (n + 63) / 64 * 64;  // keep the second array 256-B aligned
    const size_t need = 2 * pitch * sizeof(Real) + (f32 ? pitch * sizeof(double) : 0);
    HB_TRY(ensure_buffers(*d, need));
    Real* bufs[2] = {static_cast<Real*>(d->buf[0]), static_cast<Real*>(d->buf[0]) + pitch};
    double* staging = f32 ? reinterpret_cast<double*>(bufs[1] + pitch)
                          : reinterpret_cast<double*>(bufs[0]);
    cudaStream_t st = d->stream;
    HB_TRY(upload_prepared(*d, u0, n, bc_kind, c1, c2, staging));
    if (f32) {
        narrow_kernel<<<d->sms * 4, 256, 0, st>>>(staging, reinterpret_cast<float*>(bufs[0]),
                                                  (long long)n);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }

    std::vector<Real> host;  // f32 staging for snapshots only
    size_t ns = 0;
    // Copies the device field into snapshot row `ns` (or `final_out`).
    auto fetch = [&](const Real* dev, double* out_row) -> int {
        if (!f32) {
            HB_CUDA(cudaMemcpyAsync(out_row, dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
            return HEAT_OK;
        }
        host.resize(n);
        HB_CUDA(cudaMemcpyAsync(host.data(), dev, n * sizeof(Real), cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        for (size_t i = 0; i < n; ++i) out_row[i] = double(host[i]);
        return HEAT_OK;
    };
    auto record = [&](const Real* dev, size_t k) -> int {
        if (ns < max_snapshots) {
            if (snapshots) HB_TRY(fetch(dev, snapshots + ns * n));
            if (steps_out) steps_out[ns] = k;
        }
        ++ns;
        return HEAT_OK;
    };
    const bool want_snaps = snapshots != nullptr || steps_out != nullptr;
    int cur = 0;
    size_t k = 0;
    const int periodic = bc_kind == HEAT_BC_PERIODIC;
    if (!f32 && snapshots && n >= kOverlapSnapPoints && max_snapshots > 0 && !kernel_ms &&
        !std::getenv("HEAT_NO_OVERLAP_SNAPS"))
        return sync_run_overlapped(*d, reinterpret_cast<double**>(bufs), n, r, periodic, c1, c2,
                                   k_end, stride, final_out, snapshots, steps_out, max_snapshots,
                                   n_snapshots);
    if (want_snaps) HB_TRY(record(bufs[0], 0));

    while (k < k_end) {
        // advance to the next recorded step (or straight to k_end)
        size_t next = want_snaps ? std::min(k_end, (k / stride + 1) * stride) : k_end;
        EventPair ev;
        if (kernel_ms) HB_TRY(ev.begin(st));
        HB_TRY(sync_advance<Real>(d->sms, bufs, cur, (long long)n, r, periodic, c1, c2, next - k,
                                  d->flag, st));
        if (kernel_ms) HB_TRY(ev.end(st));
        k = next;
        unsigned int flags[2] = {0, 0};
        HB_CUDA(cudaMemcpyAsync(flags, d->flag, sizeof flags, cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        if (kernel_ms) {
            float seg = 0.f;
            HB_TRY(ev.elapsed(&seg));
            *kernel_ms += seg;
        }
        if (flags[0]) {
            if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
            return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
        }
        if (want_snaps) HB_TRY(record(bufs[cur], k));
    }
    if (final_out) HB_TRY(fetch(bufs[cur], final_out));
    HB_CUDA(cudaStreamSynchronize(st));
    if (n_snapshots) *n_snapshots = ns;  // 0 when no trajectory was requested
    return HEAT_OK;
}

}  // namespace
}  // namespace hb

using namespace hb;

namespace hb {
int sync_run_timed(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t k_end, double* final_out, float* kernel_ms) {
    *kernel_ms = 0.f;
    // exec_run(Barriered): K7, the executor whose PE warps all meet at one CTA
    // barrier per round (K7c, sync_run's kernel, has no barrier across CTAs)
    return sync_run_impl<double>(u0, n, r, bc_kind, c1, c2, k_end, k_end, final_out, nullptr,
                                 nullptr, 0, nullptr, kernel_ms, true);
}
}  // namespace hb

extern "C" int heat_stream_chunk_plan(size_t n, size_t wave_points, size_t* bounds, size_t cap,
                                      size_t* count) {
    const std::vector<long long> B = stream_chunk_plan((long long)n, (long long)wave_points);
    for (size_t j = 0; j < B.size() && j < cap; ++j) bounds[j] = size_t(B[j]);
    if (count) *count = B.size();
    return HEAT_OK;
}

extern "C" int heat_sync_kernel_info(int* points_per_lane, int* buffers,
                                     int* exact_points_per_tile, int* steps_per_pass) {
    const SyncVariant& v = sync_variant_entry<double>();
    if (points_per_lane) *points_per_lane = v.V;
    if (buffers) *buffers = v.nbuf;
    if (exact_points_per_tile) *exact_points_per_tile = v.out;
    if (steps_per_pass) *steps_per_pass = v.halo;
    return HEAT_OK;
}

extern "C" int heat_sync_step(const double* u, size_t n, double r, int bc_kind, double c1,
                              double c2, double* out) {
    return sync_run_impl<double>(u, n, r, bc_kind, c1, c2, 1, 1, out, nullptr, nullptr, 0,
                                 nullptr);
}

extern "C" int heat_sync_run(const double* u0, size_t n, double r, int bc_kind, double c1,
                             double c2, size_t k_end, size_t stride, double* final_out,
                             double* snapshots, size_t* steps, size_t max_snapshots,
                             size_t* n_snapshots) {
    // Small fields go to K7 (one CTA, sync_small.cu), large Dirichlet runs
    // that want only the final state to the streamed path, the rest to K1.
    return sync_run_impl<double>(u0, n, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                                 steps, max_snapshots, n_snapshots);
}

extern "C" int heat_sync_run_f32(const double* u0, size_t n, double r, int bc_kind, double c1,
                                 double c2, size_t k_end, size_t stride, double* final_out,
                                 double* snapshots, size_t* steps, size_t max_snapshots,
                                 size_t* n_snapshots) {
    return sync_run_impl<float>(u0, n, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                                steps, max_snapshots, n_snapshots);
}
