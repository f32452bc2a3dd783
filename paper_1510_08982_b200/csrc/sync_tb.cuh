// sync_tb.cuh -- K1: temporal-blocked synchronous FTCS pass for sm_100a.
//
// Replaces detail::sync_step_into (sync_solver.hpp:26-39) iterated by
// run_impl (sync_solver.cpp:70-75) and run_barriered (async_exec.cpp:57-114):
// one launch advances a range of the field by `nsteps` (<= H) Jacobi steps.
//
// Layout / mapping (template V points per lane, halo H; default 48 x 64)
//   * A WARP owns one tile: 32 lanes x V consecutive points (a "window" of
//     32V points).  Lane l holds points [w0 + lV, w0 + (l+1)V) in registers.
//   * Neighbour values inside a lane are registers; across lanes one
//     __shfl_up / __shfl_down of the boundary PRODUCT r*u per step.
//   * The first and last H points of the window are halo (redundant
//     recompute): after s <= H steps points [H, 32V - H) are exact, so a tile
//     emits 32V - 2H points: tile t covers outputs [out_lo + t*kOut,
//     out_lo + (t+1)*kOut), window w0 = that - H.  (V = 32, H = 32: lanes
//     1..30.)
//   * No block barrier anywhere: warps are independent.  Tiles are dealt
//     statically (warp w: tiles w, w + nwarps, ...) or, in the DYN variants
//     (the default), by an atomic counter so no warp idles at a pass's end.
//   * Each warp double-buffers its window in shared memory.  One elected lane
//     moves a whole window with ONE TMA tensor copy (cp.async.bulk.tensor.3d,
//     SASS UTMALDG) into a 128B-swizzled buffer -- the tensor map views the
//     array in 32-point units of two 128-B rows, and the swizzle makes the
//     per-lane 16-B shared loads conflict-light -- while the previous tile is
//     being stepped; results return through the same buffer, staged shifted
//     by the halo, with one TMA tensor store (UTMASTG) of the exact units.
//   * Tiles whose window touches a pinned end, leaves [0, len) or whose
//     outputs overrun out_hi take the generic path: per-lane element loads
//     (zero fill or modular wrap), Dirichlet ends re-pinned after every
//     step, bounds-checked stores.
//
// HBM traffic per pass: read 32V + write 32V - 2H points per (32V - 2H)*s
// updates, i.e. ~16/s bytes per lattice update (0.25 B at s = 64) -- the
// pass is bound by the FP64 pipe (4 DP instructions per update), not by HBM.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace hb {

template <typename Real, int V, int H = 32, int W = 4>
struct SyncTB {
    static constexpr int kChunkBytes = V * int(sizeof(Real));
    static constexpr int kRowsPerChunk = kChunkBytes / 128;       // 128-B swizzle rows
    static constexpr int kRowElems = 128 / int(sizeof(Real));
    static constexpr int kPer16 = 16 / int(sizeof(Real));         // elements per 16-B unit
    static constexpr int kBufBytes = kWarp * kChunkBytes;         // dense window
    // The halo is H points per side (32 unless a variant asks for more): a
    // pass of <= H steps leaves window points [H, 32V-H) exact.  At V = 32,
    // H = 32 that is lanes 1..30; wider lanes (V = 48, 64) waste a smaller
    // share on the halo and pay the per-tile costs (TMA, staging, pipeline
    // fill) over more points; a wider halo (H = 64) pays the per-pass costs
    // over more steps.
    static constexpr int kHalo = H;
    static constexpr int kUnit = 32;  // tensor-map coordinate unit (points); windows start on one
    static constexpr int kWinUnits = kWarp * V / kUnit;
    static constexpr int kOutUnits = kWinUnits - 2 * kHalo / kUnit;
    static constexpr int kOut = kWarp * V - 2 * kHalo;            // exact points per tile
    static constexpr int kHaloRows = kHalo * int(sizeof(Real)) / 128;
    static constexpr int kWarpsPerCta = W;  // 3 for 64-point f64 lanes: 2 CTAs x 3 x 2 x 16 KB fit an SM
    static constexpr int kThreads = kWarpsPerCta * kWarp;
    // shared memory for NBUF window buffers per warp (+ mbarriers, + 1 KB alignment slack)
    static constexpr int smem_bytes(int nbuf) {
        return kWarpsPerCta * nbuf * kBufBytes + kWarpsPerCta * 2 * 8 + 1024;
    }
    static constexpr int kMaxSteps = kHalo;
    // resident CTAs per SM the launch bounds promise (registers: V doubles per
    // lane in registers; V > 32 needs ~210 registers)
    static constexpr int min_blocks(int nbuf) { return V == 32 ? (nbuf == 1 ? 4 : 3) : 2; }
    static_assert(kChunkBytes % 128 == 0, "chunk must be whole 128-B swizzle rows");
    static_assert(kBufBytes % 1024 == 0, "window buffers must keep the 1 KB swizzle alignment");
    static_assert((kWarp * V) % kUnit == 0 && kHalo % kUnit == 0, "windows of whole units");
    static_assert(2 * kHalo < kWarp * V, "a window must keep exact points");
};

// Byte offset of 16-B unit `m` of lane-slot `slot`'s chunk in a 128B-swizzled
// buffer (row = slot*rows_per_chunk + m/8, unit ^= row & 7).
template <typename Real, int V>
__device__ __forceinline__ uint32_t swz_off(int slot, int m) {
    using T = SyncTB<Real, V>;
    const int row = slot * T::kRowsPerChunk + (m >> 3);
    return uint32_t(row * 128 + (((m & 7) ^ (row & 7)) << 4));
}

template <typename Real, int V>
__device__ __forceinline__ void chunk_from_smem(const unsigned char* buf, int slot, Real (&u)[V]) {
    using T = SyncTB<Real, V>;
#pragma unroll
    for (int m = 0; m < V / T::kPer16; ++m) {
        const unsigned char* p = buf + swz_off<Real, V>(slot, m);
        if constexpr (sizeof(Real) == 8) {
            const double2 v = *reinterpret_cast<const double2*>(p);
            u[2 * m] = v.x;
            u[2 * m + 1] = v.y;
        } else {
            const float4 v = *reinterpret_cast<const float4*>(p);
            u[4 * m] = v.x;
            u[4 * m + 1] = v.y;
            u[4 * m + 2] = v.z;
            u[4 * m + 3] = v.w;
        }
    }
}
// Stage the exact elements [el_lo, el_hi) of lane `lane`'s chunk for the TMA
// store of the tile's output units: window row w lands at row w - kHaloRows,
// so the store box starts at the (1 KB aligned) buffer start.  The halo
// bounds are multiples of 32 elements, i.e. of whole 16-B units.
template <typename Real, int V, int H = 32>
__device__ __forceinline__ void chunk_to_smem_out(unsigned char* buf, int lane, const Real (&u)[V],
                                                  int el_lo, int el_hi) {
    using T = SyncTB<Real, V, H>;
#pragma unroll
    for (int m = 0; m < V / T::kPer16; ++m) {
        const int e0 = m * T::kPer16;
        if (e0 < el_lo || e0 + T::kPer16 > el_hi) continue;
        const int row = lane * T::kRowsPerChunk + (m >> 3) - T::kHaloRows;
        unsigned char* p = buf + row * 128 + (((m & 7) ^ (row & 7)) << 4);
        if constexpr (sizeof(Real) == 8)
            *reinterpret_cast<double2*>(p) = make_double2(u[e0], u[e0 + 1]);
        else
            *reinterpret_cast<float4*>(p) = make_float4(u[e0], u[e0 + 1], u[e0 + 2], u[e0 + 3]);
    }
}

// chunk_to_smem_out with an unpredicated path for whole interior lanes
// (measured: faster for the stream kernel K5, 0.5% slower for K1).
template <typename Real, int V, int H = 32>
__device__ __forceinline__ void chunk_to_smem_out_split(unsigned char* buf, int lane,
                                                        const Real (&u)[V], int el_lo, int el_hi) {
    using T = SyncTB<Real, V, H>;
    if (el_lo != 0 || el_hi != V) {
        chunk_to_smem_out<Real, V, H>(buf, lane, u, el_lo, el_hi);
        return;
    }
#pragma unroll
    for (int m = 0; m < V / T::kPer16; ++m) {
        const int e0 = m * T::kPer16;
        const int row = lane * T::kRowsPerChunk + (m >> 3) - T::kHaloRows;
        unsigned char* p = buf + row * 128 + (((m & 7) ^ (row & 7)) << 4);
        if constexpr (sizeof(Real) == 8)
            *reinterpret_cast<double2*>(p) = make_double2(u[e0], u[e0 + 1]);
        else
            *reinterpret_cast<float4*>(p) = make_float4(u[e0], u[e0 + 1], u[e0 + 2], u[e0 + 3]);
    }
}

template <typename Real, int V>
__device__ __forceinline__ void chunk_to_smem(unsigned char* buf, int slot, const Real (&u)[V]) {
    using T = SyncTB<Real, V>;
#pragma unroll
    for (int m = 0; m < V / T::kPer16; ++m) {
        unsigned char* p = buf + swz_off<Real, V>(slot, m);
        if constexpr (sizeof(Real) == 8)
            *reinterpret_cast<double2*>(p) = make_double2(u[2 * m], u[2 * m + 1]);
        else
            *reinterpret_cast<float4*>(p) = make_float4(u[4 * m], u[4 * m + 1], u[4 * m + 2], u[4 * m + 3]);
    }
}

// One Jacobi step of a lane's V points given the neighbours' boundary
// products pL = r*u_{left of u[0]} and pR = r*u_{right of u[V-1]} (old values).
template <typename Real, int V>
__device__ __forceinline__ void chunk_step(Real (&u)[V], Real r, Real c, Real pL, Real pR,
                                           Real pFirst, Real pLast) {
    using A = Arith<Real>;
    Real pm1 = pL;
    Real p0 = pFirst;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        Real p1;
        if (i + 1 == V)
            p1 = pR;
        else if (i + 1 == V - 1)
            p1 = pLast;
        else
            p1 = A::mul(r, u[i + 1]);
        const Real cs = A::mul(c, u[i]);
        u[i] = stencil_p(p1, cs, pm1);
        pm1 = p0;
        p0 = p1;
    }
}

// Warp-cooperative step: exchange boundary products with the adjacent lanes.
template <typename Real, int V>
__device__ __forceinline__ void warp_step(Real (&u)[V], Real r, Real c) {
    const Real pFirst = Arith<Real>::mul(r, u[0]);
    const Real pLast = Arith<Real>::mul(r, u[V - 1]);
    const Real pL = __shfl_up_sync(0xffffffffu, pLast, 1);
    const Real pR = __shfl_down_sync(0xffffffffu, pFirst, 1);
    chunk_step<Real, V>(u, r, c, pL, pR, pFirst, pLast);
}

// `nsteps` warp steps, software-pipelined across the step boundary: each step
// first computes the lane's two boundary points, multiplies them by r and
// issues the shuffles the NEXT step needs, and only then computes the V-2
// interior points -- the shuffle latency hides behind them instead of
// stalling the start of every step.  Same products, same rounding sequence
// as warp_step (4 DP instructions per point).  No pinned ends allowed.
template <typename Real, int V, int PU = 2>
__device__ __forceinline__ void warp_steps_pipelined(Real (&u)[V], Real r, Real c, int nsteps) {
    static_assert(V >= 4, "pipelined step needs >= 4 points per lane");
    using A = Arith<Real>;
    Real pF = A::mul(r, u[0]);
    Real pLs = A::mul(r, u[V - 1]);
    Real pL = __shfl_up_sync(0xffffffffu, pLs, 1);
    Real pR = __shfl_down_sync(0xffffffffu, pF, 1);
#pragma unroll PU
    for (int s = 0; s < nsteps; ++s) {
        const Real p1 = A::mul(r, u[1]);        // r*u[1]   (old)
        const Real pVm2 = A::mul(r, u[V - 2]);  // r*u[V-2] (old)
        const Real nF = stencil_p(p1, A::mul(c, u[0]), pL);
        const Real nL = stencil_p(pR, A::mul(c, u[V - 1]), pVm2);
        const Real pF2 = A::mul(r, nF);
        const Real pLs2 = A::mul(r, nL);
        pL = __shfl_up_sync(0xffffffffu, pLs2, 1);  // for step s+1
        pR = __shfl_down_sync(0xffffffffu, pF2, 1);
        Real pm1 = pF, p0 = p1;
#pragma unroll
        for (int i = 1; i <= V - 2; ++i) {
            Real pn;
            if (i + 1 == V - 1)
                pn = pLs;
            else if (i + 1 == V - 2)
                pn = pVm2;
            else
                pn = A::mul(r, u[i + 1]);
            u[i] = stencil_p(pn, A::mul(c, u[i]), pm1);
            pm1 = p0;
            p0 = pn;
        }
        u[0] = nF;
        u[V - 1] = nL;
        pF = pF2;
        pLs = pLs2;
    }
}

template <typename Real, int V>
__device__ __forceinline__ void pin_ends(Real (&u)[V], long long g0, long long pin_lo,
                                         long long pin_hi, Real c1, Real c2) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const long long g = g0 + i;
        if (g == pin_lo) u[i] = c1;
        if (g == pin_hi) u[i] = c2;
    }
}

// ---- TMA tensor copies (3-D tile mode, 128B swizzle) ----------------------
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2,
                                             const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::
                     "l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// One pass over an array of `len` points.  Outputs [out_lo, out_hi) are
// advanced by `nsteps`; reads outside [0, len) wrap (single-domain periodic)
// or read as zero (their influence cannot reach the outputs in <= V steps, or
// is cut off by a pinned Dirichlet end).  pin_lo / pin_hi (or -1) are pinned
// to c1 / c2 after every step.  A whole Dirichlet domain is
// {len=N, out=[0,N), pin_lo=0, pin_hi=N-1}; a multi-GPU slab with H ghost
// points per side is {len=n+2H, out=[H,H+n), pins only at true global ends}.
// out_lo must be a multiple of V (tensor-map chunk coordinates).
struct SyncPassArgs {
    const void* src;
    void* dst;
    long long len;
    long long nchunks;  // whole V-point chunks of the array the tensor maps cover
    long long out_lo, out_hi;
    long long pin_lo, pin_hi;
    long long tiles;
    double r, c, c1, c2;  // converted to Real inside
    int wrap;
    int nsteps;
    unsigned int* nonfinite;  // set to 1 when an exact output value is not finite
    int check_finite;         // test the outputs of this pass (the last of an advance)
    unsigned long long* counter;  // DYN kernels: tile counter, zero at launch
    long long big_chunks;         // K1s: chunks of CH tiles before the single-tile tail
};

// NBUF = 2: the window of the next tile lands in the second buffer while this
//           tile is stepped; outputs are staged in the swizzled buffer and
//           leave with one TMA tensor store.
// NBUF = 1: the next tile's window lands in the (only) buffer as soon as this
//           tile is in registers; outputs leave with 16-B vector stores
//           straight from registers (half the shared memory -> more warps).
// UNR:      unroll factor of the step loop; 0 = software-pipelined steps
//           (warp_steps_pipelined) for tiles without pinned ends.
// TMA_ST: outputs leave through the window buffer with one TMA tensor store
//         (NBUF = 2 only); false: 16-B vector stores straight from registers.
// DYN:    tiles handed out by an atomic counter (grabbed as soon as the
//         current window is read) instead of a static round-robin deal.
template <typename Real, int V, int NBUF, int UNR, bool TMA_ST = true, int H = 32, bool DYN = false,
          int W = 4>
__global__ void __launch_bounds__(SyncTB<Real, V, H, W>::kThreads, SyncTB<Real, V, H, W>::min_blocks(NBUF))
    sync_tb_kernel(const __grid_constant__ CUtensorMap tm_src,
                   const __grid_constant__ CUtensorMap tm_dst, const SyncPassArgs a) {
    using T = SyncTB<Real, V, H, W>;
    static_assert(NBUF == 1 || NBUF == 2, "one or two window buffers per warp");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 128B swizzle needs 1024-B aligned buffers
    // aligned by an offset from the __shared__ array itself: a round trip
    // through uintptr_t loses the address space (generic LD/ST, ptxas SASS)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const Real* __restrict__ src = static_cast<const Real*>(a.src);
    Real* __restrict__ dst = static_cast<Real*>(a.dst);
    const long long len = a.len;
    const Real r = Real(a.r), c = Real(a.c), c1 = Real(a.c1), c2 = Real(a.c2);
    const bool wrap = a.wrap != 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + warp * NBUF * T::kBufBytes;
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem + T::kWarpsPerCta * NBUF * T::kBufBytes) + 2 * warp;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        if (warp == 0) {
            tma_prefetch_desc(&tm_src);
            if (NBUF == 2) tma_prefetch_desc(&tm_dst);
        }
    }
    __syncwarp();

    const long long nwarps = (long long)gridDim.x * T::kWarpsPerCta;
    const long long tma_len = a.nchunks * T::kUnit;  // points the tensor maps cover
    auto window = [&](long long t) { return a.out_lo + t * T::kOut - T::kHalo; };
    auto in_window = [&](long long g, long long w0) {
        return g >= 0 && g >= w0 && g < w0 + kWarp * V;
    };
    // TMA fast path: whole window inside the tensor, no pinned point inside.
    auto interior = [&](long long t) {
        const long long w0 = window(t);
        return w0 >= 0 && w0 + kWarp * V <= tma_len && !in_window(a.pin_lo, w0) &&
               !in_window(a.pin_hi, w0);
    };
    auto bufp = [&](int b) { return wbase + b * T::kBufBytes; };
    auto issue = [&](int b, long long t) {
        fence_proxy_async_smem();  // this lane's generic accesses to the buffer come first
        __syncwarp();
        if (lane == 0) {
            if (NBUF == 2 && TMA_ST) bulk_wait_read_all();  // the TMA store that last used it has read it
            mbar_arrive_expect_tx(&bars[b], T::kBufBytes);
            tma_load_3d(bufp(b), &tm_src, 0, 0, int(window(t) / T::kUnit), &bars[b]);
        }
    };

    uint32_t phase = 0;
    bool bad = false;
    auto grab = [&]() -> long long {
        unsigned long long i = 0;
        if (lane == 0) i = atomicAdd(a.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, i, 0);
    };
    long long t = DYN ? grab() : (long long)blockIdx.x * T::kWarpsPerCta + warp;
    if (t < a.tiles && interior(t)) issue(0, t);
    for (int it = 0; t < a.tiles; ++it) {
        // DYN: the next tile's index -- the atomic is issued now and read once
        // this window is in, so its latency hides behind the window wait
        unsigned long long nraw = 0;
        if (DYN && lane == 0) nraw = atomicAdd(a.counter, 1ull);
        const int b = NBUF == 2 ? (it & 1) : 0;
        unsigned char* buf = bufp(b);
        const long long w0 = window(t);
        const bool inter = interior(t);
        const long long g0 = w0 + (long long)lane * V;
        Real u[V];
        if (inter) {
            mbar_wait(&bars[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            chunk_from_smem<Real, V>(buf, lane, u);
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                long long g = g0 + i;
                if (wrap) {
                    g %= len;
                    if (g < 0) g += len;
                    u[i] = src[g];
                } else {
                    u[i] = (g >= 0 && g < len) ? src[g] : Real(0);
                }
            }
        }
        const long long tn = DYN ? (long long)__shfl_sync(0xffffffffu, nraw, 0) : t + nwarps;
        if (tn < a.tiles && interior(tn)) issue(NBUF == 2 ? (b ^ 1) : 0, tn);

        if (inter || (!in_window(a.pin_lo, w0) && !in_window(a.pin_hi, w0))) {
            if constexpr (UNR <= 0) {  // pipelined steps, unrolled 2 (UNR = 0) or -UNR
                warp_steps_pipelined<Real, V, (UNR == 0 ? 2 : -UNR)>(u, r, c, a.nsteps);
            } else {
#pragma unroll UNR
                for (int s = 0; s < a.nsteps; ++s) warp_step<Real, V>(u, r, c);
            }
        } else {
            for (int s = 0; s < a.nsteps; ++s) {
                warp_step<Real, V>(u, r, c);
                pin_ends<Real, V>(u, g0, a.pin_lo, a.pin_hi, c1, c2);
            }
        }

        // exact elements of this lane: window points [kHalo, 32V - kHalo)
        const int el_lo = min(V, max(0, T::kHalo - lane * V));
        const int el_hi = min(V, max(0, kWarp * V - T::kHalo - lane * V));
        // Finite check only on the last pass of an advance: a non-finite value
        // at a non-pinned point never becomes finite again (c*NaN = NaN,
        // c*(+-Inf) = +-Inf or NaN), so the outcome of the reference's per-step
        // check (sync_solver.cpp:11-17) is decided by the final state.
        if (a.check_finite) {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi && g0 + i < a.out_hi && !isfinite(u[i])) bad = true;
        }
        const bool full = w0 + kWarp * V - T::kHalo <= a.out_hi;
        if (NBUF == 2 && TMA_ST && inter && full) {
            // stage the exact units as a [kOutUnits x rows] box at the buffer start
            chunk_to_smem_out<Real, V, H>(buf, lane, u, el_lo, el_hi);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_3d(&tm_dst, 0, 0, int((w0 + T::kHalo) / T::kUnit), buf);
                bulk_commit();
            }
        } else if (full && g0 >= 0) {
            // whole exact 16-B units in range: vector stores from registers
#pragma unroll
            for (int m = 0; m < V / T::kPer16; ++m) {
                const int e0 = m * T::kPer16;
                if (e0 < el_lo || e0 + T::kPer16 > el_hi) continue;
                if constexpr (sizeof(Real) == 8)
                    reinterpret_cast<double2*>(dst + g0)[m] = make_double2(u[e0], u[e0 + 1]);
                else
                    reinterpret_cast<float4*>(dst + g0)[m] =
                        make_float4(u[e0], u[e0 + 1], u[e0 + 2], u[e0 + 3]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi && g0 + i < a.out_hi) dst[g0 + i] = u[i];
        }
        t = tn;
    }
    if (NBUF == 2 && TMA_ST && lane == 0) bulk_wait_all();
    if (bad) atomicOr(a.nonfinite, 1u);
}

}  // namespace hb
