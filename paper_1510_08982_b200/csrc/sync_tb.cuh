// sync_tb.cuh -- K1: temporal-blocked synchronous FTCS pass for sm_100a.
//
// Replaces detail::sync_step_into (sync_solver.hpp:26-39) iterated by
// run_impl (sync_solver.cpp:70-75) and run_barriered (async_exec.cpp:57-114):
// one launch advances the whole field by `nsteps` (<= V) Jacobi steps.
//
// Layout / mapping
//   * A WARP owns one tile: 32 lanes x V consecutive points (a "window" of
//     32V points).  Lane l holds points [w0 + lV, w0 + (l+1)V) in registers.
//   * Neighbour values inside a lane are registers; across lanes one
//     __shfl_up / __shfl_down of the boundary PRODUCT r*u per step.
//   * Lanes 0 and 31 are halo (redundant recompute).  After s <= V steps
//     lanes 1..30 are exact, so a tile emits 30V points: tile t covers
//     outputs [30Vt, 30V(t+1)), window start w0 = 30Vt - V.
//   * No block barrier anywhere: warps are independent.  Each warp
//     double-buffers its window in shared memory: a 1-D TMA bulk copy
//     (cp.async.bulk, one V-point chunk per lane, padded by 16 B so the
//     per-lane 16-B shared loads are bank-conflict free) lands the NEXT tile
//     while the current one is being stepped; results go back through the
//     same padded buffer with cp.async.bulk shared->global.
//   * Tiles whose window touches a domain end (or is not 16-B aligned / in
//     bounds) take the generic path: coalesced element loads with zero fill
//     (Dirichlet) or modular wrap (periodic), Dirichlet ends re-pinned after
//     every step, bounds-checked stores.
//
// HBM traffic per pass: read 32V + write 30V points per 30V*s updates, i.e.
// ~16.5/s bytes per lattice update (0.52 B at s = 32) -- the pass is bound by
// the FP64 pipe (4 DP instructions per update), not by HBM.
#pragma once

#include "common.cuh"

namespace hb {

template <typename Real, int V>
struct SyncTB {
    static constexpr int kChunkBytes = V * int(sizeof(Real));
    static constexpr int kStrideBytes = kChunkBytes + 16;
    static constexpr int kStrideElems = kStrideBytes / int(sizeof(Real));
    static constexpr int kBufBytes = kWarp * kStrideBytes;
    static constexpr int kOut = (kWarp - 2) * V;  // exact points per tile
    static constexpr int kWarpsPerCta = 4;
    static constexpr int kThreads = kWarpsPerCta * kWarp;
    static constexpr int kSmemBytes = kWarpsPerCta * 2 * kBufBytes + kWarpsPerCta * 2 * 8;
    static constexpr int kMaxSteps = V;  // halo of one lane per side
    static_assert((V * sizeof(Real)) % 16 == 0, "chunk must be a multiple of 16 B");
};

// Padded shared chunk <-> registers, 16-byte vector accesses.
template <typename Real, int V>
__device__ __forceinline__ void chunk_from_smem(const Real* p, Real (&u)[V]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int m = 0; m < V / 2; ++m) {
            double2 v = reinterpret_cast<const double2*>(p)[m];
            u[2 * m] = v.x;
            u[2 * m + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int m = 0; m < V / 4; ++m) {
            float4 v = reinterpret_cast<const float4*>(p)[m];
            u[4 * m] = v.x;
            u[4 * m + 1] = v.y;
            u[4 * m + 2] = v.z;
            u[4 * m + 3] = v.w;
        }
    }
}
template <typename Real, int V>
__device__ __forceinline__ void chunk_to_smem(Real* p, const Real (&u)[V]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int m = 0; m < V / 2; ++m)
            reinterpret_cast<double2*>(p)[m] = make_double2(u[2 * m], u[2 * m + 1]);
    } else {
#pragma unroll
        for (int m = 0; m < V / 4; ++m)
            reinterpret_cast<float4*>(p)[m] =
                make_float4(u[4 * m], u[4 * m + 1], u[4 * m + 2], u[4 * m + 3]);
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

// One pass over an array of `len` points.  Outputs [out_lo, out_hi) are
// advanced by `nsteps`; reads outside [0, len) wrap (single-domain periodic)
// or read as zero (their influence cannot reach the outputs in <= V steps, or
// is cut off by a pinned Dirichlet end).  pin_lo / pin_hi (or -1) are pinned
// to c1 / c2 after every step.  A whole Dirichlet domain is
// {len=N, out=[0,N), pin_lo=0, pin_hi=N-1}; a multi-GPU slab with H ghost
// points per side is {len=n+2H, out=[H,H+n), pins only at true global ends}.
struct SyncPassArgs {
    const void* src;
    void* dst;
    long long len;
    long long out_lo, out_hi;
    long long pin_lo, pin_hi;
    long long tiles;
    double r, c, c1, c2;  // converted to Real inside
    int wrap;
    int nsteps;
    unsigned int* nonfinite;  // set to 1 when an exact output value is not finite
};

template <typename Real, int V>
__global__ void __launch_bounds__(SyncTB<Real, V>::kThreads)
    sync_tb_kernel(const SyncPassArgs a) {
    using T = SyncTB<Real, V>;
    extern __shared__ __align__(128) unsigned char smem[];
    const Real* __restrict__ src = static_cast<const Real*>(a.src);
    Real* __restrict__ dst = static_cast<Real*>(a.dst);
    const long long len = a.len;
    const Real r = Real(a.r), c = Real(a.c), c1 = Real(a.c1), c2 = Real(a.c2);
    const bool wrap = a.wrap != 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + warp * 2 * T::kBufBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::kWarpsPerCta * 2 * T::kBufBytes) + 2 * warp;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const long long nwarps = (long long)gridDim.x * T::kWarpsPerCta;
    auto window = [&](long long t) { return a.out_lo + t * T::kOut - V; };
    auto in_window = [&](long long g, long long w0) { return g >= 0 && g >= w0 && g < w0 + kWarp * V; };
    // Bulk-copy fast path: window in bounds, 16-B aligned, no pinned point inside.
    auto interior = [&](long long t) {
        const long long w0 = window(t);
        return w0 >= 0 && w0 + kWarp * V <= len && ((w0 * (long long)sizeof(Real)) & 15) == 0 &&
               !in_window(a.pin_lo, w0) && !in_window(a.pin_hi, w0);
    };
    auto bufp = [&](int b) { return reinterpret_cast<Real*>(wbase + b * T::kBufBytes); };
    auto issue = [&](int b, long long t) {
        bulk_wait_read_all();      // this lane's earlier bulk stores have left the buffer
        fence_proxy_async_smem();  // and its generic accesses are ordered before the copy
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&bars[b], kWarp * T::kChunkBytes);
        __syncwarp();
        bulk_g2s(bufp(b) + lane * T::kStrideElems, src + window(t) + (long long)lane * V,
                 T::kChunkBytes, &bars[b]);
    };

    uint32_t phase = 0;
    bool bad = false;
    long long t = (long long)blockIdx.x * T::kWarpsPerCta + warp;
    if (t < a.tiles && interior(t)) issue(0, t);
    for (int it = 0; t < a.tiles; ++it, t += nwarps) {
        const int b = it & 1;
        Real* buf = bufp(b);
        const long long w0 = window(t);
        const bool inter = interior(t);
        Real u[V];
        if (inter) {
            mbar_wait(&bars[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            chunk_from_smem<Real, V>(buf + lane * T::kStrideElems, u);
        } else {
            bulk_wait_read_all();
            __syncwarp();
            for (int j = lane; j < kWarp * V; j += kWarp) {
                long long g = w0 + j;
                Real v;
                if (wrap) {
                    g %= len;
                    if (g < 0) g += len;
                    v = src[g];
                } else {
                    v = (g >= 0 && g < len) ? src[g] : Real(0);
                }
                buf[(j / V) * T::kStrideElems + (j % V)] = v;
            }
            __syncwarp();
            chunk_from_smem<Real, V>(buf + lane * T::kStrideElems, u);
        }
        const long long tn = t + nwarps;
        if (tn < a.tiles && interior(tn)) issue(b ^ 1, tn);

        if (inter || (!in_window(a.pin_lo, w0) && !in_window(a.pin_hi, w0))) {
            for (int s = 0; s < a.nsteps; ++s) warp_step<Real, V>(u, r, c);
        } else {
            const long long g0 = w0 + (long long)lane * V;
            for (int s = 0; s < a.nsteps; ++s) {
                warp_step<Real, V>(u, r, c);
                pin_ends<Real, V>(u, g0, a.pin_lo, a.pin_hi, c1, c2);
            }
        }

        if (lane >= 1 && lane <= kWarp - 2) {
            const long long g0 = w0 + (long long)lane * V;
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (g0 + i < a.out_hi && !isfinite(u[i])) bad = true;
        }
        __syncwarp();
        chunk_to_smem<Real, V>(buf + lane * T::kStrideElems, u);
        if (inter && w0 + (kWarp - 1) * V <= a.out_hi) {
            fence_proxy_async_smem();
            if (lane >= 1 && lane <= kWarp - 2) {
                bulk_s2g(dst + w0 + (long long)lane * V, buf + lane * T::kStrideElems,
                         T::kChunkBytes);
                bulk_commit();
            }
        } else {
            __syncwarp();
            for (int j = V + lane; j < (kWarp - 1) * V; j += kWarp) {
                const long long g = w0 + j;
                if (g < a.out_hi) dst[g] = buf[(j / V) * T::kStrideElems + (j % V)];
            }
            __syncwarp();
        }
    }
    bulk_wait_all();
    if (bad) atomicOr(a.nonfinite, 1u);
}

}  // namespace hb
