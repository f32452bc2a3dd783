// sync_col.cuh -- K1s: temporal-blocked synchronous pass over STRIPS of
// tiles with a carried boundary column (the same update as K1, sync_tb.cuh;
// replaces sync_step_into, sync_solver.hpp:26-39, iterated by run_impl,
// sync_solver.cpp:70-75).
//
// K1 recomputes an H-point halo on BOTH sides of every warp tile: 1408 of
// 1536 points per 48x64 tile are exact.  Here a warp steps a chunk of CH
// consecutive tiles left to right.  The first tile of a chunk is a K1 tile
// (left and right halo, E0 = 32V - 2H exact points).  While stepping it, the
// lane holding its last exact point stores that point's product r*u at every
// time level into a shared-memory COLUMN.  The next tile's window starts at
// its first output point: its lane 0 takes the left neighbour product of each
// step from the column instead of a halo, so it needs only the right halo and
// emits E1 = 32V - H exact points (1472 of 1536), and it writes its own column
// for the tile after it.  Chunks are dealt by an atomic counter (one grab per
// chunk); at CH = 8, 11712 of every 12288 points a chunk steps are exact
// (95.3% against K1's 91.7%).  The last few tiles per warp of a pass are dealt
// one by one (plain K1 tiles), so warps finish within one tile of each other.
// Every value is the same stencil_p of the same products: bit-identical to K1.
#pragma once

#include "sync_tb.cuh"

namespace hb {

template <typename Real, int V, int H, int CH>
struct SyncCol {
    using T = SyncTB<Real, V, H>;
    static constexpr int kW = kWarp * V;            // window points
    static constexpr int kE0 = kW - 2 * H;           // exact points of a chunk's first tile
    static constexpr int kE1 = kW - H;               // ... of the tiles after it
    static constexpr int kChunkOut = kE0 + (CH - 1) * kE1;
    static constexpr int kLastPos = H + kE0 - 1;     // window position of a tile's last output
    static constexpr int kPL = kLastPos / V, kPE = kLastPos % V;  // its lane and element
    static constexpr int kOut0Units = kE0 / T::kUnit, kOut1Units = kE1 / T::kUnit;
    static constexpr int kColBytes = 2 * H * int(sizeof(Real));  // two columns of H products
    static constexpr int smem_bytes() {
        return T::kWarpsPerCta * (2 * T::kBufBytes + kColBytes + 2 * 8) + 1024;
    }
    static_assert(kE1 - 1 == kLastPos, "both tile kinds end at the same window position");
    // (the pipelined step takes element PE's product as pn of interior point
    // PE-1: PE = V-2 is pVm2 and PE = V-1 is the lane's last product pLs)
    static_assert(kPE >= 2 && kPE <= V - 1, "the column point is a pn of the step");
    static_assert(kE0 % T::kUnit == 0 && kE1 % T::kUnit == 0, "outputs of whole units");
};

// K1's software-pipelined steps, with the chunk's column: lane 0 takes its
// left neighbour product from colr (null: a chunk's first tile, which has a
// left halo instead), and lane kPL stores its element kPE's product of every
// time level into colw.
// Steps s0 .. s1-1 of the tile (the column index is the step).
template <typename Real, int V, int PU, int PE>
__device__ __forceinline__ void warp_steps_col(Real (&u)[V], Real r, Real c, int s0, int s1,
                                               const Real* colr, Real* colw, bool wlane,
                                               int lane) {
    using A = Arith<Real>;
    Real pF = A::mul(r, u[0]);
    Real pLs = A::mul(r, u[V - 1]);
    Real pL = __shfl_up_sync(0xffffffffu, pLs, 1);
    Real pR = __shfl_down_sync(0xffffffffu, pF, 1);
    const bool rd = colr != nullptr && lane == 0;
    // the column value of the next step is loaded beside its shuffle and
    // selected only where the step uses it (selecting at once would wait for
    // the shuffle: -2.8%, ncu short_sb)
    Real pLc = rd ? colr[s0] : Real(0);
#pragma unroll PU
    for (int s = s0; s < s1; ++s) {
        const Real p1 = A::mul(r, u[1]);
        const Real pVm2 = A::mul(r, u[V - 2]);
        const Real nF = stencil_p(p1, A::mul(c, u[0]), rd ? pLc : pL);
        const Real nL = stencil_p(pR, A::mul(c, u[V - 1]), pVm2);
        const Real pF2 = A::mul(r, nF);
        const Real pLs2 = A::mul(r, nL);
        pL = __shfl_up_sync(0xffffffffu, pLs2, 1);  // for step s+1
        pR = __shfl_down_sync(0xffffffffu, pF2, 1);
        if (rd && s + 1 < s1) pLc = colr[s + 1];
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
            if (i + 1 == PE && wlane) colw[s] = pn;  // r*u[PE] at time s
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

// MID: issue the next tile's TMA load half way through this tile's steps
// instead of right after its window is read.  The load goes into the other
// buffer, whose last TMA store (the previous tile's output) must have read
// it first: right after the window read that store was only just committed.
template <typename Real, int V, int H, int CH, int PU, bool MID = false>
__global__ void __launch_bounds__(SyncTB<Real, V, H>::kThreads, V <= 32 ? 3 : 2)
    sync_col_kernel(const __grid_constant__ CUtensorMap tm_src,
                    const __grid_constant__ CUtensorMap tm_dst0,
                    const __grid_constant__ CUtensorMap tm_dst1, const SyncPassArgs a) {
    using T = SyncTB<Real, V, H>;
    using K = SyncCol<Real, V, H, CH>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const Real* __restrict__ src = static_cast<const Real*>(a.src);
    Real* __restrict__ dst = static_cast<Real*>(a.dst);
    const long long len = a.len;
    const Real r = Real(a.r), c = Real(a.c), c1 = Real(a.c1), c2 = Real(a.c2);
    const bool wrap = a.wrap != 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + warp * 2 * T::kBufBytes;
    Real* cols = reinterpret_cast<Real*>(smem + T::kWarpsPerCta * 2 * T::kBufBytes) +
                 warp * 2 * H;  // [2][H]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::kWarpsPerCta * (2 * T::kBufBytes +
                                                                           K::kColBytes)) +
                     2 * warp;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        if (warp == 0) {
            tma_prefetch_desc(&tm_src);
            tma_prefetch_desc(&tm_dst0);
            tma_prefetch_desc(&tm_dst1);
        }
    }
    __syncwarp();

    const long long tma_len = a.nchunks * T::kUnit;
    // tile (chunk ch, index i): its first output and its window start.  The
    // first a.big_chunks chunks hold CH tiles; the rest of the range is dealt
    // as single K1 tiles, so the pass does not end waiting for whole chunks
    auto out_start = [&](long long ch, int i) {
        if (ch >= a.big_chunks)
            return a.out_lo + a.big_chunks * K::kChunkOut + (ch - a.big_chunks) * K::kE0;
        return a.out_lo + ch * K::kChunkOut + (i == 0 ? 0 : K::kE0 + (long long)(i - 1) * K::kE1);
    };
    auto win_start = [&](long long ch, int i) { return out_start(ch, i) - (i == 0 ? H : 0); };
    auto in_window = [&](long long g, long long w0) { return g >= 0 && g >= w0 && g < w0 + K::kW; };
    auto interior = [&](long long w0) {
        return w0 >= 0 && w0 + K::kW <= tma_len && !in_window(a.pin_lo, w0) &&
               !in_window(a.pin_hi, w0);
    };
    auto bufp = [&](int b) { return wbase + b * T::kBufBytes; };
    auto issue = [&](int b, long long w0) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            bulk_wait_read_all();  // the TMA store that last used this buffer has read it
            mbar_arrive_expect_tx(&bars[b], T::kBufBytes);
            tma_load_3d(bufp(b), &tm_src, 0, 0, int(w0 / T::kUnit), &bars[b]);
        }
    };
    auto grab = [&]() -> long long {
        unsigned long long x = 0;
        if (lane == 0) x = atomicAdd(a.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, x, 0);
    };

    uint32_t phase = 0;
    bool bad = false;
    long long ch = grab();
    int ti = 0;
    if (ch < a.tiles && interior(win_start(ch, 0))) issue(0, win_start(ch, 0));
    for (int it = 0; ch < a.tiles; ++it) {
        const long long o0 = out_start(ch, ti);
        const long long w0 = win_start(ch, ti);
        const long long o1 = min(o0 + (ti == 0 ? K::kE0 : K::kE1), a.out_hi);
        // the next tile: this chunk's next one, or the first of the next chunk
        const bool more = ch < a.big_chunks && ti + 1 < CH && out_start(ch, ti + 1) < a.out_hi;
        unsigned long long nraw = 0;
        if (!more && lane == 0) nraw = atomicAdd(a.counter, 1ull);  // read after the window wait
        const int b = it & 1;
        unsigned char* buf = bufp(b);
        const bool inter = interior(w0);
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
        const long long nch = more ? ch : (long long)__shfl_sync(0xffffffffu, nraw, 0);
        const int nti = more ? ti + 1 : 0;
        const bool next_tma = nch < a.tiles && interior(win_start(nch, nti));
        const bool plain_steps = !(inter || (!in_window(a.pin_lo, w0) && !in_window(a.pin_hi, w0)));
        if (next_tma && (!MID || plain_steps)) issue(b ^ 1, win_start(nch, nti));

        const Real* colr = ti == 0 ? nullptr : cols + ((ti - 1) & 1) * H;
        Real* colw = cols + (ti & 1) * H;
        const bool wlane = lane == K::kPL;
        if (!plain_steps) {
            if (MID) {
                const int half = a.nsteps / 2;
                warp_steps_col<Real, V, PU, K::kPE>(u, r, c, 0, half, colr, colw, wlane, lane);
                if (next_tma) issue(b ^ 1, win_start(nch, nti));
                warp_steps_col<Real, V, PU, K::kPE>(u, r, c, half, a.nsteps, colr, colw, wlane,
                                                    lane);
            } else {
                warp_steps_col<Real, V, PU, K::kPE>(u, r, c, 0, a.nsteps, colr, colw, wlane, lane);
            }
        } else {
            for (int s = 0; s < a.nsteps; ++s) {
                const Real pFirst = Arith<Real>::mul(r, u[0]);
                const Real pLast = Arith<Real>::mul(r, u[V - 1]);
                Real pL = __shfl_up_sync(0xffffffffu, pLast, 1);
                const Real pR = __shfl_down_sync(0xffffffffu, pFirst, 1);
                if (colr && lane == 0) pL = colr[s];
                if (wlane) colw[s] = Arith<Real>::mul(r, u[K::kPE]);
                chunk_step<Real, V>(u, r, c, pL, pR, pFirst, pLast);
                pin_ends<Real, V>(u, g0, a.pin_lo, a.pin_hi, c1, c2);
            }
        }
        __syncwarp();  // this tile's column is complete before the next tile reads it

        // exact elements of this lane: window points [o0 - w0, o1 - w0)
        const int lo_pos = int(o0 - w0), hi_pos = int(o1 - w0);
        const int el_lo = min(V, max(0, lo_pos - lane * V));
        const int el_hi = min(V, max(0, hi_pos - lane * V));
        if (a.check_finite) {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi && !isfinite(u[i])) bad = true;
        }
        const bool full = o1 == o0 + (ti == 0 ? K::kE0 : K::kE1);
        if (inter && full) {
            if (ti == 0) {  // exact units start kHalo into the window: staged row-shifted
                chunk_to_smem_out<Real, V, H>(buf, lane, u, el_lo, el_hi);
            } else {        // exact units start at the window
#pragma unroll
                for (int m = 0; m < V / T::kPer16; ++m) {
                    const int e0 = m * T::kPer16;
                    if (e0 < el_lo || e0 + T::kPer16 > el_hi) continue;
                    const int row = lane * T::kRowsPerChunk + (m >> 3);
                    unsigned char* p = buf + row * 128 + (((m & 7) ^ (row & 7)) << 4);
                    *reinterpret_cast<double2*>(p) = make_double2(u[e0], u[e0 + 1]);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (ti == 0)
                    tma_store_3d(&tm_dst0, 0, 0, int(o0 / T::kUnit), buf);
                else
                    tma_store_3d(&tm_dst1, 0, 0, int(o0 / T::kUnit), buf);
                bulk_commit();
            }
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi) dst[g0 + i] = u[i];
        }
        ch = nch;
        ti = nti;
    }
    if (lane == 0) bulk_wait_all();
    if (bad) atomicOr(a.nonfinite, 1u);
}

}  // namespace hb
