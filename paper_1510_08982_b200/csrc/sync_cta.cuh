// sync_cta.cuh -- K1c: temporal-blocked synchronous FTCS pass with CTA-wide
// windows (the same update as K1, sync_tb.cuh; replaces sync_step_into,
// sync_solver.hpp:26-39, iterated by run_impl, sync_solver.cpp:70-75).
//
// K1 gives every warp its own 32V-point window with an H-point halo on each
// side: at 48 x 64 only 1408 of 1536 points per tile are exact, so 8.3% of
// the FP64 work is redundant halo recompute.  K1c lets the G warps of a CTA
// step ONE window of G x 32V points together: warp w holds points
// [w*32V, (w+1)*32V) of it, lanes exchange boundary products by shuffles as
// in K1, and the two lanes at a warp seam exchange theirs through shared
// memory once per step.  The halo is paid once per CTA window: at G = 4,
// V = 48, H = 64 a tile emits 6016 of 6144 points (97.9% exact).
//
// Seam exchange without barriers: a slot is two 64-bit words
// {tag : 32 | half of the double : 32} (an aligned 64-bit shared store is
// single-copy atomic), so a reader that sees its expected tag in both words
// has the whole value -- no fence, no flag, no block barrier per step.  The
// tag is a per-CTA running count of exchanges; every warp of a CTA makes the
// same exchanges in the same order.  A warp publishes the products of step
// s+1 right after computing its two end points (before its V-2 interior
// points) and reads its neighbours' only at the end of the step, so the
// exchange latency hides behind the interior work.  Slots form a ring of 4:
// a producer can be at most one exchange ahead of a consumer that has not yet
// read (it needs the consumer's own product of the same exchange first), and
// tiles are separated by block barriers.
//
// Data movement: the CTA window is ONE TMA tensor load (G*32V points) into a
// 128B-swizzled buffer (two buffers: the next tile's window lands while this
// one is stepped); outputs are staged row-shifted by the halo into the same
// buffer and leave with ONE TMA tensor store of the CTA's exact units.
// Tiles are dealt to CTAs by an atomic counter.  Tiles whose window touches a
// pinned end or leaves the tensor take the generic path (element loads with
// zero fill / wrap, per-step pins, bounds-checked stores) with the same seam
// exchange.
#pragma once

#include "sync_tb.cuh"

namespace hb {

template <typename Real, int V, int H, int G>
struct SyncCTA {
    using T = SyncTB<Real, V, H, G>;
    static constexpr int kWin = G * kWarp * V;            // points per CTA window
    static constexpr int kOut = kWin - 2 * H;              // exact points per tile
    static constexpr int kWinUnits = kWin / T::kUnit;
    static constexpr int kOutUnits = kOut / T::kUnit;
    static constexpr int kBufBytes = G * T::kBufBytes;     // one CTA window
    static constexpr int kRing = 4;                        // seam slots per (warp, side)
    static constexpr int kXchBytes = kRing * G * 2 * 16 + 16;  // ring, dummy slot
    static constexpr int smem_bytes() { return 2 * kBufBytes + 2 * 8 + 16 + kXchBytes + 1024; }
    static_assert(kWinUnits <= 256 && kOutUnits <= 256, "TMA boxes are at most 256 units");
    static_assert(kBufBytes % 1024 == 0, "window buffers keep the 1 KB swizzle alignment");
};

// Seam slot I/O (shared memory, volatile: the compiler re-reads every poll).
__device__ __forceinline__ void seam_put(uint32_t addr, uint32_t tag, double v) {
    const unsigned long long lo = (unsigned long long)tag << 32 | uint32_t(__double2loint(v));
    const unsigned long long hi = (unsigned long long)tag << 32 | uint32_t(__double2hiint(v));
    asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(lo), "l"(hi)
                 : "memory");
}
__device__ __forceinline__ double seam_get(uint32_t addr, uint32_t tag) {
    unsigned long long lo, hi;
    do {
        asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                     : "=l"(lo), "=l"(hi)
                     : "r"(addr)
                     : "memory");
    } while (uint32_t(lo >> 32) != tag || uint32_t(hi >> 32) != tag);
    return __hiloint2double(int(uint32_t(hi)), int(uint32_t(lo)));
}


// The seam roles of one lane: lane 0 of warp w > 0 reads its left product
// from warp w-1's lane 31 and publishes its own first product; lane 31 of
// warp w < G-1 mirrors it.  put/get are byte offsets into the slot ring.
struct Seam {
    uint32_t xch;   // shared address of the ring [kRing][G][2 sides] x 16 B
    uint32_t put;   // this lane's own slot in ring entry 0 (a dummy slot if it
                    // does not publish: the store stays unconditional)
    uint32_t get;   // the neighbour's slot it reads (if it reads)
    bool pub, rd;
    uint32_t tag;
    __device__ __forceinline__ uint32_t entry(uint32_t t, int G) const {
        return (t & 3u) * uint32_t(G * 2 * 16);
    }
};

// One exchange: publish this lane's end product (lane 0: first, lane 31:
// last) under the next tag.  Reading is separate (seam_read).
template <int G>
__device__ __forceinline__ void seam_publish(Seam& s, double pFirstOrLast) {
    ++s.tag;
    seam_put(s.xch + (s.pub ? s.entry(s.tag, G) : 0u) + s.put, s.tag, pFirstOrLast);
}
// The whole warp polls until lanes 0 / 31 have their neighbours' products
// (the others read their own dummy slot and are satisfied at once): a loop
// that only some lanes run would leave the warp diverged, and every later
// shuffle would take the slow collective path (measured: 3x slower).
template <int G>
__device__ __forceinline__ double seam_read(const Seam& s, double fallback) {
    const uint32_t addr = s.rd ? s.xch + s.entry(s.tag, G) + s.get : s.xch + s.put;
    while (true) {
        unsigned long long lo, hi;
        asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                     : "=l"(lo), "=l"(hi)
                     : "r"(addr)
                     : "memory");
        const bool ok = !s.rd || (uint32_t(lo >> 32) == s.tag && uint32_t(hi >> 32) == s.tag);
        if (__all_sync(0xffffffffu, ok))
            return s.rd ? __hiloint2double(int(uint32_t(hi)), int(uint32_t(lo))) : fallback;
    }
}

// nsteps software-pipelined steps (K1's warp_steps_pipelined) of a warp whose
// window continues in the neighbouring warps: lanes 0 / 31 take their outer
// products from the seam slots instead of the shuffle.
template <typename Real, int V, int G, int PU>
__device__ __forceinline__ void cta_steps_pipelined(Real (&u)[V], Real r, Real c, int nsteps,
                                                    Seam& sm, int lane) {
    using A = Arith<Real>;
    Real pF = A::mul(r, u[0]);
    Real pLs = A::mul(r, u[V - 1]);
    Real pL = __shfl_up_sync(0xffffffffu, pLs, 1);
    Real pR = __shfl_down_sync(0xffffffffu, pF, 1);
    seam_publish<G>(sm, lane == 0 ? pF : pLs);
    {
        const Real x = seam_read<G>(sm, lane == 0 ? pL : pR);
        if (lane == 0) pL = x; else pR = x;
    }
#pragma unroll PU
    for (int s = 0; s < nsteps; ++s) {
        const Real p1 = A::mul(r, u[1]);
        const Real pVm2 = A::mul(r, u[V - 2]);
        const Real nF = stencil_p(p1, A::mul(c, u[0]), pL);
        const Real nL = stencil_p(pR, A::mul(c, u[V - 1]), pVm2);
        const Real pF2 = A::mul(r, nF);
        const Real pLs2 = A::mul(r, nL);
        pL = __shfl_up_sync(0xffffffffu, pLs2, 1);  // for step s+1
        pR = __shfl_down_sync(0xffffffffu, pF2, 1);
        seam_publish<G>(sm, lane == 0 ? pF2 : pLs2);
        // ptxas sinks this store below the interior work whatever the source
        // order (arithmetic moves freely across stores), so the neighbour
        // reads it only after our interior.  Forcing the order with a
        // volatile shared reload of r and c after the store (an LDS the
        // interior depends on) measured slower: 3616 vs 3760 GLUPS.
        const Real ri = r, ci = c;
        Real pm1 = pF, p0 = p1;
#pragma unroll
        for (int i = 1; i <= V - 2; ++i) {
            Real pn;
            if (i + 1 == V - 1)
                pn = pLs;
            else if (i + 1 == V - 2)
                pn = pVm2;
            else
                pn = A::mul(ri, u[i + 1]);
            u[i] = stencil_p(pn, A::mul(ci, u[i]), pm1);
            pm1 = p0;
            p0 = pn;
        }
        u[0] = nF;
        u[V - 1] = nL;
        pF = pF2;
        pLs = pLs2;
        if (s + 1 < nsteps) {
            const Real x = seam_read<G>(sm, lane == 0 ? pL : pR);
            if (lane == 0) pL = x; else pR = x;
        }
    }
}

// Plain (non-pipelined) step with the seam exchange, for the generic tiles.
template <typename Real, int V, int G>
__device__ __forceinline__ void cta_step(Real (&u)[V], Real r, Real c, Seam& sm, int lane) {
    const Real pFirst = Arith<Real>::mul(r, u[0]);
    const Real pLast = Arith<Real>::mul(r, u[V - 1]);
    Real pL = __shfl_up_sync(0xffffffffu, pLast, 1);
    Real pR = __shfl_down_sync(0xffffffffu, pFirst, 1);
    seam_publish<G>(sm, lane == 0 ? pFirst : pLast);
    const Real x = seam_read<G>(sm, lane == 0 ? pL : pR);
    if (lane == 0) pL = x; else pR = x;
    chunk_step<Real, V>(u, r, c, pL, pR, pFirst, pLast);
}

template <typename Real, int V, int H, int G, int PU>
__global__ void __launch_bounds__(G * kWarp, 2)
    sync_cta_kernel(const __grid_constant__ CUtensorMap tm_src,
                    const __grid_constant__ CUtensorMap tm_dst, const SyncPassArgs a) {
    using T = SyncTB<Real, V, H, G>;
    using C = SyncCTA<Real, V, H, G>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB alignment by an offset from the __shared__ array itself (a round
    // trip through uintptr_t loses the address space: generic LD/ST)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * C::kBufBytes);
    long long* s_next = reinterpret_cast<long long*>(bars + 2);
    unsigned char* xch = reinterpret_cast<unsigned char*>(bars + 4);  // 16-B aligned
    const Real* __restrict__ src = static_cast<const Real*>(a.src);
    Real* __restrict__ dst = static_cast<Real*>(a.dst);
    const long long len = a.len;
    const Real r = Real(a.r), c = Real(a.c), c1 = Real(a.c1), c2 = Real(a.c2);
    const bool wrap = a.wrap != 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = warp * kWarp + lane;  // lane position in the CTA window

    constexpr int kRingBytes = C::kRing * G * 2 * 16;
    for (int i = threadIdx.x; i < kRingBytes / 8; i += blockDim.x)
        reinterpret_cast<unsigned long long*>(xch)[i] = ~0ull;  // no tag
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tm_src);
        tma_prefetch_desc(&tm_dst);
        *s_next = (long long)atomicAdd(a.counter, 1ull);
    }
    __syncthreads();

    Seam sm;
    sm.xch = smem_u32(xch);
    sm.pub = (lane == 0 && warp > 0) || (lane == kWarp - 1 && warp < G - 1);
    sm.rd = sm.pub;
    sm.put = sm.pub ? uint32_t((warp * 2 + (lane == 0 ? 0 : 1)) * 16) : uint32_t(kRingBytes);
    sm.get = uint32_t(((lane == 0 ? warp - 1 : warp + 1) * 2 + (lane == 0 ? 1 : 0)) * 16);
    sm.tag = 0;

    const long long tma_len = a.nchunks * T::kUnit;
    auto window = [&](long long t) { return a.out_lo + t * C::kOut - H; };
    auto in_window = [&](long long g, long long w0) { return g >= 0 && g >= w0 && g < w0 + C::kWin; };
    auto interior = [&](long long t) {
        const long long w0 = window(t);
        return w0 >= 0 && w0 + C::kWin <= tma_len && !in_window(a.pin_lo, w0) &&
               !in_window(a.pin_hi, w0);
    };
    auto bufp = [&](int b) { return smem + b * C::kBufBytes; };
    auto issue = [&](int b, long long t) {  // thread 0 only
        bulk_wait_read_all();  // the TMA store that last used buffer b has read it
        mbar_arrive_expect_tx(&bars[b], C::kBufBytes);
        tma_load_3d(bufp(b), &tm_src, 0, 0, int(window(t) / T::kUnit), &bars[b]);
    };

    uint32_t phase = 0;
    bool bad = false;
    long long t = *s_next;
    if (threadIdx.x == 0 && t < a.tiles && interior(t)) issue(0, t);
    for (int it = 0; t < a.tiles; ++it) {
        unsigned long long nraw = 0;
        if (threadIdx.x == 0) nraw = atomicAdd(a.counter, 1ull);
        const int b = it & 1;
        unsigned char* buf = bufp(b);
        const long long w0 = window(t);
        const bool inter = interior(t);  // CTA-uniform
        const long long g0 = w0 + (long long)slot * V;
        Real u[V];
        if (inter) {
            mbar_wait(&bars[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            chunk_from_smem<Real, V>(buf, slot, u);
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
        // every window read precedes any staging into this buffer; the next
        // window goes to the other buffer
        __syncthreads();
        const long long tn = (long long)nraw;  // meaningful on thread 0 only
        if (threadIdx.x == 0) {
            *s_next = tn;
            if (tn < a.tiles && interior(tn)) {
                fence_proxy_async_smem();
                issue(b ^ 1, tn);
            }
        }

        if (inter || (!in_window(a.pin_lo, w0) && !in_window(a.pin_hi, w0))) {
            cta_steps_pipelined<Real, V, G, PU>(u, r, c, a.nsteps, sm, lane);
        } else {
            for (int s = 0; s < a.nsteps; ++s) {
                cta_step<Real, V, G>(u, r, c, sm, lane);
                pin_ends<Real, V>(u, g0, a.pin_lo, a.pin_hi, c1, c2);
            }
        }

        // exact elements: CTA-window points [H, kWin - H)
        const int el_lo = min(V, max(0, H - slot * V));
        const int el_hi = min(V, max(0, C::kWin - H - slot * V));
        if (a.check_finite) {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi && g0 + i < a.out_hi && !isfinite(u[i])) bad = true;
        }
        const bool full = w0 + C::kWin - H <= a.out_hi;
        if (inter && full) {
            chunk_to_smem_out<Real, V, H>(buf, slot, u, el_lo, el_hi);
            fence_proxy_async_smem();
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi && g0 + i < a.out_hi) dst[g0 + i] = u[i];
        }
        __syncthreads();  // staging complete; s_next visible
        if (inter && full && threadIdx.x == 0) {
            tma_store_3d(&tm_dst, 0, 0, int((w0 + H) / T::kUnit), buf);
            bulk_commit();
        }
        t = *s_next;
    }
    if (threadIdx.x == 0) bulk_wait_all();
    if (bad) atomicOr(a.nonfinite, 1u);
}

}  // namespace hb
