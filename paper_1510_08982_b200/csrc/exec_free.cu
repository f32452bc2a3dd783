// exec_free.cu -- K10: exec_run(BarrierFree) of small and medium fields in ONE
// thread-block cluster (run_barrier_free, async_exec.cpp:156-259).
//
// The reference runs one thread per PE: each step a worker reads its two
// neighbours' latest published edge values, computes its n points with one
// ghost cell per side, and publishes its own two edges -- no barrier.  Here a
// PE is one WARP: Lc lanes x V points per lane (Lc * V = n exactly), the
// points in registers for the whole run, neighbour values inside the PE by
// warp shuffles of the r*u products (K1's step code).  The PE warps of a run
// are spread over the CTAs of one cluster (one warp per SM sub-partition when
// P <= 64), so every PE advances at the latency of its own step and no SM's
// FP64 issue is shared by more PEs than necessary.
//
// Edge exchange: every PE owns two receive rings in its CTA's shared memory
// (its left neighbour's last point, its right neighbour's first point).  A
// producer stores the value it computed for step k+1 straight into the
// consumer's ring slot (k+1) mod R over DSMEM (st.shared::cluster).  A slot
// is two 64-bit words, each {step tag : 32 | half of the double : 32}: an
// aligned 64-bit store is single-copy atomic, so a reader that sees the
// expected tag in BOTH words has the whole value -- no fence, no flag word,
// no ordering between the two stores needed (NCCL's LL protocol, applied to
// shared memory).  The consumer polls its own shared memory only.
//
// Staleness: at step k a PE uses the newest neighbour value it has seen with
// step k* <= k (never a value from the future), probing slot k (the exact,
// synchronous value) and slot m+1 (the next one after the newest seen) each
// step.  It waits only when k - k* would exceed q - 1 -- the model's bounded
// delay (paper Eq. (4)); q = 1 is therefore the exact
// synchronous scheme, bit for bit.  The two neighbours of a boundary read each
// other, so neither can lead by more than q - 1 steps, and a ring of R >= 2q
// slots is never overwritten while a reader may still need a slot.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "async_pe.cuh"
#include "runtime.cuh"
#include "sync_tb.cuh"

namespace hb {
namespace {

constexpr int kFreeR = 32;         // ring slots per receive ring (power of two, >= 2q)
constexpr int kFreeMaxQ = kFreeR / 2;
constexpr int kFreeMaxCluster = 16;
constexpr int kFreeMaxW = 8;  // PE warps per CTA (registers: up to 40 points per lane)

struct FreeArgs {
    double* field;  // [N] prepared initial field in, final field out
    int n, P, Lc, W;
    int Wp;  // warps per PE (1, 2 or 4; divides W)
    double r, c, c1, c2;
    int dirichlet;
    long long k_end;
    int q;
    unsigned int* flag;               // [0] non-finite result, [1] watchdog
    unsigned long long* stats;        // kStat* layout (async_pe.cuh) or null
    unsigned long long timeout_ns;
};

struct __align__(16) FreeSlot {
    unsigned long long lo, hi;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_cluster(uint32_t addr, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
    return out;
}
// A plain (weak) 16-B DSMEM store: ptxas turns .relaxed.cluster / .volatile
// into ST.E.128.STRONG.GPU / .SYS, ~25 ns per step slower (measured).  Each
// 64-bit half carries its own tag, so a reader accepts a slot only when both
// aligned halves (each written in one piece) show the step it wants.
__device__ __forceinline__ void st_cluster_slot(uint32_t addr, unsigned long long lo,
                                                unsigned long long hi) {
    asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(lo),
                 "l"(hi)
                 : "memory");
}
__device__ __forceinline__ FreeSlot ld_slot(uint32_t addr) {
    FreeSlot s;
    asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];"
                 : "=l"(s.lo), "=l"(s.hi)
                 : "r"(addr)
                 : "memory");
    return s;
}
__device__ __forceinline__ unsigned long long pack_half(uint32_t tag, uint32_t half) {
    return (unsigned long long)tag << 32 | half;
}
__device__ __forceinline__ bool slot_is(const FreeSlot& s, uint32_t tag) {
    return uint32_t(s.lo >> 32) == tag && uint32_t(s.hi >> 32) == tag;
}
__device__ __forceinline__ double slot_value(const FreeSlot& s) {
    return __hiloint2double(int(uint32_t(s.hi)), int(uint32_t(s.lo)));
}

// Inner-PE seam slots (CTA shared memory): the same tagged halves, local.
__device__ __forceinline__ void seam_store(uint32_t addr, uint32_t tag, double v) {
    asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(addr),
                 "l"(pack_half(tag, uint32_t(__double2loint(v)))),
                 "l"(pack_half(tag, uint32_t(__double2hiint(v))))
                 : "memory");
}
__device__ __forceinline__ FreeSlot seam_poll(uint32_t addr) {
    FreeSlot s;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                 : "=l"(s.lo), "=l"(s.hi)
                 : "r"(addr)
                 : "memory");
    return s;
}
// The ghost product a PE's edge lane consumes at step k, resolved from the
// two probes issued one step earlier (slot k and the slot after the newest
// one seen, m+1), branch-free.
__device__ __forceinline__ void resolve_ghost(const FreeSlot& s0, const FreeSlot& s1, int k,
                                              int& m, double& pg) {
    const bool h0 = slot_is(s0, uint32_t(k));
    const bool h1 = slot_is(s1, uint32_t(m + 1));
    const double x = h0 ? slot_value(s0) : slot_value(s1);
    pg = (h0 || h1) ? x : pg;
    m = h0 ? k : (h1 ? m + 1 : m);
}

// MW: PEs span several warps (seam exchange compiled in)
template <int V, bool STATS, bool MW>
__global__ void __launch_bounds__(kFreeMaxW * 32, 1) exec_free_kernel(const FreeArgs a) {
    extern __shared__ __align__(16) FreeSlot rings[];  // [W][2 sides][kFreeR]
    __shared__ FreeSlot seams[4][kFreeMaxW][2];         // inner-PE warp seams, ring of 4
    __shared__ unsigned int s_hist[kFreeMaxW * 2][kFreeMaxQ];  // STATS: one row per edge lane
    const int W = a.W, Wp = MW ? a.Wp : 1;  // single-warp PEs: the v2 loop, folded
    const uint32_t cta = cluster_ctarank();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = int(cta) * W + w;  // warp index in the cluster
    const int p = gw / Wp, wi = gw - p * Wp;  // PE, warp inside the PE
    const bool active = w < W && p < a.P;  // warp-uniform
    const int n = a.n, P = a.P, Lc = a.Lc;
    // invalidate every slot of this CTA's rings (tag 0xffffffff = no step)
    for (int i = threadIdx.x; i < W * 2 * kFreeR; i += blockDim.x)
        rings[i] = FreeSlot{~0ull, ~0ull};
    if (MW)
        for (int i = threadIdx.x; i < 4 * kFreeMaxW * 2; i += blockDim.x)
            (&seams[0][0][0])[i] = FreeSlot{~0ull, ~0ull};
    if (STATS)
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x)
            (&s_hist[0][0])[i] = 0;
    cluster_sync_all();  // no producer may write a slot before its owner cleared it

    // r and c stay kernel parameters: ptxas keeps them in uniform registers,
    // so every DMUL reads one vector register pair, not two (loading them
    // into vector registers measured 40% slower per step)
    const double r = a.r, c = a.c;
    using A = Arith<double>;
    const bool dir = a.dirichlet != 0;
    const int lpe = p > 0 ? p - 1 : (dir ? -1 : P - 1);
    const int rpe = p + 1 < P ? p + 1 : (dir ? -1 : 0);
    const bool first_lane = lane == 0, last_lane = lane == Lc - 1;
    const bool pe_first = first_lane && wi == 0;         // the PE's first point
    const bool pe_last = last_lane && wi == Wp - 1;      // the PE's last point
    const bool needL = active && lpe >= 0;  // Dirichlet PE 0 / P-1 have a pinned end instead
    const bool needR = active && rpe >= 0;
    const bool pin_first = active && dir && p == 0 && pe_first;
    const bool pin_last = active && dir && p == P - 1 && pe_last;
    // a PE wider than one warp is synchronous inside: its warps swap their
    // seam products every step through shared memory (exact, never stale)
    const bool seamL = active && first_lane && wi > 0;
    const bool seamR = active && last_lane && wi < Wp - 1;

    // The PE's first lane reads ring side 0 (its left neighbour PE's last
    // product) and publishes its own first product into that PE's side-1
    // ring; the last lane mirrors it.  Every other lane probes its warp's ring
    // too (a valid address) and ignores the result: no divergent branch.
    const bool edge = (pe_first && needL) || (pe_last && needR);
    const int side = first_lane ? 0 : 1;
    const int nb_gw = first_lane ? lpe * Wp + Wp - 1 : rpe * Wp;  // neighbour PE's edge warp
    const uint32_t my_ring = smem_u32(rings + ((size_t)(active ? w : 0) * 2 + side) * kFreeR);
    uint32_t peer_ring = 0;
    if (edge) {
        const int nb_cta = nb_gw / W, nb_w = nb_gw % W;
        const uint32_t local = smem_u32(rings + ((size_t)nb_w * 2 + (1 - side)) * kFreeR);
        peer_ring = map_cluster(local, uint32_t(nb_cta));
    }
    auto slot_addr = [&](uint32_t base, int k) { return base + uint32_t(k & (kFreeR - 1)) * 16u; };
    auto publish = [&](int k, double prod) {
        if (edge)
            st_cluster_slot(slot_addr(peer_ring, k), pack_half(uint32_t(k), uint32_t(__double2loint(prod))),
                            pack_half(uint32_t(k), uint32_t(__double2hiint(prod))));
        if (MW && (seamL || seamR))
            seam_store(smem_u32(&seams[k & 3][w][side]), uint32_t(k), prod);
    };
    // the neighbouring warp's seam product of step k, polled by the whole
    // warp until the seam lanes have theirs (it is exact: no staleness)
    const bool seam_rd = seamL || seamR;
    const int seam_w = seamL ? w - 1 : (seamR ? w + 1 : w);
    auto seam_fetch = [&](int k) {
        const uint32_t addr = smem_u32(&seams[k & 3][seam_w][first_lane ? 1 : 0]);
        while (true) {
            const FreeSlot s = seam_poll(addr);
            if (__all_sync(0xffffffffu, !seam_rd || slot_is(s, uint32_t(k)))) return slot_value(s);
        }
    };

    double u[V];
    const long long base = (long long)p * n + (long long)(wi * Lc + lane) * V;
#pragma unroll
    for (int i = 0; i < V; ++i) u[i] = (active && lane < Lc) ? a.field[base + i] : 0.0;
    if (pin_first) u[0] = a.c1;  // prepare_initial snapped them already; keep exact
    if (pin_last) u[V - 1] = a.c2;

    // products r*u of the lane's two end points; the step-0 edge products go out
    double pF = A::mul(r, u[0]);
    double pLs = A::mul(r, u[V - 1]);
    double pL = __shfl_up_sync(0xffffffffu, pLs, 1);
    double pR = __shfl_down_sync(0xffffffffu, pF, 1);
    publish(0, first_lane ? pF : pLs);

    int m = -1;        // newest neighbour step seen (edge lanes)
    double pg = 0.0;   // its product r*u
    unsigned long long waits = 0;
    int maxd = 0;
    bool dead = false;  // the watchdog fired somewhere: stop waiting
    const int qm1 = a.q - 1;
    const int k_end = int(a.k_end);
    FreeSlot s0 = ld_slot(slot_addr(my_ring, 0)), s1 = s0;
    if (active) {
        for (int k = 0; k < k_end; ++k) {
            // ---- ghost for step k: probes from the previous step, then wait
            // only when it would be more than q-1 steps old (bounded delay)
            resolve_ghost(s0, s1, k, m, pg);
            if (!MW) {
                // v2 form (measured fastest for single-warp PEs): lanes that
                // must wait spin alone, the warp reconverges below
                if (edge && !dead && k - m > qm1) {
                    if (STATS) ++waits;
                    const uint64_t t0 = globaltimer_ns();
                    unsigned spins = 0;
                    while (k - m > qm1) {
                        const FreeSlot s = ld_slot(slot_addr(my_ring, m + 1));
                        if (slot_is(s, uint32_t(m + 1))) {
                            ++m;
                            pg = slot_value(s);
                        } else if ((++spins & 1023u) == 0 &&
                                   (globaltimer_ns() - t0 > a.timeout_ns ||
                                    *(volatile unsigned int*)(a.flag + 1))) {
                            atomicOr(a.flag + 1, 1u);
                            dead = true;
                            break;
                        }
                    }
                }
                __syncwarp();
            } else {
                // warp-uniform wait: the seam polls below shuffle-vote, and a
                // loop that only some lanes run would leave the warp diverged
                bool need = edge && !dead && k - m > qm1;
                if (__any_sync(0xffffffffu, need)) {
                    if (STATS && need) ++waits;
                    const uint64_t t0 = globaltimer_ns();
                    unsigned spins = 0;
                    while (true) {
                        if (need) {
                            const FreeSlot s = ld_slot(slot_addr(my_ring, m + 1));
                            if (slot_is(s, uint32_t(m + 1))) {
                                ++m;
                                pg = slot_value(s);
                                need = k - m > qm1;
                            }
                        }
                        if (!__any_sync(0xffffffffu, need)) break;
                        if ((++spins & 1023u) == 0 &&
                            (globaltimer_ns() - t0 > a.timeout_ns ||
                             *(volatile unsigned int*)(a.flag + 1))) {
                            if (lane == 0) atomicOr(a.flag + 1, 1u);
                            dead = true;
                            break;
                        }
                    }
                }
            }
            if (STATS && edge) {
                const int d = k - m;
                maxd = d > maxd ? d : maxd;
                ++s_hist[w * 2 + side][d < kFreeMaxQ ? d : kFreeMaxQ - 1];
            }
            // probes for step k+1, answered while this step computes
            s0 = ld_slot(slot_addr(my_ring, k + 1));
            s1 = ld_slot(slot_addr(my_ring, m + 1));
            if (pe_first) pL = pg;  // the ghost product replaces the shuffle
            if (pe_last) pR = pg;
            if constexpr (MW) {  // the neighbouring warps' seam products (exact)
                const double x = seam_fetch(k);
                if (seamL) pL = x;
                if (seamR) pR = x;
            }
            // ---- one Jacobi step: the lane's end points first, their products
            // shuffled and published, then the interior points (K1's
            // software-pipelined order; same products, same roundings)
            if constexpr (V == 1) {
                double n0 = stencil_p(pR, A::mul(c, u[0]), pL);
                if (pin_first) n0 = a.c1;
                if (pin_last) n0 = a.c2;
                const double p0 = A::mul(r, n0);
                pL = __shfl_up_sync(0xffffffffu, p0, 1);
                pR = __shfl_down_sync(0xffffffffu, p0, 1);
                publish(k + 1, p0);
                u[0] = n0;
                pF = pLs = p0;
            } else {
                const double p1 = V == 2 ? pLs : A::mul(r, u[1]);
                const double pVm2 = V == 2 ? pF : (V == 3 ? p1 : A::mul(r, u[V - 2]));
                double nF = stencil_p(p1, A::mul(c, u[0]), pL);
                double nL = stencil_p(pR, A::mul(c, u[V - 1]), pVm2);
                if (pin_first) nF = a.c1;
                if (pin_last) nL = a.c2;
                const double pF2 = A::mul(r, nF);
                const double pLs2 = A::mul(r, nL);
                pL = __shfl_up_sync(0xffffffffu, pLs2, 1);  // for step k+1
                pR = __shfl_down_sync(0xffffffffu, pF2, 1);
                publish(k + 1, first_lane ? pF2 : pLs2);
                double pm1 = pF, p0 = p1;
#pragma unroll
                for (int i = 1; i <= V - 2; ++i) {
                    double pn;
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
    }
    bool bad = false;
    if (active && lane < Lc) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            bad |= !isfinite(u[i]);
            a.field[base + i] = u[i];
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
    if (STATS) {
        if (edge) {
            atomicAdd(a.stats + kStatReads, (unsigned long long)k_end);
            atomicAdd(a.stats + kStatWaits, waits);
            atomicMax(a.stats + kStatMaxDelay, (unsigned long long)maxd);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x) {
            const unsigned int v = (&s_hist[0][0])[i];
            if (v) atomicAdd(a.stats + kStatDelayHist + i % kFreeMaxQ, (unsigned long long)v);
        }
    }
    cluster_sync_all();  // no CTA leaves while a peer may still store into its shared memory
}

// K10 with lane halos and rounds, for PEs of one warp (K10r).  The plain
// kernel above exchanges lane-edge products by shuffle, polls the ghost and
// publishes the PE edges EVERY step; a single warp per SM sub-partition has
// nothing to hide those latencies behind (~200 cycles per step, measured,
// whatever V).  Here a PE advances in rounds of LH steps:
//   * each lane also holds the LH points on either side of its own V (copies
//     of its neighbours' points, refreshed by shuffle once per round) and
//     steps them redundantly, so no shuffle sits inside a round;
//   * the PE edges are polled once per round (the newest published value,
//     from a probe issued at the end of the previous round) and published
//     once per round (the edge product at the round's last step).
// The asynchronous model allows exactly this: every consumed neighbour value
// is the neighbour's value at some step k* with 0 <= k - k* <= q - 1 (paper
// Eq. (4); the lanes wait only when the round's last step would read an
// older one), and inside a PE every update is the same stencil_p on the same
// products as the synchronous scheme (bit-identical when q = 1 forces k* = k,
// which takes the plain kernel).  LH <= q/2: a neighbour one round behind
// still satisfies the bound, so lockstep PEs never wait.
// RING = false: K10w (the whole field in one warp; no ring, no ghost, no publish)
template <int V, int LH, bool STATS, bool RING = true>
__global__ void __launch_bounds__(kFreeMaxW * 32, 1) exec_free_lh_kernel(const FreeArgs a) {
    constexpr int E = V + 2 * LH;  // own points x[LH, LH+V)
    // lanes whose window holds the PE's outer neighbour position (-1 or
    // n_pe): d = 0 .. kG lanes in from either end; its end points: 0 .. kP
    constexpr int kG = (LH - 1) / V, kP = LH / V;
    extern __shared__ __align__(16) FreeSlot rings[];  // [W][2 sides][kFreeR], slot = round
    __shared__ unsigned int s_hist[kFreeMaxW * 2][kFreeMaxQ];
    const int W = a.W;
    const uint32_t cta = cluster_ctarank();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = int(cta) * W + w;
    const bool active = w < W && p < a.P;
    const int n = a.n, P = a.P, Lc = a.Lc;
    for (int i = threadIdx.x; i < W * 2 * kFreeR; i += blockDim.x)
        rings[i] = FreeSlot{~0ull, ~0ull};
    if (STATS)
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x)
            (&s_hist[0][0])[i] = 0;
    // r, c and the pinned values go through shared memory into registers
    // once: ptxas otherwise re-loads kernel parameters from the constant bank
    // inside the step loop (LDC + a short-scoreboard stall before the first
    // DMUL of every step, measured with ncu)
    __shared__ __align__(16) double s_coef[4];
    __shared__ int s_qm1;
    if (threadIdx.x == 0) {
        s_coef[0] = a.r;
        s_coef[1] = a.c;
        s_coef[2] = a.c1;
        s_coef[3] = a.c2;
        s_qm1 = a.q - 1;
    }
    cluster_sync_all();

    double r, c, c1, c2;
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r), "=d"(c) : "r"(smem_u32(s_coef)) : "memory");
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c1), "=d"(c2) : "r"(smem_u32(s_coef + 2)) : "memory");
    using A = Arith<double>;
    const bool dir = a.dirichlet != 0;
    const int lpe = p > 0 ? p - 1 : (dir ? -1 : P - 1);
    const int rpe = p + 1 < P ? p + 1 : (dir ? -1 : 0);
    const bool first_lane = lane == 0, last_lane = lane == Lc - 1;
    const bool needL = active && lpe >= 0;
    const bool needR = active && rpe >= 0;
    const bool pin_first = active && dir && p == 0 && first_lane;
    const bool pin_last = active && dir && p == P - 1 && last_lane;
    const bool pinL = active && dir && p == 0, pinR = active && dir && p == P - 1;  // warp-uniform
    const bool edge = RING && ((first_lane && needL) || (last_lane && needR));
    const int side = first_lane ? 0 : 1;
    const int nb = first_lane ? lpe : rpe;
    const uint32_t my_ring = smem_u32(rings + ((size_t)(active ? w : 0) * 2 + side) * kFreeR);
    uint32_t peer_ring = 0;
    if (edge) {
        const int nb_cta = nb / W, nb_w = nb % W;
        const uint32_t local = smem_u32(rings + ((size_t)nb_w * 2 + (1 - side)) * kFreeR);
        peer_ring = map_cluster(local, uint32_t(nb_cta));
    }
    // the value of step t (a multiple of LH, or k_end) lives in slot t / LH
    auto slot_addr = [&](uint32_t base, int t) {
        return base + uint32_t((t / LH) & (kFreeR - 1)) * 16u;
    };
    auto publish = [&](int t, double prod) {
        if (edge)
            st_cluster_slot(slot_addr(peer_ring, t), pack_half(uint32_t(t), uint32_t(__double2loint(prod))),
                            pack_half(uint32_t(t), uint32_t(__double2hiint(prod))));
    };

    double x[E];
    const long long base = (long long)p * n + (long long)lane * V;
#pragma unroll
    for (int i = 0; i < V; ++i) x[LH + i] = (active && lane < Lc) ? a.field[base + i] : 0.0;
    if (pin_first) x[LH] = c1;
    if (pin_last) x[LH + V - 1] = c2;
    double pgL = 0.0, pgR = 0.0;  // the round's ghosts, on every lane near an end
    publish(0, A::mul(r, first_lane ? x[LH] : x[LH + V - 1]));

    int m = -1;         // step of the newest neighbour value seen (a round start)
    double pg = 0.0;    // its product r*u
    unsigned long long waits = 0;
    int maxd = 0;
    bool dead = false;
    int qm1;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(qm1) : "r"(smem_u32(&s_qm1)) : "memory");
    const int k_end = int(a.k_end);
    FreeSlot sa = ld_slot(slot_addr(my_ring, 0)), sb = sa;  // probes: round starts k, k - LH
    // ghost for the round of steps k..last
    auto ghost = [&](int k, int last) {
        const bool ha = slot_is(sa, uint32_t(k)), hb = k >= LH && slot_is(sb, uint32_t(k - LH));
        if (ha && k > m) {
            m = k;
            pg = slot_value(sa);
        } else if (hb && k - LH > m) {
            m = k - LH;
            pg = slot_value(sb);
        }
        // warp-uniform test first: the common case (no lane needs to wait)
        // costs one vote, no divergent branch and no reconvergence
        const bool need = edge && !dead && last - m > qm1;
        if (__any_sync(0xffffffffu, need)) {
          if (need) {
            if (STATS) ++waits;
            const uint64_t t0 = globaltimer_ns();
            unsigned spins = 0;
            while (last - m > qm1) {
                const int t = m < 0 ? 0 : m + LH;  // the next value the neighbour publishes
                const FreeSlot s = ld_slot(slot_addr(my_ring, t));
                if (slot_is(s, uint32_t(t))) {
                    m = t;
                    pg = slot_value(s);
                } else if ((++spins & 1023u) == 0 &&
                           (globaltimer_ns() - t0 > a.timeout_ns ||
                            *(volatile unsigned int*)(a.flag + 1))) {
                    atomicOr(a.flag + 1, 1u);
                    dead = true;
                    break;
                }
            }
          }
          __syncwarp();
        }
        if (STATS && edge) {
            for (int kk = k; kk <= last; ++kk) {
                const int d = kk - m;
                maxd = d > maxd ? d : maxd;
                ++s_hist[w * 2 + side][d < kFreeMaxQ ? d : kFreeMaxQ - 1];
            }
        }
    };
    // one step of window points x[lo, hi) (lo >= 1, hi <= E-1): all the
    // products, then the sums -- the same stencil_p, the same roundings
    auto step = [&](auto lo_c, auto hi_c) {
        constexpr int lo = decltype(lo_c)::value, hi = decltype(hi_c)::value;
        double pr[E], cx[E];
#pragma unroll
        for (int i = lo - 1; i <= hi; ++i) pr[i] = A::mul(r, x[i]);
#pragma unroll
        for (int i = lo; i < hi; ++i) cx[i] = A::mul(c, x[i]);
        // the PE's outer neighbours (positions -1 and n_pe) are the ghosts, in
        // whichever lanes' windows hold them (a pinned end is re-pinned below)
#pragma unroll
        for (int d = 0; d <= kG; ++d) {
            if (LH - 1 - d * V >= lo - 1 && lane == d) pr[LH - 1 - d * V >= 0 ? LH - 1 - d * V : 0] = pgL;
            if (LH + V + d * V <= hi && lane == Lc - 1 - d) pr[LH + V + d * V < E ? LH + V + d * V : E - 1] = pgR;
        }
#pragma unroll
        for (int i = lo; i < hi; ++i) cx[i] = A::add(pr[i + 1], cx[i]);
#pragma unroll
        for (int i = lo; i < hi; ++i) x[i] = A::add(cx[i], pr[i - 1]);
        if (pinL || pinR) {  // warp-uniform: only the two end PEs of a Dirichlet run
#pragma unroll
            for (int d = 0; d <= kP; ++d) {
                if (pinL && lane == d) x[LH - d * V >= 0 ? LH - d * V : 0] = c1;
                if (pinR && lane == Lc - 1 - d) x[LH + V - 1 + d * V < E ? LH + V - 1 + d * V : E - 1] = c2;
            }
        }
    };
    // halos: the LH points on either side, from the lanes that own them
    // (one lane away when V >= LH, more when V < LH)
    auto exchange = [&]() {
        double own[V];
#pragma unroll
        for (int e = 0; e < V; ++e) own[e] = x[LH + e];
#pragma unroll
        for (int i = 0; i < LH; ++i) {
            const int g = i - LH;                  // position relative to the lane's first point
            const int dl = (-g + V - 1) / V;       // lanes up
            x[i] = __shfl_up_sync(0xffffffffu, own[g + dl * V], dl);
            const int gr = V + i, dr = gr / V;     // lanes down
            x[LH + V + i] = __shfl_down_sync(0xffffffffu, own[gr - dr * V], dr);
        }
    };
    // a round: step j updates window points [1 + j, E - 1 - j)
    auto round_steps = [&](auto j_c) {
        constexpr int j = decltype(j_c)::value;
        step(std::integral_constant<int, 1 + j>{}, std::integral_constant<int, E - 1 - j>{});
    };
    if (active) {
        int k = 0;
        for (int rounds = k_end / LH; rounds > 0; --rounds) {  // count down: no k_end reload
            exchange();
            if constexpr (RING) {
                ghost(k, k + LH - 1);
                pgL = kG > 0 ? __shfl_sync(0xffffffffu, pg, 0) : pg;
                pgR = kG > 0 ? __shfl_sync(0xffffffffu, pg, Lc - 1) : pg;
            }
            round_steps(std::integral_constant<int, 0>{});
            round_steps(std::integral_constant<int, 1>{});
            if constexpr (LH > 2) {
                round_steps(std::integral_constant<int, 2>{});
                round_steps(std::integral_constant<int, 3>{});
            }
            k += LH;
            if constexpr (RING) {
                sa = ld_slot(slot_addr(my_ring, k));  // answered while the halos move; issued
                sb = ld_slot(slot_addr(my_ring, k - LH));  // before the publish (see K10t)
                publish(k, A::mul(r, first_lane ? x[LH] : x[LH + V - 1]));
            }
        }
        if (k < k_end) {  // the remaining steps, one at a time (plain halo refresh each)
            if constexpr (RING) {
                ghost(k, k_end - 1);
                pgL = kG > 0 ? __shfl_sync(0xffffffffu, pg, 0) : pg;
                pgR = kG > 0 ? __shfl_sync(0xffffffffu, pg, Lc - 1) : pg;
            }
            for (; k < k_end; ++k) {
                exchange();
                round_steps(std::integral_constant<int, LH - 1>{});
            }
        }
    }
    bool bad = false;
    if (active && lane < Lc) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            bad |= !isfinite(x[LH + i]);
            a.field[base + i] = x[LH + i];
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
    if (STATS) {
        if (edge) {
            atomicAdd(a.stats + kStatReads, (unsigned long long)k_end);
            atomicAdd(a.stats + kStatWaits, waits);
            atomicMax(a.stats + kStatMaxDelay, (unsigned long long)maxd);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x) {
            const unsigned int v = (&s_hist[0][0])[i];
            if (v) atomicAdd(a.stats + kStatDelayHist + i % kFreeMaxQ, (unsigned long long)v);
        }
    }
    cluster_sync_all();
}

// K10 with one THREAD per PE (K10t), for PEs of up to 50 points: the
// reference's own decomposition (one worker per PE, async_exec.cpp:156-259)
// at its most literal.  Lane 0 of the PE's warp holds all n points in
// registers, so there is no intra-PE exchange at all: a step is n stencils
// with the two ghost products at the ends, and the PE edges are polled and
// published once per round of LH steps as in K10r (LH <= q/2; LH = 1 polls
// every step).  A step costs ~8n + 40 cycles of FP64 issue, so tiny PEs (the
// reference's measure() at N = 100) run well below the ~170-cycle floor of a
// PE spread over a warp's lanes.
template <int V, int LH, bool STATS>
__global__ void __launch_bounds__(kFreeMaxW * 32, 1) exec_free_pe_kernel(const FreeArgs a) {
    extern __shared__ __align__(16) FreeSlot rings[];  // [W][2 sides][kFreeR], slot = round
    __shared__ unsigned int s_hist[kFreeMaxW * 2][kFreeMaxQ];
    __shared__ __align__(16) double s_coef[4];
    const int W = a.W;
    const uint32_t cta = cluster_ctarank();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = int(cta) * W + w;
    const bool active = w < W && p < a.P && lane == 0;
    const int n = a.n, P = a.P;
    for (int i = threadIdx.x; i < W * 2 * kFreeR; i += blockDim.x)
        rings[i] = FreeSlot{~0ull, ~0ull};
    if (STATS)
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x)
            (&s_hist[0][0])[i] = 0;
    if (threadIdx.x == 0) {  // coefficients into registers via shared memory (see K10r)
        s_coef[0] = a.r;
        s_coef[1] = a.c;
        s_coef[2] = a.c1;
        s_coef[3] = a.c2;
    }
    cluster_sync_all();

    unsigned long long waits = 0;
    int maxd = 0;
    bool bad = false;
    const int k_end = int(a.k_end);
    if (active) {
        double r, c, c1, c2;
        asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r), "=d"(c) : "r"(smem_u32(s_coef)) : "memory");
        asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c1), "=d"(c2) : "r"(smem_u32(s_coef + 2)) : "memory");
        using A = Arith<double>;
        const bool dir = a.dirichlet != 0;
        const int lpe = p > 0 ? p - 1 : (dir ? -1 : P - 1);
        const int rpe = p + 1 < P ? p + 1 : (dir ? -1 : 0);
        const bool needL = lpe >= 0, needR = rpe >= 0;
        const bool pinL = dir && p == 0, pinR = dir && p == P - 1;
        // side 0: the left neighbour's last product; side 1: the right one's first
        const uint32_t ringL = smem_u32(rings + ((size_t)w * 2 + 0) * kFreeR);
        const uint32_t ringR = smem_u32(rings + ((size_t)w * 2 + 1) * kFreeR);
        uint32_t peerL = 0, peerR = 0;  // where this PE's first / last product goes
        if (needL) peerL = map_cluster(smem_u32(rings + ((size_t)(lpe % W) * 2 + 1) * kFreeR), uint32_t(lpe / W));
        if (needR) peerR = map_cluster(smem_u32(rings + ((size_t)(rpe % W) * 2 + 0) * kFreeR), uint32_t(rpe / W));
        auto slot_addr = [&](uint32_t base, int t) {
            return base + uint32_t((t / LH) & (kFreeR - 1)) * 16u;
        };
        auto put = [&](uint32_t peer, int t, double prod) {
            st_cluster_slot(slot_addr(peer, t), pack_half(uint32_t(t), uint32_t(__double2loint(prod))),
                            pack_half(uint32_t(t), uint32_t(__double2hiint(prod))));
        };
        double x[V];
        const long long base = (long long)p * n;
#pragma unroll
        for (int i = 0; i < V; ++i) x[i] = a.field[base + i];
        if (pinL) x[0] = c1;
        if (pinR) x[V - 1] = c2;
        auto publish = [&](int t) {
            if (needL) put(peerL, t, A::mul(r, x[0]));
            if (needR) put(peerR, t, A::mul(r, x[V - 1]));
        };
        publish(0);
        int mL = -1, mR = -1;           // steps of the newest neighbour values seen
        double pgL = 0.0, pgR = 0.0;    // their products
        bool dead = false;
        const int qm1 = a.q - 1;
        FreeSlot la = ld_slot(slot_addr(ringL, 0)), lb = la, ra = ld_slot(slot_addr(ringR, 0)), rb = ra;
        // resolve one side for the round k..last (probes of round starts k, k - LH)
        auto side_ghost = [&](bool need, uint32_t ring, const FreeSlot& sa, const FreeSlot& sb, int k,
                              int last, int& m, double& pg, int hrow) {
            if (!need) return;
            if (slot_is(sa, uint32_t(k)) && k > m) {
                m = k;
                pg = slot_value(sa);
            } else if (k >= LH && slot_is(sb, uint32_t(k - LH)) && k - LH > m) {
                m = k - LH;
                pg = slot_value(sb);
            }
            if (!dead && last - m > qm1) {
                if (STATS) ++waits;
                const uint64_t t0 = globaltimer_ns();
                unsigned spins = 0;
                while (last - m > qm1) {
                    const int t = m < 0 ? 0 : m + LH;
                    const FreeSlot sl = ld_slot(slot_addr(ring, t));
                    if (slot_is(sl, uint32_t(t))) {
                        m = t;
                        pg = slot_value(sl);
                    } else if ((++spins & 1023u) == 0 &&
                               (globaltimer_ns() - t0 > a.timeout_ns ||
                                *(volatile unsigned int*)(a.flag + 1))) {
                        atomicOr(a.flag + 1, 1u);
                        dead = true;
                        break;
                    }
                }
            }
            if (STATS) {
                for (int kk = k; kk <= last; ++kk) {
                    const int d = kk - m;
                    maxd = d > maxd ? d : maxd;
                    ++s_hist[hrow][d < kFreeMaxQ ? d : kFreeMaxQ - 1];
                }
            }
        };
        auto step = [&]() {
            double pr[V], cx[V];
#pragma unroll
            for (int i = 0; i < V; ++i) pr[i] = A::mul(r, x[i]);
#pragma unroll
            for (int i = 0; i < V; ++i) cx[i] = A::mul(c, x[i]);
#pragma unroll
            for (int i = 0; i < V; ++i) cx[i] = A::add(i + 1 < V ? pr[i + 1] : pgR, cx[i]);
#pragma unroll
            for (int i = 0; i < V; ++i) x[i] = A::add(cx[i], i > 0 ? pr[i - 1] : pgL);
            if (pinL) x[0] = c1;
            if (pinR) x[V - 1] = c2;
        };
        int k = 0;
        for (int rounds = k_end / LH; rounds > 0; --rounds) {
            side_ghost(needL, ringL, la, lb, k, k + LH - 1, mL, pgL, w * 2);
            side_ghost(needR, ringR, ra, rb, k, k + LH - 1, mR, pgR, w * 2 + 1);
#pragma unroll
            for (int j = 0; j < LH; ++j) step();
            k += LH;
            // probes before the publish: a load issued after a DSMEM store
            // waits for that store (~10 ns per step, measured)
            la = ld_slot(slot_addr(ringL, k));
            lb = ld_slot(slot_addr(ringL, k - LH));
            ra = ld_slot(slot_addr(ringR, k));
            rb = ld_slot(slot_addr(ringR, k - LH));
            publish(k);
        }
        if (k < k_end) {
            side_ghost(needL, ringL, la, lb, k, k_end - 1, mL, pgL, w * 2);
            side_ghost(needR, ringR, ra, rb, k, k_end - 1, mR, pgR, w * 2 + 1);
            for (; k < k_end; ++k) step();
        }
#pragma unroll
        for (int i = 0; i < V; ++i) {
            bad |= !isfinite(x[i]);
            a.field[base + i] = x[i];
        }
    }
    if (bad) atomicOr(a.flag, 1u);
    if (STATS) {
        if (active) {
            const int sides = int(p > 0 || a.dirichlet == 0) + int(p + 1 < P || a.dirichlet == 0);
            atomicAdd(a.stats + kStatReads, (unsigned long long)k_end * (unsigned long long)sides);
            atomicAdd(a.stats + kStatWaits, waits);
            atomicMax(a.stats + kStatMaxDelay, (unsigned long long)maxd);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kFreeMaxW * 2 * kFreeMaxQ; i += blockDim.x) {
            const unsigned int v = (&s_hist[0][0])[i];
            if (v) atomicAdd(a.stats + kStatDelayHist + i % kFreeMaxQ, (unsigned long long)v);
        }
    }
    cluster_sync_all();
}

// Points per lane compiled in; a PE of n points runs as Lc = n / V lanes.
constexpr int kFreeV[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 25, 32, 40, 50};

template <bool STATS>
const void* free_kernel_ptr(int V, bool MW) {
    switch (V) {
        case 1: return MW ? (const void*)exec_free_kernel<1, STATS, true> : (const void*)exec_free_kernel<1, STATS, false>;
        case 2: return MW ? (const void*)exec_free_kernel<2, STATS, true> : (const void*)exec_free_kernel<2, STATS, false>;
        case 3: return MW ? (const void*)exec_free_kernel<3, STATS, true> : (const void*)exec_free_kernel<3, STATS, false>;
        case 4: return MW ? (const void*)exec_free_kernel<4, STATS, true> : (const void*)exec_free_kernel<4, STATS, false>;
        case 5: return MW ? (const void*)exec_free_kernel<5, STATS, true> : (const void*)exec_free_kernel<5, STATS, false>;
        case 6: return MW ? (const void*)exec_free_kernel<6, STATS, true> : (const void*)exec_free_kernel<6, STATS, false>;
        case 8: return MW ? (const void*)exec_free_kernel<8, STATS, true> : (const void*)exec_free_kernel<8, STATS, false>;
        case 10: return MW ? (const void*)exec_free_kernel<10, STATS, true> : (const void*)exec_free_kernel<10, STATS, false>;
        case 12: return MW ? (const void*)exec_free_kernel<12, STATS, true> : (const void*)exec_free_kernel<12, STATS, false>;
        case 16: return MW ? (const void*)exec_free_kernel<16, STATS, true> : (const void*)exec_free_kernel<16, STATS, false>;
        case 20: return MW ? (const void*)exec_free_kernel<20, STATS, true> : (const void*)exec_free_kernel<20, STATS, false>;
        case 24: return MW ? (const void*)exec_free_kernel<24, STATS, true> : (const void*)exec_free_kernel<24, STATS, false>;
        case 25: return MW ? (const void*)exec_free_kernel<25, STATS, true> : (const void*)exec_free_kernel<25, STATS, false>;
        case 32: return MW ? (const void*)exec_free_kernel<32, STATS, true> : (const void*)exec_free_kernel<32, STATS, false>;
        case 40: return MW ? (const void*)exec_free_kernel<40, STATS, true> : (const void*)exec_free_kernel<40, STATS, false>;
        case 50: return MW ? (const void*)exec_free_kernel<50, STATS, true> : (const void*)exec_free_kernel<50, STATS, false>;
        default: return nullptr;
    }
}

template <bool STATS>
const void* free_lh_kernel_ptr(int V, int LH) {
    if (LH == 4) switch (V) {
        case 1: return (const void*)exec_free_lh_kernel<1, 4, STATS>;
        case 2: return (const void*)exec_free_lh_kernel<2, 4, STATS>;
        case 3: return (const void*)exec_free_lh_kernel<3, 4, STATS>;
        case 4: return (const void*)exec_free_lh_kernel<4, 4, STATS>;
        case 5: return (const void*)exec_free_lh_kernel<5, 4, STATS>;
        case 6: return (const void*)exec_free_lh_kernel<6, 4, STATS>;
        case 8: return (const void*)exec_free_lh_kernel<8, 4, STATS>;
        case 10: return (const void*)exec_free_lh_kernel<10, 4, STATS>;
        case 12: return (const void*)exec_free_lh_kernel<12, 4, STATS>;
        case 16: return (const void*)exec_free_lh_kernel<16, 4, STATS>;
        case 20: return (const void*)exec_free_lh_kernel<20, 4, STATS>;
        case 24: return (const void*)exec_free_lh_kernel<24, 4, STATS>;
        case 25: return (const void*)exec_free_lh_kernel<25, 4, STATS>;
        case 32: return (const void*)exec_free_lh_kernel<32, 4, STATS>;
        case 40: return (const void*)exec_free_lh_kernel<40, 4, STATS>;
        case 50: return (const void*)exec_free_lh_kernel<50, 4, STATS>;
        default: return nullptr;
    }
    if (LH == 2) switch (V) {
        case 1: return (const void*)exec_free_lh_kernel<1, 2, STATS>;
        case 2: return (const void*)exec_free_lh_kernel<2, 2, STATS>;
        case 3: return (const void*)exec_free_lh_kernel<3, 2, STATS>;
        case 4: return (const void*)exec_free_lh_kernel<4, 2, STATS>;
        case 5: return (const void*)exec_free_lh_kernel<5, 2, STATS>;
        case 6: return (const void*)exec_free_lh_kernel<6, 2, STATS>;
        case 8: return (const void*)exec_free_lh_kernel<8, 2, STATS>;
        case 10: return (const void*)exec_free_lh_kernel<10, 2, STATS>;
        case 12: return (const void*)exec_free_lh_kernel<12, 2, STATS>;
        case 16: return (const void*)exec_free_lh_kernel<16, 2, STATS>;
        case 20: return (const void*)exec_free_lh_kernel<20, 2, STATS>;
        case 24: return (const void*)exec_free_lh_kernel<24, 2, STATS>;
        case 25: return (const void*)exec_free_lh_kernel<25, 2, STATS>;
        case 32: return (const void*)exec_free_lh_kernel<32, 2, STATS>;
        case 40: return (const void*)exec_free_lh_kernel<40, 2, STATS>;
        case 50: return (const void*)exec_free_lh_kernel<50, 2, STATS>;
        default: return nullptr;
    }
    return nullptr;
}

template <bool STATS>
const void* free_pe_kernel_ptr(int V, int LH) {
    if (LH == 4) switch (V) {
        case 1: return (const void*)exec_free_pe_kernel<1, 4, STATS>;
        case 2: return (const void*)exec_free_pe_kernel<2, 4, STATS>;
        case 3: return (const void*)exec_free_pe_kernel<3, 4, STATS>;
        case 4: return (const void*)exec_free_pe_kernel<4, 4, STATS>;
        case 5: return (const void*)exec_free_pe_kernel<5, 4, STATS>;
        case 6: return (const void*)exec_free_pe_kernel<6, 4, STATS>;
        case 8: return (const void*)exec_free_pe_kernel<8, 4, STATS>;
        case 10: return (const void*)exec_free_pe_kernel<10, 4, STATS>;
        case 12: return (const void*)exec_free_pe_kernel<12, 4, STATS>;
        case 16: return (const void*)exec_free_pe_kernel<16, 4, STATS>;
        case 20: return (const void*)exec_free_pe_kernel<20, 4, STATS>;
        case 24: return (const void*)exec_free_pe_kernel<24, 4, STATS>;
        case 25: return (const void*)exec_free_pe_kernel<25, 4, STATS>;
        case 32: return (const void*)exec_free_pe_kernel<32, 4, STATS>;
        case 40: return (const void*)exec_free_pe_kernel<40, 4, STATS>;
        case 50: return (const void*)exec_free_pe_kernel<50, 4, STATS>;
        default: return nullptr;
    }
    if (LH == 2) switch (V) {
        case 1: return (const void*)exec_free_pe_kernel<1, 2, STATS>;
        case 2: return (const void*)exec_free_pe_kernel<2, 2, STATS>;
        case 3: return (const void*)exec_free_pe_kernel<3, 2, STATS>;
        case 4: return (const void*)exec_free_pe_kernel<4, 2, STATS>;
        case 5: return (const void*)exec_free_pe_kernel<5, 2, STATS>;
        case 6: return (const void*)exec_free_pe_kernel<6, 2, STATS>;
        case 8: return (const void*)exec_free_pe_kernel<8, 2, STATS>;
        case 10: return (const void*)exec_free_pe_kernel<10, 2, STATS>;
        case 12: return (const void*)exec_free_pe_kernel<12, 2, STATS>;
        case 16: return (const void*)exec_free_pe_kernel<16, 2, STATS>;
        case 20: return (const void*)exec_free_pe_kernel<20, 2, STATS>;
        case 24: return (const void*)exec_free_pe_kernel<24, 2, STATS>;
        case 25: return (const void*)exec_free_pe_kernel<25, 2, STATS>;
        case 32: return (const void*)exec_free_pe_kernel<32, 2, STATS>;
        case 40: return (const void*)exec_free_pe_kernel<40, 2, STATS>;
        case 50: return (const void*)exec_free_pe_kernel<50, 2, STATS>;
        default: return nullptr;
    }
    if (LH == 1) switch (V) {
        case 1: return (const void*)exec_free_pe_kernel<1, 1, STATS>;
        case 2: return (const void*)exec_free_pe_kernel<2, 1, STATS>;
        case 3: return (const void*)exec_free_pe_kernel<3, 1, STATS>;
        case 4: return (const void*)exec_free_pe_kernel<4, 1, STATS>;
        case 5: return (const void*)exec_free_pe_kernel<5, 1, STATS>;
        case 6: return (const void*)exec_free_pe_kernel<6, 1, STATS>;
        case 8: return (const void*)exec_free_pe_kernel<8, 1, STATS>;
        case 10: return (const void*)exec_free_pe_kernel<10, 1, STATS>;
        case 12: return (const void*)exec_free_pe_kernel<12, 1, STATS>;
        case 16: return (const void*)exec_free_pe_kernel<16, 1, STATS>;
        case 20: return (const void*)exec_free_pe_kernel<20, 1, STATS>;
        case 24: return (const void*)exec_free_pe_kernel<24, 1, STATS>;
        case 25: return (const void*)exec_free_pe_kernel<25, 1, STATS>;
        case 32: return (const void*)exec_free_pe_kernel<32, 1, STATS>;
        case 40: return (const void*)exec_free_pe_kernel<40, 1, STATS>;
        case 50: return (const void*)exec_free_pe_kernel<50, 1, STATS>;
        default: return nullptr;
    }
    return nullptr;
}

}  // namespace

// PE warps per CTA and the cluster size for `warps` PE warps: one warp per SM
// sub-partition while they fit 16 CTAs of 4, else 16 CTAs of up to
// kFreeMaxW warps.
bool free_layout(size_t warps, int* W_out, int* C_out) {
    if (warps < 2 || warps > size_t(kFreeMaxCluster) * kFreeMaxW) return false;
    int W = 4;
    if (warps > size_t(kFreeMaxCluster) * 4) {
        W = int((warps + kFreeMaxCluster - 1) / kFreeMaxCluster);
        W = W <= 4 ? 4 : 8;  // a multiple of every warps-per-PE (1, 2, 4)
    }
    *W_out = W;
    *C_out = int((warps + W - 1) / W);
    return true;
}

// The PE geometry K10 uses for P PEs of n points: Wp warps per PE (1, 2 or
// 4), Lc lanes per warp (2 <= Lc <= 32) and V points per lane, Wp*Lc*V = n.
// Step costs measured on B200 (tools/probe_k10.py, cycles per step): a
// one-warp PE in rounds with lane halos (q >= 4) ~140 + 8V for V >= 4 (halos
// from one lane away; V = 2-3: ~195, V = 1: ~224); one lane per PE (K10t)
// ~40 + 8n; the plain
// per-step kernel ~max(210, 150 + 8V); a PE over 2-4 warps (seams swapped
// every step) ~310 + 8V.  The cheapest geometry wins, as long as every PE
// warp keeps an SM sub-partition of its own (ties: fewer warps per PE).
// HEAT_K10_MAX_WP caps Wp (A/B).
bool free_geometry(size_t n, size_t P, size_t q, int* V_out, int* Lc_out, int* Wp_out) {
    static const int max_wp = [] {
        const char* e = std::getenv("HEAT_K10_MAX_WP");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    int best_V = 0, best_Lc = 0, best_Wp = 0, best_cost = 0;
    bool best_spread = false;
    for (int Wp : {1, 2, 4}) {
        if (Wp > max_wp || n % size_t(Wp) != 0) continue;
        const size_t m = n / size_t(Wp);
        int W, C;
        if (!free_layout(P * size_t(Wp), &W, &C)) continue;
        const bool spread = W == 4;  // one warp per SM sub-partition
        for (int V : kFreeV) {  // every V that fits (the cost is not monotone in V)
            if (m % size_t(V) != 0) continue;
            const size_t Lc = m / size_t(V);
            if (Lc < 1 || (Lc == 1 && Wp > 1)) break;
            if (Lc > 32) continue;
            // (one point per lane: halos from several lanes away, ~60 more)
            // one lane per PE (K10t): ~8n + 40
            const int cost = Wp > 1    ? 310 + 8 * V
                             : Lc == 1 ? 40 + 8 * V + (q >= 4 ? 0 : 60)
                             : (q >= 4 ? (V >= 4 ? 140 + 8 * V : V >= 2 ? 195 : 224)
                                       : std::max(210, 150 + 8 * V));
            const bool better = best_Wp == 0 || (spread && !best_spread) ||
                                (spread == best_spread && cost < best_cost);
            if (better) {
                best_V = V;
                best_Lc = int(Lc);
                best_Wp = Wp;
                best_cost = cost;
                best_spread = spread;
            }
        }
    }
    if (best_Wp == 0) return false;
    *V_out = best_V;
    *Lc_out = best_Lc;
    *Wp_out = best_Wp;
    return true;
}

// A Dirichlet field that fits ONE warp at >= 4 points per lane (N <= 128,
// e.g. the reference's measure() at N = 100): all PEs share that warp (K10w).
// Their edges move with the warp's own halo shuffles, so every PE reads its
// neighbours' current values -- no barrier, no ring, every delay 0 (the
// synchronous trajectory, which the free-running model allows) -- in K10r's
// rounds with the whole field as one segment.
bool free_one_warp(size_t N, int bc_kind, int* V_out, int* Lc_out) {
    if (bc_kind != HEAT_BC_DIRICHLET || std::getenv("HEAT_K10_NO_ONE_WARP")) return false;
    for (int V : kFreeV) {
        if (V > 5) return false;  // wider lanes: the PE warps of K10r/K10t are faster
        if (V < 4 || N % size_t(V) != 0) continue;
        const size_t Lc = N / size_t(V);
        if (Lc < 2) return false;
        if (Lc <= 32) {
            *V_out = V;
            *Lc_out = int(Lc);
            return true;
        }
    }
    return false;
}

bool free_eligible(size_t N, size_t per_pe, size_t q, size_t k_end) {
    int V, Lc, Wp, W, C;
    return q >= 1 && q <= size_t(kFreeMaxQ) && per_pe < N && N % per_pe == 0 &&
           k_end < size_t(1) << 31 &&
           free_geometry(per_pe, N / per_pe, q, &V, &Lc, &Wp) &&
           free_layout(N / per_pe * size_t(Wp), &W, &C) &&
           !std::getenv("HEAT_NO_FREE_CLUSTER");
}

// exec_run(BarrierFree) on K10: upload + validate + snap, one cluster launch
// (timed with events around it), download.  stats (kStat layout) optional.
int exec_free_run(DevCtx& d, const double* u0, size_t N, double r, int bc_kind, double c1,
                  double c2, size_t per_pe, size_t q, size_t k_end, double* field_out,
                  unsigned long long* stats_host, float* kernel_ms) {
    int V = 0, Lc = 0, Wp = 0, W = 0, C = 0;
    const bool one_warp = free_one_warp(N, bc_kind, &V, &Lc);
    if (one_warp) {
        Wp = 1;
        W = 1;
        C = 1;
    } else if (!free_geometry(per_pe, N / per_pe, q, &V, &Lc, &Wp) ||
               !free_layout(N / per_pe * size_t(Wp), &W, &C)) {
        return fail(HEAT_EINVAL, "exec_run: no K10 layout for this partition");
    }
    const size_t pitch = (N + 63) / 64 * 64;
    HB_TRY(ensure_buffers(d, pitch * sizeof(double)));
    double* field = static_cast<double*>(d.buf[0]);
    cudaStream_t st = d.stream;
    HB_TRY(upload_prepared(d, u0, N, bc_kind, c1, c2, field));
    HB_CUDA(cudaMemsetAsync(d.flag, 0, 4 * sizeof(unsigned int), st));
    unsigned long long* dstats = nullptr;
    if (stats_host) {
        HB_TRY(ensure_scratch(d, kStatWords * sizeof(unsigned long long)));
        dstats = static_cast<unsigned long long*>(d.scratch);
        HB_CUDA(cudaMemsetAsync(dstats, 0, kStatWords * sizeof(unsigned long long), st));
    }
    FreeArgs a{};
    a.field = field;
    a.n = one_warp ? int(N) : int(per_pe);  // K10w: the field is one segment
    a.P = one_warp ? 1 : int(N / per_pe);
    a.Lc = Lc;
    a.W = W;
    a.Wp = Wp;
    a.r = r;
    a.c = 1.0 - 2.0 * r;  // core.hpp:108
    a.c1 = c1;
    a.c2 = c2;
    a.dirichlet = bc_kind == HEAT_BC_DIRICHLET;
    a.k_end = (long long)k_end;
    a.q = int(q);
    a.flag = d.flag;
    a.stats = dstats;
    a.timeout_ns = 20ull * 1000000000ull;
    // single-warp PEs: rounds of LH steps with lane halos (K10r) when the
    // staleness bound allows LH <= q/2 and the halo fits one lane (V >= LH);
    // q <= 3 and V = 1 take the plain per-step kernel.  HEAT_K10_PLAIN=1: always plain.
    static const bool plain = std::getenv("HEAT_K10_PLAIN") != nullptr;
    const int LH = one_warp ? 4 : plain || Wp > 1 ? 0 : q >= 8 ? 4 : q >= 4 ? 2 : 0;
    const int LHt = q >= 8 ? 4 : q >= 4 ? 2 : 1;  // K10t rounds
    const void* fn =
        one_warp ? (stats_host ? (V == 4 ? (const void*)exec_free_lh_kernel<4, 4, true, false>
                                         : (const void*)exec_free_lh_kernel<5, 4, true, false>)
                               : (V == 4 ? (const void*)exec_free_lh_kernel<4, 4, false, false>
                                         : (const void*)exec_free_lh_kernel<5, 4, false, false>))
        : Lc == 1 ? (stats_host ? free_pe_kernel_ptr<true>(V, LHt) : free_pe_kernel_ptr<false>(V, LHt))
        : LH    ? (stats_host ? free_lh_kernel_ptr<true>(V, LH) : free_lh_kernel_ptr<false>(V, LH))
                : (stats_host ? free_kernel_ptr<true>(V, Wp > 1) : free_kernel_ptr<false>(V, Wp > 1));
    if (!fn) return fail(HEAT_ELOGIC, "K10: points per lane not compiled");
    const int smem = W * 2 * kFreeR * int(sizeof(FreeSlot));
    if (C > 8) HB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(C));
    cfg.blockDim = dim3(unsigned(32 * W));
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* params[] = {&a};
    EventPair ev;
    HB_TRY(ev.begin(st));
    HB_CUDA(cudaLaunchKernelExC(&cfg, fn, params));
    HB_TRY(ev.end(st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    HB_CUDA(cudaMemcpyAsync(field_out, field, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    unsigned int flags[4] = {0, 0, 0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, d.flag, sizeof flags, cudaMemcpyDeviceToHost, st));
    if (stats_host)
        HB_CUDA(cudaMemcpyAsync(stats_host, dstats, kStatWords * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    if (kernel_ms) HB_TRY(ev.elapsed(kernel_ms));
    if (flags[1]) return fail(HEAT_ECUDA, "exec_run: K10 watchdog fired (a PE stopped advancing)");
    if (flags[0]) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    return HEAT_OK;
}

}  // namespace hb

extern "C" int heat_free_geometry(size_t N, size_t per_pe, size_t q, int* points_per_lane,
                                  int* lanes, int* warps_per_cta, int* cluster, int* warps_per_pe) {
    int V = 0, Lc = 0, Wp = 0, W = 0, C = 0;
    if (hb::free_eligible(N, per_pe, q, 1) && hb::free_one_warp(N, HEAT_BC_DIRICHLET, &V, &Lc)) {
        // K10w (Dirichlet fields of <= 128 points): one warp holds the field
        if (points_per_lane) *points_per_lane = V;
        if (lanes) *lanes = Lc;
        if (warps_per_cta) *warps_per_cta = 1;
        if (cluster) *cluster = 1;
        if (warps_per_pe) *warps_per_pe = 0;  // all PEs share the warp
        return HEAT_OK;
    }
    const bool ok = hb::free_eligible(N, per_pe, q, 1) &&
                    hb::free_geometry(per_pe, N / per_pe, q, &V, &Lc, &Wp) &&
                    hb::free_layout(N / per_pe * size_t(Wp), &W, &C);
    if (points_per_lane) *points_per_lane = ok ? V : 0;
    if (lanes) *lanes = ok ? Lc : 0;
    if (warps_per_cta) *warps_per_cta = ok ? W : 0;
    if (cluster) *cluster = ok ? C : 0;
    if (warps_per_pe) *warps_per_pe = ok ? Wp : 0;
    return ok ? HEAT_OK : HEAT_EINVAL;
}
