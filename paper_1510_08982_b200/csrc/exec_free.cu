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
__device__ __forceinline__ void st_cluster_slot(uint32_t addr, unsigned long long lo,
                                                unsigned long long hi) {
    asm volatile("st.relaxed.cluster.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(lo),
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

template <int V, bool STATS>
__global__ void __launch_bounds__(kFreeMaxW * 32, 1) exec_free_kernel(const FreeArgs a) {
    extern __shared__ __align__(16) FreeSlot rings[];  // [W][2 sides][kFreeR]
    const int W = a.W;
    const uint32_t cta = cluster_ctarank();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = int(cta) * W + w;
    const bool active = w < W && p < a.P;  // warp-uniform
    const int n = a.n, P = a.P, Lc = a.Lc;
    // invalidate every slot of this CTA's rings (tag 0xffffffff = no step)
    for (int i = threadIdx.x; i < W * 2 * kFreeR; i += blockDim.x)
        rings[i] = FreeSlot{~0ull, ~0ull};
    cluster_sync_all();  // no producer may write a slot before its owner cleared it

    const double r = a.r, c = a.c;
    using A = Arith<double>;
    const bool dir = a.dirichlet != 0;
    const int lpe = p > 0 ? p - 1 : (dir ? -1 : P - 1);
    const int rpe = p + 1 < P ? p + 1 : (dir ? -1 : 0);
    const bool needL = active && lpe >= 0;  // Dirichlet PE 0 / P-1 have a pinned end instead
    const bool needR = active && rpe >= 0;
    const bool first_lane = lane == 0, last_lane = lane == Lc - 1;
    const bool pin_first = active && dir && p == 0 && first_lane;
    const bool pin_last = active && dir && p == P - 1 && last_lane;

    // lane 0 reads ring side 0 (left neighbour's last point) and publishes its
    // first point into the left neighbour's side-1 ring; lane Lc-1 mirrors it
    const bool edge = (first_lane && needL) || (last_lane && needR);
    const int side = first_lane ? 0 : 1;
    const int nb = first_lane ? lpe : rpe;
    const uint32_t my_ring =
        smem_u32(rings + ((size_t)(active ? w : 0) * 2 + side) * kFreeR);
    uint32_t peer_ring = 0;
    if (edge) {
        const int nb_cta = nb / W, nb_w = nb % W;
        const uint32_t local = smem_u32(rings + ((size_t)nb_w * 2 + (1 - side)) * kFreeR);
        peer_ring = map_cluster(local, uint32_t(nb_cta));
    }

    double u[V];
    const long long base = (long long)p * n + (long long)lane * V;
#pragma unroll
    for (int i = 0; i < V; ++i) u[i] = (active && lane < Lc) ? a.field[base + i] : 0.0;
    if (pin_first) u[0] = a.c1;  // prepare_initial snapped them already; keep exact
    if (pin_last) u[V - 1] = a.c2;

    // step-0 edge values
    if (edge) {
        const double v = first_lane ? u[0] : u[V - 1];
        st_cluster_slot(peer_ring, pack_half(0, uint32_t(__double2loint(v))),
                        pack_half(0, uint32_t(__double2hiint(v))));
    }

    long long m = -1;  // newest neighbour step seen (per edge lane)
    double g = 0.0;    // its value
    unsigned long long reads = 0, waits = 0, maxd = 0;
    __shared__ unsigned int s_hist[64];
    if (STATS) {
        for (int i = threadIdx.x; i < 64; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
    }
    bool abort = false;
    const long long qm1 = a.q - 1;
    if (active) {
        for (long long k = 0; k < a.k_end; ++k) {
            // ---- ghost: the exact value (slot k) or the next unseen one (m+1)
            if (edge) {
                const uint32_t tk = uint32_t(k);
                const FreeSlot sk = ld_slot(my_ring + uint32_t(k & (kFreeR - 1)) * 16u);
                const FreeSlot sn = ld_slot(my_ring + uint32_t((m + 1) & (kFreeR - 1)) * 16u);
                if (slot_is(sk, tk)) {
                    m = k;
                    g = slot_value(sk);
                } else if (slot_is(sn, uint32_t(m + 1))) {
                    ++m;
                    g = slot_value(sn);
                }
                if (k - m > qm1) {  // too stale: wait for the neighbour (bounded delay)
                    if (STATS) ++waits;
                    const uint64_t t0 = globaltimer_ns();
                    unsigned spins = 0;
                    while (k - m > qm1) {
                        const FreeSlot s = ld_slot(my_ring + uint32_t((m + 1) & (kFreeR - 1)) * 16u);
                        if (slot_is(s, uint32_t(m + 1))) {
                            ++m;
                            g = slot_value(s);
                        } else if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > a.timeout_ns) {
                            atomicOr(a.flag + 1, 1u);
                            abort = true;
                            break;
                        }
                    }
                }
                if (STATS) {
                    const unsigned long long d = (unsigned long long)(k - m);
                    ++reads;
                    maxd = d > maxd ? d : maxd;
                    atomicAdd(&s_hist[d < 64 ? d : 63], 1u);
                }
            }
            if (__any_sync(0xffffffffu, abort)) break;
            // ---- one Jacobi step of the PE's points; the ghost products enter
            // at the PE's two ends (lane 0's left, lane Lc-1's right)
            const double pFirst = A::mul(r, u[0]);
            const double pLast = A::mul(r, u[V - 1]);
            const double up = __shfl_up_sync(0xffffffffu, pLast, 1);
            const double dn = __shfl_down_sync(0xffffffffu, pFirst, 1);
            const double pg = A::mul(r, g);
            const double pL = first_lane ? pg : up;
            const double pR = last_lane ? pg : dn;
            chunk_step<double, V>(u, r, c, pL, pR, pFirst, pLast);
            if (pin_first) u[0] = a.c1;
            if (pin_last) u[V - 1] = a.c2;
            // ---- publish step k+1's edge value into the neighbour's ring
            if (edge) {
                const double v = first_lane ? u[0] : u[V - 1];
                const uint32_t t = uint32_t(k + 1);
                st_cluster_slot(peer_ring + uint32_t((k + 1) & (kFreeR - 1)) * 16u,
                                pack_half(t, uint32_t(__double2loint(v))),
                                pack_half(t, uint32_t(__double2hiint(v))));
            }
        }
    }
    // a watchdog abort anywhere ends every PE (their neighbours would spin)
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
            atomicAdd(a.stats + kStatReads, reads);
            atomicAdd(a.stats + kStatWaits, waits);
            atomicMax(a.stats + kStatMaxDelay, maxd);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 64; i += blockDim.x)
            if (s_hist[i]) atomicAdd(a.stats + kStatDelayHist + i, (unsigned long long)s_hist[i]);
    }
    cluster_sync_all();  // no CTA leaves while a peer may still store into its shared memory
}

// Points per lane compiled in; a PE of n points runs as Lc = n / V lanes.
constexpr int kFreeV[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 25, 32, 40};

template <bool STATS>
const void* free_kernel_ptr(int V) {
    switch (V) {
        case 1: return (const void*)exec_free_kernel<1, STATS>;
        case 2: return (const void*)exec_free_kernel<2, STATS>;
        case 3: return (const void*)exec_free_kernel<3, STATS>;
        case 4: return (const void*)exec_free_kernel<4, STATS>;
        case 5: return (const void*)exec_free_kernel<5, STATS>;
        case 6: return (const void*)exec_free_kernel<6, STATS>;
        case 8: return (const void*)exec_free_kernel<8, STATS>;
        case 10: return (const void*)exec_free_kernel<10, STATS>;
        case 12: return (const void*)exec_free_kernel<12, STATS>;
        case 16: return (const void*)exec_free_kernel<16, STATS>;
        case 20: return (const void*)exec_free_kernel<20, STATS>;
        case 24: return (const void*)exec_free_kernel<24, STATS>;
        case 25: return (const void*)exec_free_kernel<25, STATS>;
        case 32: return (const void*)exec_free_kernel<32, STATS>;
        case 40: return (const void*)exec_free_kernel<40, STATS>;
        default: return nullptr;
    }
}

}  // namespace

// The PE geometry K10 uses for PEs of n points: V points per lane, Lc = n / V
// lanes (2 <= Lc <= 32), the smallest compiled V that fits; false if none.
bool free_geometry(size_t n, int* V_out, int* Lc_out) {
    for (int V : kFreeV) {
        if (n % size_t(V) != 0) continue;
        const size_t Lc = n / size_t(V);
        if (Lc < 2) break;
        if (Lc <= 32) {
            *V_out = V;
            *Lc_out = int(Lc);
            return true;
        }
    }
    return false;
}

// PE warps per CTA and the cluster size: one warp per SM sub-partition while
// the PEs fit 16 CTAs of 4, else 16 CTAs of up to kFreeMaxW warps.
bool free_layout(size_t P, int* W_out, int* C_out) {
    if (P < 2 || P > size_t(kFreeMaxCluster) * kFreeMaxW) return false;
    int W = 4;
    if (P > size_t(kFreeMaxCluster) * 4) W = int((P + kFreeMaxCluster - 1) / kFreeMaxCluster);
    *W_out = W;
    *C_out = int((P + W - 1) / W);
    return true;
}

bool free_eligible(size_t N, size_t per_pe, size_t q) {
    int V, Lc, W, C;
    return q >= 1 && q <= size_t(kFreeMaxQ) && per_pe < N && N % per_pe == 0 &&
           free_geometry(per_pe, &V, &Lc) && free_layout(N / per_pe, &W, &C) &&
           !std::getenv("HEAT_NO_FREE_CLUSTER");
}

// exec_run(BarrierFree) on K10: upload + validate + snap, one cluster launch
// (timed with events around it), download.  stats (kStat layout) optional.
int exec_free_run(DevCtx& d, const double* u0, size_t N, double r, int bc_kind, double c1,
                  double c2, size_t per_pe, size_t q, size_t k_end, double* field_out,
                  unsigned long long* stats_host, float* kernel_ms) {
    int V = 0, Lc = 0, W = 0, C = 0;
    if (!free_geometry(per_pe, &V, &Lc) || !free_layout(N / per_pe, &W, &C))
        return fail(HEAT_EINVAL, "exec_run: no K10 layout for this partition");
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
    a.n = int(per_pe);
    a.P = int(N / per_pe);
    a.Lc = Lc;
    a.W = W;
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
    const void* fn = stats_host ? free_kernel_ptr<true>(V) : free_kernel_ptr<false>(V);
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
                                  int* lanes, int* warps_per_cta, int* cluster) {
    int V = 0, Lc = 0, W = 0, C = 0;
    const bool ok = hb::free_eligible(N, per_pe, q) && hb::free_geometry(per_pe, &V, &Lc) &&
                    hb::free_layout(N / per_pe, &W, &C);
    if (points_per_lane) *points_per_lane = ok ? V : 0;
    if (lanes) *lanes = ok ? Lc : 0;
    if (warps_per_cta) *warps_per_cta = ok ? W : 0;
    if (cluster) *cluster = ok ? C : 0;
    return ok ? HEAT_OK : HEAT_EINVAL;
}
