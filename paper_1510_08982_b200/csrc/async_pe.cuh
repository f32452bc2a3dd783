// async_pe.cuh -- K3/K4: asynchronous FTCS with one WARP per processing
// element (PE), PEs exchanging their boundary values through halo rings
// under acquire/release flags -- no grid-wide or block-wide barrier.
//
// Replaces (GPU-side):
//   * async_step_into / AsyncSimulator / async_run (async_sim.cpp:77-160)
//     in DETERMINISTIC mode: every cross-PE read u_j(k - d) uses exactly the
//     delay d the reference draws for it.  The reference's single sequential
//     SplitMix64 stream is replayed per PE in counter form: the draw for the
//     read with in-step rank `off` at step k is draw number k*D + off of the
//     stream (D = cross-PE reads per step), i.e. mix(seed + (k*D+off+1)*gamma)
//     (rng.hpp:20-26, async_sim.cpp:57-73, draw order async_sim.cpp:86-101).
//   * run_barrier_free (async_exec.cpp:156-259) in FREE mode: a PE reads the
//     newest published neighbour value u_j(k*) with k - k* <= q - 1 (bounded
//     staleness, the paper's Eq. (4) with k* in {k, ..., k-q+1}); it only
//     waits when the neighbour is more than q-1 steps behind.  Observed
//     delays k - k* are logged.
//
// Mapping: PE p = warp p (global warp index).  Its n <= 32*V points live in
// registers for the whole launch: lane l holds local points [lV, lV+V).
// Per step a PE needs the LEFT neighbour's last point and the RIGHT
// neighbour's first point; it publishes its own first and last point for
// step k+1 into ring slot (k+1) mod R and then releases prog[p] = k+1.
// Rings live in shared memory (CTA scope) when all PEs fit in one CTA, else
// in global memory (GPU scope).  The ring/progress state persists in global
// memory between launches, so runs can be split at recorded steps.
//
// Flow control: a producer may overwrite the slot of step k+1-R only when
// every consumer has reached step >= k+1+q-R (it never reads older than
// k_c-q+1).  Deadlock freedom requires all P warps to be co-resident
// (single CTA, or a cooperative launch).  Spins carry a %globaltimer
// watchdog that aborts the whole grid with HEAT_ETIMEOUT.
#pragma once

#include "common.cuh"

namespace hb {

struct AsyncPeArgs {
    double* field;  // N doubles; PE p reads/writes only [p*n, (p+1)*n)
    long long N;
    int n;
    int P;
    double r, c, c1, c2;
    int dirichlet;
    long long k0, k1;  // steps [k0, k1) of this launch
    int mode;          // 0 deterministic replay, 1 free-running (bounded)
    int q;             // delays in {0, ..., q-1}
    int R;             // ring slots per PE side (power of two, > q)
    int law;           // HEAT_DELAY_*
    int fixed_d;
    unsigned long long seed;
    ModQ modq;              // x mod q (uniform law, steps k >= q-1)
    long long D;            // cross-PE reads (draws) per step
    const int* off_left;    // [P] in-step draw rank of the first point's left read, -1 none
    const int* off_right;   // [P] ... of the last point's right read, -1 none
    const uint64_t* gthr;         // GEOMETRIC: the q-1 delay thresholds (geometric_thresholds)
    double* ring;                 // [P][2][R]: side 0 = first point, 1 = last point
    unsigned long long* prog;     // [P] published step count
    unsigned long long* stats;    // see kStat* offsets
    double* edge_log;             // optional [(k_total+1)][P][2] published edge values
    int* used_log;                // optional [k_total][P][2] step k* actually read
    unsigned int* flag;           // [0] non-finite, [1] watchdog timeout
    unsigned int* abort_word;     // set on timeout: every spin bails out
    unsigned long long timeout_ns;
    // optional in-kernel trajectory: snapshot j (j >= 1) of the run lands at
    // snaps[j*N ...]; recorded steps are multiples of snap_stride plus k_final
    double* snaps;
    long long snap_stride;
    long long k_final;
    int seg;  // lanes per PE (a power of two, 2..32): 32/seg PEs share a warp
};

// off_left/off_right value of an edge between two units of the same PE (a
// PE wider than one warp's 1024 points runs as several units, see
// async_pe_run): exact, no draw
constexpr int kUnitEdge = -2;

// stats layout (u64 words)
constexpr int kStatReads = 0, kStatWaits = 1, kStatMaxDelay = 2, kStatDelayHist = 3,
              kStatLagMin = 67, kStatLagMax = 68, kStatLagHist = 69, kStatLagOverflow = 133,
              kStatWords = 134;

template <bool kShared>
struct RingOps;

template <>
struct RingOps<false> {
    static __device__ __forceinline__ uint64_t load_prog(const uint64_t* p) { return ld_acquire_gpu(p); }
    static __device__ __forceinline__ void store_prog(uint64_t* p, uint64_t v) { st_release_gpu(p, v); }
    static __device__ __forceinline__ double load_val(const double* p) { return ld_relaxed_gpu_f64(p); }
    static __device__ __forceinline__ void store_val(double* p, double v) { st_relaxed_gpu_f64(p, v); }
};

template <>
struct RingOps<true> {
    static __device__ __forceinline__ uint64_t load_prog(const uint64_t* p) {
        return ld_acquire_cta_shared(p);
    }
    static __device__ __forceinline__ void store_prog(uint64_t* p, uint64_t v) {
        st_release_cta_shared(p, v);
    }
    static __device__ __forceinline__ double load_val(const double* p) {
        return *reinterpret_cast<const volatile double*>(p);
    }
    static __device__ __forceinline__ void store_val(double* p, double v) {
        *reinterpret_cast<volatile double*>(p) = v;
    }
};

// Delay of the draw with in-step rank `off` at step k (async_sim.cpp:57-73).

__device__ __forceinline__ int det_delay(const AsyncPeArgs& a, long long k, int off) {
    const long long bound = k < (long long)(a.q - 1) ? k : (long long)(a.q - 1);
    if (bound == 0) return 0;  // every law yields 0 (the draw is still "consumed" by index)
    if (a.law == 1) return a.fixed_d < bound ? a.fixed_d : int(bound);
    const uint64_t x = splitmix_draw(a.seed, uint64_t(k) * uint64_t(a.D) + uint64_t(off));
    if (a.law == 0) return uniform_delay(x, bound, a.modq);
    return geometric_delay(x, a.gthr, int(bound));
}

// Spin until prog[pe] >= need (acquire).  Returns the observed progress, or
// ~0ull when the watchdog fired.
template <bool kShared>
__device__ __forceinline__ uint64_t wait_prog(const AsyncPeArgs& a, const uint64_t* prog,
                                              long long need, bool* waited) {
    uint64_t v = RingOps<kShared>::load_prog(prog);
    if ((long long)v >= need) return v;
    *waited = true;
    const uint64_t t0 = globaltimer_ns();
    unsigned spins = 0;
    while ((long long)(v = RingOps<kShared>::load_prog(prog)) < need) {
        if ((++spins & 255u) == 0) {
            if (*reinterpret_cast<volatile unsigned int*>(a.abort_word)) return ~0ull;
            if (globaltimer_ns() - t0 > a.timeout_ns) {
                atomicOr(a.flag + 1, 1u);
                atomicExch(a.abort_word, 1u);
                return ~0ull;
            }
        }
    }
    return v;
}

// Ring state at step 0: slot 0 of every PE's two rings holds its step-0 edge
// values, prog = 0 (everything else zero); the edge log gets step 0 too.
static __global__ void async_init_kernel(const double* __restrict__ field, int n, int P, int R,
                                  double* ring, unsigned long long* prog, double* edge_log) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)P * 2 * R;
         i += (long long)gridDim.x * blockDim.x) {
        const long long ps = i / R;  // p*2 + side
        const int slot = int(i % R);
        const long long p = ps >> 1;
        double v = 0.0;
        if (slot == 0) v = field[p * n + ((ps & 1) ? n - 1 : 0)];
        ring[i] = v;
        if (slot == 0 && edge_log) edge_log[ps] = v;
        if (slot == 0 && (ps & 1) == 0) prog[p] = 0;
    }
}

// kBarrier (single CTA, deterministic mode only): the PEs advance in
// lockstep with one block barrier per step -- the GPU analogue of
// run_barriered (async_exec.cpp:57-114).  Every value a deterministic read
// can ask for (step k-d <= k) was published before the previous barrier, so
// no progress flags are needed; results are identical to the flag protocol.
template <int V, bool kShared, bool kBarrier>
__global__ void __launch_bounds__(kShared ? 512 : 256) async_pe_kernel(const AsyncPeArgs a) {
    static_assert(kShared || !kBarrier, "barrier mode needs every PE in one CTA");
    extern __shared__ __align__(16) unsigned char smem[];
    // A PE is a segment of S lanes; the warp's 32/S segments are independent
    // PEs, and every shuffle is confined to its segment (width S).
    const int S = a.seg;
    const int wl = threadIdx.x & 31;  // lane in the warp
    const int lane = wl & (S - 1);    // lane in the PE's segment
    const int p = int(((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5) * (32 / S) + wl / S);
    const int R = a.R;
    double* ring = a.ring;
    uint64_t* prog = reinterpret_cast<uint64_t*>(a.prog);
    if constexpr (kShared) {
        // stage the persistent ring state into shared memory (one CTA holds every PE)
        double* sring = reinterpret_cast<double*>(smem);
        uint64_t* sprog = reinterpret_cast<uint64_t*>(sring + (size_t)a.P * 2 * R);
        for (int i = threadIdx.x; i < a.P * 2 * R; i += blockDim.x) sring[i] = a.ring[i];
        for (int i = threadIdx.x; i < a.P; i += blockDim.x) sprog[i] = a.prog[i];
        __syncthreads();
        ring = sring;
        prog = sprog;
    }
    const bool active = p < a.P;
    if constexpr (!kShared) {
        // no block barrier in the global-ring variant; inactive segments of a
        // partly active warp stay for the shuffles (their writes are guarded)
        if (!__any_sync(0xffffffffu, active)) return;
    }
    // [0,64) delay histogram, [64,128) writer-lag histogram, [128] lag overflow
    __shared__ unsigned int s_hist[16][129];
    unsigned int* whist = s_hist[(threadIdx.x >> 5) & 15];
    for (int i = wl; i < 129; i += 32) whist[i] = 0;
    __syncwarp();
    const int n = a.n;
    const long long lo = (long long)p * n;
    const double r = a.r, c = a.c;
    using A = Arith<double>;

    // neighbours (periodic wraps, Dirichlet ends have none); P >= 2 here
    const int lpe = p > 0 ? p - 1 : (a.dirichlet ? -1 : a.P - 1);
    const int rpe = p + 1 < a.P ? p + 1 : (a.dirichlet ? -1 : 0);
    const bool pin_first = a.dirichlet && p == 0;
    const bool pin_last = a.dirichlet && p == a.P - 1;
    const bool needL = active && lpe >= 0 && !pin_first;
    const bool needR = active && rpe >= 0 && !pin_last;
    const int offL = active ? a.off_left[p] : -1;
    const int offR = active ? a.off_right[p] : -1;
    const int lastLane = (n - 1) / V, lastElem = (n - 1) % V;

    double u[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int li = lane * V + i;
        u[i] = (active && li < n) ? a.field[lo + li] : 0.0;
    }

    unsigned long long reads = 0, waits = 0, maxd = 0, lag_min = ~0ull, lag_max = 0;
    // next recorded step and its snapshot index (no per-step 64-bit division)
    long long next_snap = 0, next_snap_idx = 0;
    if (a.snaps) {
        next_snap_idx = a.k0 / a.snap_stride + 1;
        next_snap = next_snap_idx * a.snap_stride;
    }
    // Lane 0 fetches the left ghost (left PE's LAST point), lane 31 the right
    // ghost (right PE's FIRST point); lane 0 publishes.  Everything a step
    // touches is precomputed here so the loop body stays short: the paper's
    // regime is latency-bound (one neighbour handshake per step).
    const bool fetch = (lane == 0 && needL) || (lane == S - 1 && needR);
    const int nb = lane == 0 ? lpe : rpe;
    const double* gring = ring + ((size_t)(nb < 0 ? 0 : nb) * 2 + (lane == 0 ? 1 : 0)) * R;
    const uint64_t* gprog = prog + (nb < 0 ? 0 : nb);
    const int my_off = lane == 0 ? offL : offR;
    // an edge between two units of one PE (kUnitEdge): read the neighbour's
    // value of the same step, no draw (the PE is synchronous inside)
    const bool exact_edge = my_off == kUnitEdge;
    double* my0 = ring + (size_t)(active ? p : 0) * 2 * R;
    double* my1 = my0 + R;
    const bool stats = a.stats != nullptr;
    const int rmask = R - 1;
    bool abort = false;
    const int k1 = int(a.k1);
    for (int k = int(a.k0); k < k1; ++k) {
        // ---- 1. ghosts
        double ghost = 0.0;
        if (fetch) {
            bool waited = false;
            int m;
            uint64_t v;
            if (kBarrier) {
                m = exact_edge ? k : k - det_delay(a, k, my_off);
                v = uint64_t(k);  // lockstep: the neighbour has published step k
            } else if (a.mode == 0 || exact_edge) {
                m = exact_edge ? k : k - det_delay(a, k, my_off);
                v = wait_prog<kShared>(a, gprog, m, &waited);
            } else {
                v = wait_prog<kShared>(a, gprog, k - (a.q - 1), &waited);
                m = (long long)v < k ? int(v) : k;
            }
            if (v == ~0ull) {
                abort = true;
            } else {
                ghost = RingOps<kShared>::load_val(gring + (m & rmask));
                if (stats && !exact_edge) {
                    const unsigned used = unsigned(k - m);
                    // writer lag as LagStats measures it: producer progress - step consumed
                    const unsigned long long lag = v - (unsigned long long)m;
                    reads++;
                    waits += waited;
                    maxd = used > maxd ? used : maxd;
                    lag_min = lag < lag_min ? lag : lag_min;
                    lag_max = lag > lag_max ? lag : lag_max;
                    // per-warp shared histograms (a global atomic here would sit
                    // in front of every release of the publish step below)
                    atomicAdd(&whist[used < 64 ? used : 63], 1u);
                    atomicAdd(&whist[64 + (lag < 64 ? lag : 64)], 1u);
                }
                if (a.used_log) a.used_log[((size_t)k * a.P + p) * 2 + (lane == 0 ? 0 : 1)] = m;
            }
        }
        if constexpr (!kBarrier) {
            if (__any_sync(0xffffffffu, abort)) {
                abort = true;
                break;
            }
        }
        const double gL = __shfl_sync(0xffffffffu, ghost, 0, S);
        const double gR = __shfl_sync(0xffffffffu, ghost, S - 1, S);

        // ---- 2. one step of the PE's points.  The PE's last point (lane
        // lastLane, element lastElem) takes r*gR as its right product; a
        // per-element select keeps u[] in registers (a dynamic index would
        // push it to local memory on the critical path).
        const double pG = A::mul(r, gR);
        const bool last_lane = lane == lastLane;
        const double pFirst = A::mul(r, u[0]);
        const double pLast = A::mul(r, u[V - 1]);
        double pL = __shfl_up_sync(0xffffffffu, pLast, 1, S);
        double pR = __shfl_down_sync(0xffffffffu, pFirst, 1, S);
        if (lane == 0) pL = A::mul(r, gL);
        {
            double pm1 = pL, p0 = pFirst;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                double p1;
                if (i + 1 == V)
                    p1 = pR;
                else if (i + 1 == V - 1)
                    p1 = pLast;
                else
                    p1 = A::mul(r, u[i + 1]);
                if (last_lane && i == lastElem) p1 = pG;
                const double cs = A::mul(c, u[i]);
                u[i] = stencil_p(p1, cs, pm1);
                if (pin_last && last_lane && i == lastElem) u[i] = a.c2;
                pm1 = p0;
                p0 = p1;
            }
        }
        if (pin_first && lane == 0) u[0] = a.c1;

        // ---- 3. publish u_first(k+1), u_last(k+1), then release prog = k+1.
        // No flow control: the two sides of a boundary read each other, so
        // neither gets more than q-1 steps ahead, and R >= 4q slots cannot be
        // overwritten while still readable.
        double last = 0.0;
#pragma unroll
        for (int i = 0; i < V; ++i)
            if (i == lastElem) last = u[i];
        last = __shfl_sync(0xffffffffu, last, lastLane, S);
        if (lane == 0 && active) {
            const int slot = (k + 1) & rmask;
            RingOps<kShared>::store_val(my0 + slot, u[0]);
            RingOps<kShared>::store_val(my1 + slot, last);
            if (a.edge_log) {
                a.edge_log[((size_t)(k + 1) * a.P + p) * 2 + 0] = u[0];
                a.edge_log[((size_t)(k + 1) * a.P + p) * 2 + 1] = last;
            }
            if (!kBarrier) RingOps<kShared>::store_prog(prog + p, (uint64_t)(k + 1));
        }
        if (a.snaps && active) {
            const long long kk = k + 1;
            long long j = -1;
            if (kk == next_snap) {
                j = next_snap_idx++;
                next_snap += a.snap_stride;
            } else if (kk == a.k_final) {
                j = a.k_final / a.snap_stride + 1;
            }
            if (j >= 0) {
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    const int li = lane * V + i;
                    if (li < n) a.snaps[j * a.N + lo + li] = u[i];
                }
            }
        }
        if constexpr (kBarrier) __syncthreads();  // step k+1 published by every PE
    }
    if (kBarrier && lane == 0 && active) prog[p] = uint64_t(a.k1);

    // ---- results, finite check, statistics, ring state back to global
    bool bad = false;
    if (active && !abort) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const int li = lane * V + i;
            if (li < n) {
                a.field[lo + li] = u[i];
                bad |= !isfinite(u[i]);
            }
        }
    }
    if (bad) atomicOr(a.flag, 1u);
    __syncwarp();
    if (a.stats) {
        for (int i = wl; i < 129; i += 32) {
            const unsigned int cnt = whist[i];
            if (cnt) atomicAdd(a.stats + (i < 64 ? kStatDelayHist + i : kStatLagHist + (i - 64)),
                               (unsigned long long)cnt);
        }
    }
    if (a.stats && reads) {
        atomicAdd(a.stats + kStatReads, reads);
        atomicAdd(a.stats + kStatWaits, waits);
        atomicMax(a.stats + kStatMaxDelay, maxd);
        atomicMin(a.stats + kStatLagMin, lag_min);
        atomicMax(a.stats + kStatLagMax, lag_max);
    }
    if constexpr (kShared) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.P * 2 * R; i += blockDim.x) a.ring[i] = ring[i];
        for (int i = threadIdx.x; i < a.P; i += blockDim.x) a.prog[i] = prog[i];
    }
}

}  // namespace hb
