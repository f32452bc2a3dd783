// async_stream.cuh -- K5: asynchronous FTCS at scale (PEs far wider than a
// warp), one persistent launch for the whole run, no grid-wide barrier.
//
// Semantics (async_sim.cpp:77-106 / Eq. (4) of the paper): the field is split
// into P contiguous PEs of n points.  Inside a PE every read is synchronous
// (Jacobi); the first point of PE p reads the LAST point of PE p-1 at step
// k - d, the last point reads the FIRST point of PE p+1 at step k - d, with d
// replayed from the reference's SplitMix64 stream (deterministic mode, bit-
// exact with async_run) or the newest value within the bound q (free mode).
//
// Execution: each PE's slab is cut into K1 tiles (32V - 64 exact points,
// V = 48 by default, 32-point halo) advanced s <= 32 steps per HBM pass with
// redundant halo recompute (the same
// warp_step, TMA tensor loads/stores and 128B-swizzled buffers as K1).  Work
// items (pass, tile) are handed out in pass-major order by one atomic counter;
// a tile may start pass pi once its same-PE neighbours finished pass pi-1
// (per-tile pass counters, acquire/release) -- a local dependency, never a
// barrier.  The two tiles at a PE boundary inject the neighbour's value into
// the stencil every step: the lanes holding the PE's first and last point
// (an element cut inside the lane) spin on the neighbour's progress counter, read the edge ring
// slot, and publish their own new edge value + progress (release).  Within a
// pass the boundary tiles are handed out first, in (right edge of PE b, left
// edge of PE b+1) pairs, so every pair that handshakes is co-resident and the
// kernel cannot deadlock with >= 2 warps.
//
// Rings: ringL[p][R] = history of PE p's first point, ringR[p][R] of its last
// point, progL/progR = published step counts.  The two sides of a boundary
// read each other, so neither runs more than q-1 steps ahead of the other and
// R >= 2q + 2 slots can never be overwritten while still readable.
#pragma once

#include "async_pe.cuh"
#include "sync_tb.cuh"

namespace hb {

// Where a PE's boundary tiles read their neighbours' edge histories and where
// they publish their own (built on the host).  Within one device every link
// points into the local rings (GPU scope).  At a device boundary the reader
// owns a receive ring that the neighbour device fills with P2P stores over
// NVLink (system scope), so every load stays local and NCCL only sets up.
enum : int {
    kLinkSrcLSys = 1,   // srcL/progL_src are written by another device
    kLinkSrcRSys = 2,
    kLinkPubF1Sys = 4,  // pubF[1] lives on another device
    kLinkPubL1Sys = 8,
};
struct PeLink {
    const double* srcL;                 // left neighbour's LAST-point history (null: none)
    const unsigned long long* progL_src;
    const double* srcR;                 // right neighbour's FIRST-point history
    const unsigned long long* progR_src;
    double* pubF[2];                    // rings mirroring this PE's first point
    unsigned long long* pubF_prog[2];
    double* pubL[2];                    // rings mirroring this PE's last point
    unsigned long long* pubL_prog[2];
    int flags;
};

struct AsyncStreamArgs {
    double* buf[2];  // ping-pong fields (pass pi reads buf[pi & 1])
    long long N;
    long long n;   // points per PE (multiple of V)
    int P;
    int Tp;        // tiles per PE (>= 2)
    double r, c, c1, c2;
    int dirichlet;
    long long k0;  // absolute step of the first pass
    long long steps;
    int s;         // steps per pass (<= V)
    long long npass;
    int mode;      // 0 deterministic, 1 free
    int q, R;
    int law, fixed_d;
    unsigned long long seed;
    ModQ modq;
    long long D;
    const int* off_left;
    const int* off_right;
    const uint64_t* gthr;         // GEOMETRIC: the q-1 delay thresholds (geometric_thresholds)
    const struct PeLink* links;   // [P] neighbour sources / publish targets
    int pin_first_pe;             // PE whose first point is the pinned global end 0 (or -1)
    int pin_last_pe;              // PE whose last point is the pinned global end N-1 (or -1)
    unsigned int* done;           // [P*Tp] passes completed in this launch
    unsigned long long* counter;  // work-item counter
    unsigned long long* stats;
    unsigned int* flag;
    unsigned int* abort_word;
    unsigned long long timeout_ns;
    int pend_max;   // done-signals published per release fence (1..kMaxPend)
    // optional logs for the a-posteriori bound (heat_async_free_run):
    // edge_log[(k*P + p)*2 + side] = PE p's first (0) / last (1) point at step
    // k (k >= 1; the host fills k = 0); used_log[(k*P + p)*2 + side] = the step
    // k* of the neighbour value PE p's first / last point read at step k
    double* edge_log;
    int* used_log;
};
constexpr int kMaxPend = 16;
#ifndef HEAT_K5_UNROLL
#define HEAT_K5_UNROLL 2
#endif
// interior step loop unroll: 2 (4: -1.4%, 1: -2.5%, measured with the single
// interior loop; K1 gains 0.45% from 4)
constexpr int kK5Unroll = HEAT_K5_UNROLL;

__device__ __forceinline__ int det_delay_s(const AsyncStreamArgs& a, long long k, int off) {
    const long long bound = k < (long long)(a.q - 1) ? k : (long long)(a.q - 1);
    if (a.law == 1) return a.fixed_d < bound ? a.fixed_d : int(bound);
    const uint64_t x = splitmix_draw(a.seed, uint64_t(k) * uint64_t(a.D) + uint64_t(off));
    if (a.law == 0) return uniform_delay(x, bound, a.modq);
    return geometric_delay(x, a.gthr, int(bound));
}

__device__ __forceinline__ uint64_t ld_acq(const unsigned long long* w, bool sys) {
    return sys ? ld_acquire_sys(reinterpret_cast<const uint64_t*>(w))
               : ld_acquire_gpu(reinterpret_cast<const uint64_t*>(w));
}

__device__ __forceinline__ bool spin_until(const AsyncStreamArgs& a, const unsigned long long* w,
                                           long long need, unsigned long long* seen, bool* waited,
                                           bool sys) {
    uint64_t v = ld_acq(w, sys);
    if ((long long)v >= need) {
        *seen = v;
        return true;
    }
    *waited = true;
    const uint64_t t0 = globaltimer_ns();
    unsigned spins = 0;
    while ((long long)(v = ld_acq(w, sys)) < need) {
        if ((++spins & 127u) == 0) {
            if (*reinterpret_cast<volatile unsigned int*>(a.abort_word)) return false;
            if (globaltimer_ns() - t0 > a.timeout_ns) {
                atomicOr(a.flag + 1, 1u);
                atomicExch(a.abort_word, 1u);
                return false;
            }
        }
    }
    *seen = v;
    return true;
}

__device__ __forceinline__ bool wait_done(const AsyncStreamArgs& a, const unsigned int* w,
                                          unsigned int need) {
    if (ld_acquire_gpu_u32(w) >= need) return true;
    const uint64_t t0 = globaltimer_ns();
    unsigned spins = 0;
    while (ld_acquire_gpu_u32(w) < need) {
        __nanosleep(64);
        if ((++spins & 127u) == 0) {
            if (*reinterpret_cast<volatile unsigned int*>(a.abort_word)) return false;
            if (globaltimer_ns() - t0 > a.timeout_ns) {
                atomicOr(a.flag + 1, 1u);
                atomicExch(a.abort_word, 1u);
                return false;
            }
        }
    }
    return true;
}

// One Jacobi step of a lane's V points in a PE-boundary tile: on the lane
// with cutL, element FE takes the ghost product gp as its LEFT neighbour
// product; on the lane with cutR, element LE takes it as its RIGHT one.
// Points beyond a cut belong to the neighbour PE's side of the window and are
// never output.  FE / LE are compile-time (the edge positions are warp-
// uniform and few), so the cut costs one select, not one per element.
template <int V, int FE, int LE>
__device__ __forceinline__ void chunk_step_cut(double (&u)[V], double r, double c, double pL,
                                               double pR, double pFirst, double pLast, bool cutL,
                                               bool cutR, double gp) {
    using A = Arith<double>;
    double pm1 = pL, p0 = pFirst;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const double p1 = i + 1 == V ? pR : (i + 1 == V - 1 ? pLast : A::mul(r, u[i + 1]));
        const double right = (i == LE && cutR) ? gp : p1;
        const double left = (i == FE && cutL) ? gp : pm1;
        u[i] = stencil_p(right, A::mul(c, u[i]), left);
        pm1 = p0;
        p0 = p1;
    }
}

// One boundary-tile step, edge writes and the new edge values: the PE's
// first point is element FE of its lane, the last point element LE.
template <int V, int FE, int LE>
__device__ __forceinline__ void boundary_step(double (&u)[V], double r, double c, bool cutL,
                                              bool cutR, double ghost, bool pinF, double c1,
                                              bool pinL, double c2, double& first, double& last) {
    using A = Arith<double>;
    const double pFirst = A::mul(r, u[0]);
    const double pLast = A::mul(r, u[V - 1]);
    const double pL = __shfl_up_sync(0xffffffffu, pLast, 1);
    const double pR = __shfl_down_sync(0xffffffffu, pFirst, 1);
    chunk_step_cut<V, FE, LE>(u, r, c, pL, pR, pFirst, pLast, cutL, cutR, A::mul(r, ghost));
    if (pinF) u[FE] = c1;
    if (pinL) u[LE] = c2;
    first = u[FE];
    last = u[LE];
}

// Decoded work item.
struct StreamItem {
    long long pass;
    int p;   // PE
    int m;   // tile within the PE
};

__device__ __forceinline__ StreamItem decode_item(const AsyncStreamArgs& a, long long i) {
    const long long T = (long long)a.P * a.Tp;
    StreamItem it;
    it.pass = i / T;
    long long idx = i % T;
    if (idx < 2LL * a.P) {  // boundary pairs first: (right edge of b, left edge of b+1)
        const int b = int(idx >> 1);
        if ((idx & 1) == 0) {
            it.p = b;
            it.m = a.Tp - 1;
        } else {
            it.p = (b + 1) % a.P;
            it.m = 0;
        }
    } else {
        idx -= 2LL * a.P;
        const int inner = a.Tp - 2;
        it.p = int(idx / inner);
        it.m = 1 + int(idx % inner);
    }
    return it;
}

template <int V, int H = 32>
__global__ void __launch_bounds__(SyncTB<double, V, H>::kThreads, SyncTB<double, V, H>::min_blocks(2))
    async_stream_kernel(const __grid_constant__ CUtensorMap tm_load0,
                        const __grid_constant__ CUtensorMap tm_load1,
                        const __grid_constant__ CUtensorMap tm_store0,
                        const __grid_constant__ CUtensorMap tm_store1, const AsyncStreamArgs a) {
    using T = SyncTB<double, V, H>;
    using A = Arith<double>;
    static_assert(V == 32 || V == 48, "PE last points sit at element 31 mod 32: 31 | 15, 31, 47");
    // the host guarantees a PE's last tile holds >= H points, so no interior
    // tile's window reaches into the next PE
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // aligned by an offset from the __shared__ array itself: a round trip
    // through uintptr_t loses the address space (generic LD/ST, ptxas SASS)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + warp * 2 * T::kBufBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::kWarpsPerCta * 2 * T::kBufBytes) + 2 * warp;
    __shared__ unsigned int s_hist[T::kWarpsPerCta][129];
    unsigned int* whist = s_hist[warp];
    for (int i = lane; i < 129; i += 32) whist[i] = 0;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const double r = a.r, c = a.c;
    const long long T_all = (long long)a.P * a.Tp;
    const long long total = a.npass * T_all;
    const long long tma_len = (a.N / T::kUnit) * T::kUnit;
    uint32_t phase = 0;
    bool bad = false, abort = false;
    unsigned long long reads = 0, waits = 0, maxd = 0, lag_min = ~0ull, lag_max = 0;
    int b = 0;

    // Items are handed out dynamically in pass-major order (one atomic
    // counter): boundary tiles take ~5x longer than interior ones, and a
    // static deal lets the warps that drew them hold back their neighbours'
    // next pass (measured: -20%).
    auto grab = [&]() -> long long {
        unsigned long long i = 0;
        if (lane == 0) i = atomicAdd(a.counter, 1ull);
        return (long long)__shfl_sync(0xffffffffu, i, 0);
    };
    auto geometry = [&](const StreamItem& it, long long& lo, long long& w0, long long& out_hi) {
        lo = (long long)it.p * a.n;
        w0 = lo + (long long)it.m * T::kOut - T::kHalo;
        out_hi = lo + a.n;
    };
    auto deps_ready = [&](const StreamItem& it, bool block) -> bool {
        if (it.pass == 0) return true;
        const unsigned int need = unsigned(it.pass);
        const int base = it.p * a.Tp;
        bool ok = true;
        if (lane < 3) {
            const int mm = it.m + lane - 1;
            if (mm >= 0 && mm < a.Tp) {
                const unsigned int* w = a.done + base + mm;
                ok = block ? wait_done(a, w, need) : (ld_acquire_gpu_u32(w) >= need);
            }
        }
        return __all_sync(0xffffffffu, ok);
    };
    auto tma_ok = [&](long long w0) { return w0 >= 0 && w0 + kWarp * V <= tma_len; };
    auto issue = [&](int bb, const StreamItem& it, long long w0) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            bulk_wait_read_all();
            asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired data -> async proxy
            mbar_arrive_expect_tx(&bars[bb], T::kBufBytes);
            tma_load_3d(wbase + bb * T::kBufBytes, (it.pass & 1) ? &tm_load1 : &tm_load0, 0, 0,
                        int(w0 / T::kUnit), &bars[bb]);
        }
    };

    // Done-signals are deferred and published in pairs: one release fence
    // (fence.acq_rel.gpu, the costly part of a release store -- ncu: ERRBAR +
    // MEMBAR were the largest non-FP64 stalls) then relaxed stores for both.
    // Pending (tile, pass) pairs live in shared memory; only lane 0 uses them.
    __shared__ uint2 s_pend[T::kWarpsPerCta][kMaxPend];
    uint2* wpend = s_pend[warp];
    int npend = 0;
    bool pend_generic = false;  // a pending tile left through per-lane stores
    // Publish done[] of the pending tiles once their stores have landed.
    // keep_groups = 1 only when the NEWEST bulk group is the current item's
    // (not a pending one): every other group must be complete.
    auto signal_pending = [&](int keep_groups) {
        if (npend == 0) return;
        if (pend_generic) __threadfence();  // every lane's generic stores first
        __syncwarp();
        if (lane == 0) {  // TMA store groups done, async-proxy writes ordered, release
            if (keep_groups)
                asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
            else
                bulk_wait_all();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            fence_acq_rel_gpu();
            for (int j = 0; j < npend; ++j) st_relaxed_gpu_u32(a.done + wpend[j].x, wpend[j].y);
        }
        __syncwarp();
        npend = 0;
        pend_generic = false;
    };

    // this lane's share of an item's dependency flags (lanes 0..2: tiles m-1,
    // m, m+1 of the same PE at the previous pass), loaded with acquire
    auto dep_load = [&](const StreamItem& x) -> unsigned int {
        unsigned int v = 0xffffffffu;
        if (x.pass > 0 && lane < 3) {
            const int mm = x.m + lane - 1;
            if (mm >= 0 && mm < a.Tp) v = ld_acquire_gpu_u32(a.done + x.p * a.Tp + mm);
        }
        return v;
    };
    // Items are held two ahead: while item i runs, the warp already holds
    // item i+1 (grabbed during item i-1, its flags loaded then), so i+1's
    // window is issued as soon as i's window is in registers -- as K1 issues
    // its next window -- and interior tiles step in one uninterrupted loop.
    long long cur = grab();
    long long nxt = grab();
    unsigned int nxt_dep = nxt < total ? dep_load(decode_item(a, nxt)) : 0xffffffffu;
    bool cur_pref = false;  // window of `cur` already in flight into buffer b
    while (cur < total && !abort) {
        const StreamItem it = decode_item(a, cur);
        long long lo, w0, out_hi;
        geometry(it, lo, w0, out_hi);
        const bool left_edge = it.m == 0, right_edge = it.m == a.Tp - 1;
        const double* src = a.buf[it.pass & 1];
        double* dst = a.buf[(it.pass & 1) ^ 1];
        const long long kbeg = a.k0 + it.pass * a.s;
        const int nst = int(min((long long)a.s, a.k0 + a.steps - kbeg));

        // item i+2: the atomic is issued now and read once this window is in
        unsigned long long nn_raw = 0;
        if (lane == 0) nn_raw = atomicAdd(a.counter, 1ull);
        // ---- window in
        if (!cur_pref) {
            if (!deps_ready(it, false)) signal_pending(0);  // never block holding a signal
            if (!deps_ready(it, true)) { abort = true; break; }
            if (tma_ok(w0)) issue(b, it, w0);
        }
        double u[V];
        const long long g0 = w0 + (long long)lane * V;
        if (tma_ok(w0)) {
            mbar_wait(&bars[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            chunk_from_smem<double, V>(wbase + b * T::kBufBytes, lane, u);
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                const long long g = g0 + i;
                u[i] = (g >= 0 && g < a.N) ? ld_relaxed_gpu_f64(src + g) : 0.0;
            }
        }
        // ---- item i+1: its flags were loaded one item ago
        bool nxt_pref = false;
        StreamItem ni{};
        long long nlo = 0, nw0 = 0, nhi = 0;
        bool nxt_cand = false;
        if (nxt < total) {
            ni = decode_item(a, nxt);
            geometry(ni, nlo, nw0, nhi);
            nxt_cand = tma_ok(nw0);
        }
        unsigned int dep_seen = nxt_dep;
        auto try_prefetch = [&]() {
            if (!nxt_cand || nxt_pref) return;
            const bool ok = ni.pass == 0 || dep_seen >= unsigned(ni.pass);
            if (__all_sync(0xffffffffu, ok)) {
                issue(b ^ 1, ni, nw0);
                nxt_pref = true;
            }
        };
        try_prefetch();
        if (nxt_cand && !nxt_pref) dep_seen = dep_load(ni);  // tested again after the steps
        const long long nn = (long long)__shfl_sync(0xffffffffu, nn_raw, 0);
        const unsigned int nn_dep = nn < total ? dep_load(decode_item(a, nn)) : 0xffffffffu;

        // ---- step the tile; boundary tiles exchange edge values every step.
        // The PE's first point sits kHalo points into a left-edge window, its
        // last point wherever the PE ends: (lane, element) of each.
        const int fl = T::kHalo / V;  // lane of the first point (lo - w0 = kHalo)
        const int lpos = int(out_hi - 1 - w0);
        const int ll = lpos / V, le = lpos % V;
        if (!left_edge && !right_edge) {
            warp_steps_pipelined<double, V, kK5Unroll>(u, r, c, nst);
            try_prefetch();
        } else {
            try_prefetch();
            signal_pending(0);  // boundary tiles spin on other PEs: flush first
            // where this PE's neighbour values come from / its edge values go
            const PeLink lk = a.links[it.p];  // into registers once per boundary tile
            const bool pin_first = it.p == a.pin_first_pe;
            const bool pin_last = it.p == a.pin_last_pe;
            const bool needL = left_edge && lk.srcL != nullptr && !pin_first;
            const bool needR = right_edge && lk.srcR != nullptr && !pin_last;
            // lane fl holds the PE's first point, lane ll its last one (different
            // tiles: Tp >= 2)
            const bool left = lane == fl && needL;
            const bool mine = left || (lane == ll && needR);
            const unsigned long long* pw = left ? lk.progL_src : lk.progR_src;
            const double* gring = left ? lk.srcL : lk.srcR;
            const bool gsys = (lk.flags & (left ? kLinkSrcLSys : kLinkSrcRSys)) != 0;
            for (int s = 0; s < nst && !abort; ++s) {
                const long long k = kbeg + s;
                double ghost = 0.0;
                if (mine) {
                    unsigned long long seen = 0;
                    bool waited = false;
                    long long mstep;
                    if (a.mode == 0) {
                        mstep = k - det_delay_s(a, k, left ? a.off_left[it.p] : a.off_right[it.p]);
                        if (!spin_until(a, pw, mstep, &seen, &waited, gsys)) abort = true;
                    } else {
                        if (!spin_until(a, pw, k - (a.q - 1), &seen, &waited, gsys)) abort = true;
                        mstep = (long long)seen < k ? (long long)seen : k;
                    }
                    if (!abort) {
                        if (a.used_log)
                            a.used_log[(k * a.P + it.p) * 2 + (left ? 0 : 1)] = int(mstep);
                        const double* slotp = gring + (mstep & (a.R - 1));
                        ghost = gsys ? ld_relaxed_sys_f64(slotp) : ld_relaxed_gpu_f64(slotp);
                        const unsigned long long used = (unsigned long long)(k - mstep);
                        const unsigned long long lag = seen - (unsigned long long)mstep;
                        reads++;
                        waits += waited;
                        maxd = used > maxd ? used : maxd;
                        lag_min = lag < lag_min ? lag : lag_min;
                        lag_max = lag > lag_max ? lag : lag_max;
                        atomicAdd(&whist[used < 64 ? used : 63], 1u);
                        atomicAdd(&whist[64 + (lag < 64 ? lag : 64)], 1u);
                    }
                }
                if (__any_sync(0xffffffffu, abort)) {
                    abort = true;
                    break;
                }
                // edge elements: first at kHalo % V (always), last at le, which
                // is 31 mod 32 -- warp-uniform, dispatched to a compile-time cut
                const bool cutR = lane == ll && needR;
                const bool pinF = left_edge && pin_first && lane == fl;
                const bool pinL = right_edge && pin_last && lane == ll;
                double first, last;
                constexpr int FE = T::kHalo % V;
                if (V == 32 || le == 31)
                    boundary_step<V, FE, 31>(u, r, c, left, cutR, ghost, pinF, a.c1, pinL, a.c2,
                                             first, last);
                else if (le == 15)
                    boundary_step<V, FE, (V > 15 ? 15 : 0)>(u, r, c, left, cutR, ghost, pinF,
                                                            a.c1, pinL, a.c2, first, last);
                else
                    boundary_step<V, FE, (V > 47 ? 47 : V - 1)>(u, r, c, left, cutR, ghost, pinF,
                                                                 a.c1, pinL, a.c2, first, last);
                // publish u_first(k+1) / u_last(k+1) to every ring that mirrors
                // it (local, plus the neighbour device's receive ring for a
                // device boundary -- a P2P store over NVLink), then release
                // the progress word with the matching scope
                const long long slot = (k + 1) & (a.R - 1);
                if (a.edge_log) {
                    if (left_edge && lane == fl) a.edge_log[((k + 1) * a.P + it.p) * 2 + 0] = first;
                    if (right_edge && lane == ll) a.edge_log[((k + 1) * a.P + it.p) * 2 + 1] = last;
                }
                if (left_edge && lane == fl) {
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (!lk.pubF[t]) continue;
                        if (lk.flags & (t ? kLinkPubF1Sys : 0)) {
                            st_relaxed_sys_f64(lk.pubF[t] + slot, first);
                            st_release_sys(reinterpret_cast<uint64_t*>(lk.pubF_prog[t]), uint64_t(k + 1));
                        } else {
                            st_relaxed_gpu_f64(lk.pubF[t] + slot, first);
                            st_release_gpu(reinterpret_cast<uint64_t*>(lk.pubF_prog[t]), uint64_t(k + 1));
                        }
                    }
                }
                if (right_edge && lane == ll) {
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (!lk.pubL[t]) continue;
                        if (lk.flags & (t ? kLinkPubL1Sys : 0)) {
                            st_relaxed_sys_f64(lk.pubL[t] + slot, last);
                            st_release_sys(reinterpret_cast<uint64_t*>(lk.pubL_prog[t]), uint64_t(k + 1));
                        } else {
                            st_relaxed_gpu_f64(lk.pubL[t] + slot, last);
                            st_release_gpu(reinterpret_cast<uint64_t*>(lk.pubL_prog[t]), uint64_t(k + 1));
                        }
                    }
                }
            }
            if (abort) break;
        }

        // ---- window out: the tile's exact points [w0 + kHalo, w0 + 32V - kHalo)
        // that lie inside this PE (bounds are multiples of 32 points)
        const bool full = w0 + kWarp * V - T::kHalo <= out_hi && w0 + T::kHalo >= lo;
        int el_lo = min(V, max(0, T::kHalo - lane * V));  // a whole window inside the PE
        int el_hi = min(V, max(0, kWarp * V - T::kHalo - lane * V));
        if (!full) {  // clipped to the PE
            const long long ex_lo = max(w0 + T::kHalo, lo);
            const long long ex_hi = min(w0 + kWarp * V - T::kHalo, out_hi);
            el_lo = int(max(0LL, min((long long)V, ex_lo - g0)));
            el_hi = int(max(0LL, min((long long)V, ex_hi - g0)));
        }
        if (it.pass == a.npass - 1) {  // non-finite values are absorbing
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (i >= el_lo && i < el_hi) bad |= !isfinite(u[i]);
        }
        unsigned char* bufb = wbase + b * T::kBufBytes;
        if (tma_ok(w0) && full) {
            chunk_to_smem_out_split<double, V, H>(bufb, lane, u, el_lo, el_hi);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_3d((it.pass & 1) ? &tm_store0 : &tm_store1, 0, 0,
                             int((w0 + T::kHalo) / T::kUnit), bufb);
                bulk_commit();
            }
        } else {
#pragma unroll
            for (int m = 0; m < V / 2; ++m)
                if (2 * m >= el_lo && 2 * m + 2 <= el_hi)
                    reinterpret_cast<double2*>(dst + g0)[m] = make_double2(u[2 * m], u[2 * m + 1]);
        }
        // Declare the PREVIOUS item done (its store has had a whole compute
        // phase to land: wait until at most this item's store group is in
        // flight), and keep this one pending.  Blocking waits flush first.
        const bool cur_bulk = tma_ok(w0) && full;  // this item's store is the newest group
        if (npend >= a.pend_max) signal_pending(cur_bulk ? 1 : 0);
        if (lane == 0) wpend[npend] = make_uint2(unsigned(it.p * a.Tp + it.m), unsigned(it.pass + 1));
        ++npend;
        pend_generic |= !cur_bulk;
        cur = nxt;
        nxt = nn;
        nxt_dep = nn_dep;
        cur_pref = nxt_pref;
        if (nxt_pref) b ^= 1;
    }
    signal_pending(0);
    if (bad) atomicOr(a.flag, 1u);
    __syncwarp();
    if (a.stats) {
        for (int i = lane; i < 129; i += 32) {
            const unsigned int cnt = whist[i];
            if (cnt) atomicAdd(a.stats + (i < 64 ? kStatDelayHist + i : kStatLagHist + (i - 64)),
                               (unsigned long long)cnt);
        }
        if (reads) {
            atomicAdd(a.stats + kStatReads, reads);
            atomicAdd(a.stats + kStatWaits, waits);
            atomicMax(a.stats + kStatMaxDelay, maxd);
            atomicMin(a.stats + kStatLagMin, lag_min);
            atomicMax(a.stats + kStatLagMax, lag_max);
        }
    }
}

}  // namespace hb
