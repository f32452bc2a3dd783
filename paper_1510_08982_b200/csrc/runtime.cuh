// runtime.cuh -- host-side runtime shared by the C-ABI translation units:
// error reporting, the per-device workspace, launch accounting.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/heat_b200.h"

// Every plan is a slab with kSlabHalo ghost points on each side:
// array = [ghost H | n owned points | ghost H].  A single-GPU plan
// (world == 1) ignores the ghosts and advances the owned points as a whole
// domain; a multi-GPU slab (world > 1) gets its ghosts refreshed by the caller
// (heat_plan_halo_pack / _unpack around an NCCL or peer exchange) before each
// pass of <= H steps, and only the true global ends are pinned.
struct heat_plan {
    int device = 0;
    int rank = 0, world = 1;
    size_t n = 0;
    size_t pitch = 0;
    double* base = nullptr;
    int cur = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    unsigned int* flag = nullptr;
    int sms = 0;
    double* bufs[2] = {nullptr, nullptr};  // owned points (base + H)
    double* ext[2] = {nullptr, nullptr};   // ghosted arrays (base)
    void* async_scratch = nullptr;         // rings / counters of heat_plan_async_advance
    size_t async_bytes = 0;
    void* xlink = nullptr;                 // multi-GPU P2P state (xlink.cu)
};

namespace hb {

void set_error(const std::string& msg);
std::string last_error_msg();  // this thread's last fail() message
inline int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

extern std::atomic<uint64_t> g_launches;
extern std::atomic<bool> g_strict;

#define HB_CUDA(x)                                                                         \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return ::hb::fail(HEAT_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define HB_TRY(x)                 \
    do {                          \
        int s_ = (x);             \
        if (s_ != HEAT_OK) return s_; \
    } while (0)

// A pair of timing events on one stream (destroyed with the pair).
struct EventPair {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    EventPair() = default;
    EventPair(const EventPair&) = delete;
    EventPair& operator=(const EventPair&) = delete;
    ~EventPair() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
    int begin(cudaStream_t st) {
        if (!e0) HB_CUDA(cudaEventCreate(&e0));
        if (!e1) HB_CUDA(cudaEventCreate(&e1));
        HB_CUDA(cudaEventRecord(e0, st));
        return HEAT_OK;
    }
    int end(cudaStream_t st) {
        HB_CUDA(cudaEventRecord(e1, st));
        return HEAT_OK;
    }
    int elapsed(float* ms) {
        HB_CUDA(cudaEventSynchronize(e1));
        HB_CUDA(cudaEventElapsedTime(ms, e0, e1));
        return HEAT_OK;
    }
};

// Flag words of a context (DevCtx / plan): [0] non-finite, [1] watchdog,
// [2] input validation, [3] spare, [4..5] the K1 tile counter (u64) of the
// context's stream, [6..7] that of its second compute stream (the streamed
// sync_run) -- one per stream, so concurrent launches never share one.
constexpr int kFlagWords = 8;
inline unsigned long long* tile_counter_of(unsigned int* flag) {
    return reinterpret_cast<unsigned long long*>(flag + 4);
}

// Per-device state: a grow-only pair of field buffers for the one-shot
// entry points, the non-finite flag word, and a private stream.
struct DevCtx {
    std::mutex mu;
    int device = -1;
    int sms = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the streamed sync_run
    cudaStream_t stream2 = nullptr;             // its second compute stream
    void* buf[2] = {nullptr, nullptr};
    size_t bytes = 0;
    unsigned int* flag = nullptr;  // [0] non-finite, [1] watchdog timeout
    void* scratch = nullptr;       // async rings / logs
    size_t scratch_bytes = 0;
    void* snaps = nullptr;         // in-kernel trajectories of small runs
    size_t snaps_bytes = 0;
    void* host = nullptr;          // pinned staging of the small one-shot calls
    size_t host_bytes = 0;
    // pinned ring for large PAGEABLE fields (the streamed sync_run): slots
    // filled / drained by host threads while the copy engines move the rest
    void* ring = nullptr;
    cudaEvent_t ring_ev[8] = {};
};

// A ring of kRingSlots pinned slots of kRingSlotBytes for staging a pageable
// host field through the copy engines (allocated once per device).
constexpr int kRingSlots = 8;  // 4 for uploads, 4 for downloads
constexpr size_t kRingSlotBytes = 128ull << 20;
int host_ring(DevCtx& d, unsigned char** slots);
// memcpy with up to `threads` host threads (large pageable <-> pinned copies)
void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads);
// true when `p` is ordinary (unregistered, pageable) host memory
bool host_pageable(const void* p);

// Closes a plan's IPC mappings and frees its xlink state (xlink.cu).
void xlink_release(heat_plan* p);

// Locks and initialises the context of the current (or given) device.
int dev_ctx(int device, DevCtx** out);
int ensure_buffers(DevCtx& d, size_t bytes);
int ensure_scratch(DevCtx& d, size_t bytes);
// Pinned host staging for the small one-shot calls (K7 / K9): their copies are
// a few KB, and pageable copies cost ~10 us each.  Returns nullptr above
// kHostStageMax (callers then copy from / to the caller's pageable memory).
constexpr size_t kHostStageMax = 64ull << 20;
unsigned char* host_stage(DevCtx& d, size_t bytes);

// Sets `fn`'s dynamic shared memory limit to `smem` on the CURRENT device
// (the attribute is per device) and returns its resident CTAs per SM for
// `threads`-thread blocks; cached per (kernel, device).
int kernel_smem_config(const void* fn, int smem, int threads, int* per_sm);

// Validation helpers mirroring the reference's constructors.
int check_field(const double* u, size_t n);  // BasicField ctor, core.hpp:45-51

// The geometric law (sample_delay, async_sim.cpp:64-69) as thresholds on a
// draw's top 53 bits m = x >> 11: d = #{j : m >= T[j-1]}, j = 1..q-1, then
// min(d, bound).  Exact because the reference's floor(log1p(-u)/log1p(-p))
// is non-decreasing in m away from each integer crossing, and every m in a
// window around each threshold -- wider than log1p's rounding error can move
// a crossing -- is checked with glibc's log1p itself.  HEAT_EINVAL when p is
// so small that the quotient leaves size_t's range (the reference's
// conversion is undefined there); cached per (p, q).
int geometric_thresholds(double p, size_t q, std::vector<uint64_t>& T);

// An AsyncSimulator handle's current field (device) and stream (async_host.cu).
void async_sim_device_field(heat_async_sim* sim, const double** field, cudaStream_t* st);
int prepare_initial(const double* u0, size_t n, int bc_kind, double c1, double c2,
                    std::vector<double>& out);  // sync_solver.cpp:25-37

inline size_t default_stride(size_t n) { return n <= 1000 ? 1 : 100; }

// Geometry of one synchronous pass (see SyncPassArgs in sync_tb.cuh).
struct SlabGeom {
    long long len = 0, out_lo = 0, out_hi = 0, pin_lo = -1, pin_hi = -1;
    int wrap = 0;
};
// ghost points per side of a multi-GPU slab = steps per exchange: the default
// K1 variant's halo, so slab passes run the same 64-step kernel as one GPU
constexpr int kSlabHalo = 64;

template <typename Real>
int sync_advance_slab(int sms, Real* bufs[2], int& cur, const SlabGeom& g, double r, double c1,
                      double c2, size_t steps, unsigned int* flag, cudaStream_t st,
                      int max_steps_per_pass = 0);

// Tensor map over an f64 array viewed as [chunk of 32][128-B row][16]
// (128B swizzle), `box_chunks` chunks per box (sync_host.cu).
int make_chunk_map_f64(struct CUtensorMap_st* m, const void* base, long long nchunks,
                       int box_chunks);

// Upload + validate + snap a host field into `dst` (sync_host.cu).
int upload_prepared(DevCtx& d, const double* u0, size_t n, int bc_kind, double c1, double c2,
                    double* dst);

// Shared driver of async_run (deterministic) and exec_run(BarrierFree) (free).
// Advances `field` (device, prepared) from step 0 to k_end, calling
// on_record(k) after every `stride` steps when stride > 0.
struct AsyncRunSpec {
    size_t N, n;
    double r;
    int bc_kind;
    double c1, c2;
    int mode;  // 0 deterministic, 1 free
    size_t q;
    int law;
    size_t fixed_d;
    double geometric_p;
    uint64_t seed;
    size_t k_end;
    bool want_logs;
};

// async_run after validation (async_host.cu).
int async_run_core(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                   size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                   uint64_t seed, size_t k_end, size_t stride, double* final_out,
                   double* snapshots, size_t* steps_out, size_t max_snapshots,
                   size_t* n_snapshots);

// In-step draw ranks of the cross-PE reads (async_host.cu), returns D.
int draw_offsets(size_t N, size_t n, int dirichlet, std::vector<int>& offL, std::vector<int>& offR);

// K7 (sync_small.cu): the whole sync_run of a field of <= sync_small_max_points()
// points in one CTA; arguments and errors as heat_sync_run (validated by the caller).
// K9 (async_small.cu): deterministic async_run of small fields on one CTA
bool async_small_eligible(size_t N, size_t per_pe, size_t q);
// K6 with one member (ensemble.cu): async_run of fields K9 does not lay out
bool async_member_eligible(size_t n, size_t per_pe, size_t q);
int async_run_member(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                     size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                     uint64_t seed, size_t k_end, size_t stride, double* final_out,
                     double* snapshots, size_t* steps_out, size_t max_snapshots,
                     size_t* n_snapshots);
int async_run_small(const double* u0, size_t N, double r, int bc_kind, double c1, double c2,
                    size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                    uint64_t seed, size_t k_end, size_t stride, double* final_out,
                    double* snapshots, size_t* steps_out, size_t max_snapshots,
                    size_t* n_snapshots);
size_t sync_small_max_points();
int sync_run_small(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t k_end, size_t stride, double* final_out, double* snapshots,
                   size_t* steps_out, size_t max_snapshots, size_t* n_snapshots,
                   float* kernel_ms = nullptr, bool one_cta = false);
// K10 (exec_free.cu): exec_run(BarrierFree) of PEs that fit one warp each, all
// in one thread-block cluster; stats in the kStat layout (optional).
bool free_eligible(size_t N, size_t per_pe, size_t q, size_t k_end);
int exec_free_run(DevCtx& d, const double* u0, size_t N, double r, int bc_kind, double c1,
                  double c2, size_t per_pe, size_t q, size_t k_end, double* field_out,
                  unsigned long long* stats_host, float* kernel_ms);
// exec_run(Barriered) (async_exec.cpp:57-114): sync_run to the final state
// with the compute kernels' device time (events on the run's stream around
// the launches only -- the bracket BarrierFree's kernels are timed over).
int sync_run_timed(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t k_end, double* final_out, float* kernel_ms);

// Synchronous advance on device buffers (ping-pong).  `cur` selects the
// buffer holding u(k) on entry and is updated.  Does not synchronise.
template <typename Real>
int sync_advance(int sms, Real* bufs[2], int& cur, long long n, double r, int periodic,
                 double c1, double c2, size_t steps, unsigned int* flag, cudaStream_t st);

}  // namespace hb
