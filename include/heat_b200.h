/*
 * heat_b200.h -- C-ABI of the B200-native FTCS hot path (arXiv 1510.08982).
 *
 * Drop-in boundary for the reference's solver API in namespace heat
 * (/root/reference/proj/include/heat/{sync_solver,async_sim,async_exec}.hpp).
 * Plain pointers and sizes only: no torch, no CUDA types in the signatures.
 * Host buffers are caller-owned; device memory belongs to the library (a
 * per-device workspace, or an explicit heat_plan for resident runs).
 *
 * Conventions shared by every entry point
 *   - Fields are IEEE-754 binary64 arrays u[0..n-1] (TemperatureField,
 *     core.hpp:42-64).  `r` is the exact bits of SolverParams::r()
 *     (core.hpp:27); the caller derives it, the library never re-derives it.
 *   - Boundary condition (core.hpp:68-81): bc_kind HEAT_BC_DIRICHLET with
 *     ends (c1, c2), or HEAT_BC_PERIODIC (c1, c2 ignored).
 *   - Return value: HEAT_OK or a status that maps 1:1 onto the reference's
 *     exception types; heat_last_error() gives the message.
 *   - Trajectory recording follows sync_run (sync_solver.cpp:52-77): step 0,
 *     every `stride`-th step and the final step; stride 0 selects the
 *     default (1 when n <= 1000, else 100; sync_solver.hpp:52-54).  Use
 *     heat_trajectory_length() to size `snapshots` (rows of n doubles) and
 *     `steps`.  Either may be NULL when only the final state is wanted
 *     (then pass `final_out`).
 *   - Thread safety: every entry point may be called from any host thread;
 *     the per-device workspace is guarded by a mutex (the reference's
 *     ensemble_run calls AsyncSimulator from many threads, analysis.cpp:68-85).
 */
#ifndef HEAT_B200_H
#define HEAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define HEAT_OK        0
#define HEAT_EDOMAIN   1  /* std::domain_error      (core.cpp:8-31, core.hpp:46-50, async_sim.cpp:8-22) */
#define HEAT_EINVAL    2  /* std::invalid_argument  (sync_solver.cpp:31-32, async_exec.cpp:266-270)     */
#define HEAT_ELOGIC    3  /* std::logic_error       (async_sim.cpp:35,44)                                 */
#define HEAT_EDIVERGE  4  /* heat::DivergenceError  (sync_solver.hpp:81-83)                              */
#define HEAT_ECUDA     5  /* CUDA runtime failure   -> std::runtime_error                                */
#define HEAT_ETIMEOUT  6  /* async watchdog: a halo-ring wait exceeded its deadline                      */
#define HEAT_ENOMEM    7  /* device or host allocation failure                                           */
#define HEAT_ENODEV    8  /* no CUDA device / extension unusable: never falls back to the CPU            */

#define HEAT_BC_DIRICHLET 0
#define HEAT_BC_PERIODIC  1

/* DelayModel::Distribution (async_sim.hpp:16-28) */
#define HEAT_DELAY_UNIFORM   0
#define HEAT_DELAY_FIXED     1
#define HEAT_DELAY_GEOMETRIC 2

/* ExecMode (async_exec.hpp:15) */
#define HEAT_EXEC_BARRIERED   0
#define HEAT_EXEC_BARRIER_FREE 1

/* LagStats (async_exec.hpp:42-51); kLagHistogramSize = 64 (async_exec.cpp:42). */
typedef struct heat_lag_stats {
    uint64_t reads;
    uint64_t min_lag;
    uint64_t max_lag;
    uint64_t overflow;
    uint64_t histogram[64];
} heat_lag_stats;

/* Free-running async diagnostics (GPU-only, no reference counterpart):
 * reader-relative delay k - k* of every cross-PE read (the paper's quantity),
 * plus the writer lag the reference's LagStats measures. */
typedef struct heat_async_stats {
    uint64_t reads;
    uint64_t max_delay;
    uint64_t delay_histogram[64];
    uint64_t waits;        /* reads that had to spin for the bound q          */
    double   residual_sum; /* sum_k ||u(k+1) - A u(k)||_inf (a-posteriori bound), when logged */
} heat_async_stats;

/* ---- AsyncSimulator (async_sim.hpp:73-90) on the GPU ---------------------
 * create = the ctor (prepared field, partition and q checks), step(count) =
 * count x AsyncSimulator::step(), current = current() + step_index().  The
 * handle owns its device state; any slicing of the steps is bit-identical to
 * async_run over the whole (counter-form draws, persistent PE rings). */
typedef struct heat_async_sim heat_async_sim;
int heat_async_sim_create(heat_async_sim** sim, const double* u0, size_t n, double r, int bc_kind,
                          double c1, double c2, size_t per_pe, size_t q, int law,
                          size_t fixed_delay, double geometric_p, uint64_t seed);
int heat_async_sim_step(heat_async_sim* sim, size_t count);
int heat_async_sim_current(heat_async_sim* sim, double* field_out, size_t* step_index);
int heat_async_sim_destroy(heat_async_sim* sim);

/* ---- HistoryRing (async_sim.hpp:31-57) in HBM + async_step (:68-71) -------
 * heat_history_create: a ring of `depth` snapshots of n points at step
 * `step`, holding `count` = min(depth, step + 1) of them; row d of
 * `snapshots` (n doubles each) is u(step - d).  HistoryRing(depth, initial)
 * is step = 0, count = 1.  push / read / snapshot / info follow the class
 * (logic_error -> HEAT_ELOGIC).  heat_async_step is async_step(hist, params,
 * bc, part, model, rng) (async_sim.cpp:107-116): *rng_state is the caller's
 * SplitMix64 state, advanced as the reference's stream (D draws per step;
 * only through the failing draw on a logic_error).  `out` (host, may be
 * NULL) gets the new field; push != 0 also pushes it (AsyncSimulator::step,
 * async_sim.cpp:136-140) without a host round trip.  Kernels K8a/K8b. */
typedef struct heat_history heat_history;
int heat_history_create(heat_history** hist, size_t depth, size_t n, size_t step,
                        const double* snapshots, size_t count, int device);
int heat_history_destroy(heat_history* hist);
int heat_history_info(const heat_history* hist, size_t* depth, size_t* current_step,
                      size_t* grid_size);
int heat_history_push(heat_history* hist, const double* state, size_t n);
int heat_history_read(const heat_history* hist, size_t i, size_t d, double* value);
int heat_history_snapshot(const heat_history* hist, size_t d, double* out);
int heat_async_step(heat_history* hist, double r, int bc_kind, double c1, double c2,
                    size_t part_total, size_t per_pe, size_t q, int law, size_t fixed_delay,
                    double geometric_p, uint64_t* rng_state, double* out, int push);

/* ---- planning queries (host only, no device needed; for tests/tools) -----
 * The streamed sync_run's chunk boundaries for n points and a "wave" of
 * wave_points (one tile per resident warp); K3's layout (lanes per PE, points
 * per lane, warps, shared rings) for P PEs of n points, bound q, mode (0
 * lockstep, 1 free); K5's tile geometry (points per lane, halo) for PEs of n. */
int heat_stream_chunk_plan(size_t n, size_t wave_points, size_t* bounds, size_t cap, size_t* count);
int heat_k3_geometry(size_t n, size_t P, size_t q, int mode, int* lanes_per_pe, int* points_per_lane,
                     size_t* warps, int* shared_rings);
int heat_k5_geometry(size_t n, int* points_per_lane, int* halo);
/* K10, exec_run(BarrierFree) in one thread-block cluster (exec_free.cu): for
 * N points in PEs of per_pe and delay bound q, the points per lane, lanes per
 * warp, warps per CTA, cluster size and warps per PE; HEAT_EINVAL (all 0)
 * when the run takes the K3/K5 path instead. */
int heat_free_geometry(size_t N, size_t per_pe, size_t q, int* points_per_lane, int* lanes,
                       int* warps_per_cta, int* cluster, int* warps_per_pe);
/* The geometric law's q-1 delay thresholds on a draw's top 53 bits
 * (thresholds[j-1] = first m = x >> 11 whose delay is >= j; 2^53 = never),
 * as the device kernels use them; HEAT_EINVAL for p too small. */
int heat_geometric_thresholds(double p, size_t q, uint64_t* thresholds);

/* ---- library state ---------------------------------------------------- */
const char* heat_last_error(void);
const char* heat_version(void);
int heat_device_count(void);
/* Device of the calling thread's one-shot calls (sync_run, async_run,
 * ensemble_run, ...): cudaSetDevice for this library.  One process per GPU
 * under torchrun calls it with its local rank (multigpu.ensemble_run_sharded).
 * HEAT_EINVAL for a device that does not exist. */
int heat_set_device(int device);
/* Number of kernels this library has launched in this process (all devices). */
uint64_t heat_kernel_launches(void);
/* The f64 synchronous pass kernel in use (HEAT_SYNC_VARIANT selects among
 * compiled variants): points per lane, window buffers per warp, exact points
 * per tile (K1s: per chunk of tiles), steps per HBM pass (= halo points per
 * side).  Host-only; no device needed. */
int heat_sync_kernel_info(int* points_per_lane, int* buffers, int* exact_points_per_tile,
                          int* steps_per_pass);

/* set_strict_finite_checks / strict_finite_checks (sync_solver.hpp:77-78) */
void heat_set_strict_finite_checks(int enabled);
int heat_strict_finite_checks(void);

/* detail::prepare_initial (sync_solver.cpp:25-37): copy u0 to out, and for
 * Dirichlet check |u0[0]-c1|, |u0[n-1]-c2| <= 1e-9 (HEAT_EINVAL) and snap the
 * ends.  Host-only. */
int heat_prepare_initial(const double* u0, size_t n, int bc_kind, double c1, double c2,
                         double* out);

/* Snapshot count sync_run / async_run record for (n, k_end, stride). */
size_t heat_trajectory_length(size_t n, size_t k_end, size_t stride);

/* ---- synchronous solver (sync_solver.hpp:60-73) ------------------------- */
/* sync_step (sync_solver.hpp:60-62): one step of u (ends snapped per BC). */
int heat_sync_step(const double* u, size_t n, double r, int bc_kind, double c1, double c2,
                   double* out);

/* sync_run (sync_solver.hpp:64-67). */
int heat_sync_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                  size_t k_end, size_t stride, double* final_out, double* snapshots,
                  size_t* steps, size_t max_snapshots, size_t* n_snapshots);

/* sync_run_f32 (sync_solver.hpp:69-73): FP32 arithmetic, results widened. */
int heat_sync_run_f32(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                      size_t k_end, size_t stride, double* final_out, double* snapshots,
                      size_t* steps, size_t max_snapshots, size_t* n_snapshots);

/* ---- deterministic asynchronous solver (async_sim.hpp:59-101) ----------- */
/* async_run: Eq. (4) with the model's seeded delay stream replayed exactly.
 * per_pe = PartitionSpec::per_pe (core.hpp:85-102). */
int heat_async_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                   size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                   uint64_t seed, size_t k_end, size_t stride, double* final_out,
                   double* snapshots, size_t* steps, size_t max_snapshots,
                   size_t* n_snapshots);

/* sample_delay (async_sim.cpp:57-73) for draw index j of a stream (counter
 * form): the delay the j-th draw yields at step k. */
int heat_sample_delay(size_t q, int law, size_t fixed_delay, double geometric_p, uint64_t seed,
                      uint64_t j, size_t k, size_t* delay);

/* Free-running asynchronous run (bounded staleness: every neighbour value a PE
 * consumes at step k is u_j(k*) with 0 <= k - k* <= q-1) with full edge logs,
 * for PEs of <= 1024 points (K3) or of whole 32-point units (K5, e.g. cfg3:
 * 512 PEs of 2^21 points).  On return `stats` holds the reader-relative
 * delay histogram and stats->residual_sum = sum_k ||u(k+1) - A u(k)||_inf, the
 * a-posteriori bound on ||u_async(K) - u_sync(K)||_inf (A = one synchronous
 * step; valid for 0 < r <= 1/2 where A is inf-norm non-expansive, plus a
 * K*8*eps*max|u| rounding allowance).  SURVEY.md §8a row 12. */
int heat_async_free_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                        size_t per_pe, size_t q, size_t k_end, double* final_out,
                        heat_async_stats* stats);

/* ---- ensembles (analysis.hpp:36-52) -------------------------------------- */
/* ensemble_run: `runs` members of the deterministic asynchronous scheme with
 * seeds base_seed + j (analysis.cpp:51-104), each recording l2_norm at steps
 * 0, stride, 2*stride, ... and k_end.  Fills steps_out[S] (S via n_steps),
 * norms[runs][S], terminals[runs][n] (may be NULL), mean_series[S] and
 * std_series[S] (population std), bit-identical to the reference.  All
 * three delay laws.  One CTA per member (K6) when the member's history fits
 * shared memory (N <= 4096, (q+1)*N*8 bytes <= 200 KB); otherwise members run
 * one after another on AsyncSimulator handles (K3/K5). */
int heat_ensemble_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                      size_t per_pe, size_t q, int law, size_t fixed_delay, double geometric_p,
                      size_t k_end,
                      size_t stride, size_t runs, uint64_t base_seed, size_t* steps_out,
                      size_t max_steps, size_t* n_steps, double* norms, double* terminals,
                      double* mean_series, double* std_series);

/* ---- executors (async_exec.hpp:53-70) ----------------------------------- */
/* exec_run: Barriered = bit-identical to sync_run (one launch-chain on the
 * GPU, no per-step barrier); BarrierFree = free-running PEs on the GPU with
 * bounded staleness q_free (0 selects the default 8) through acquire/release
 * halo rings.  duration_ns is device time of the run (CUDA events).  lag is
 * filled when record_lag != 0 (writer lag, LagStats semantics); stats (may be
 * NULL) receives the reader-relative delay log. */
int heat_exec_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                  size_t per_pe, size_t workers, size_t k_end, int mode, int record_lag,
                  size_t q_free, double* field_out, uint64_t* duration_ns, heat_lag_stats* lag,
                  heat_async_stats* stats);

/* ---- device-resident plans (bench, multi-GPU slabs) --------------------- */
typedef struct heat_plan heat_plan;
/* Allocates two device arrays of n doubles on `device` (ping-pong). */
int heat_plan_create(heat_plan** plan, size_t n, int device);
int heat_plan_destroy(heat_plan* plan);
/* Stream the plan's work is issued on (a cudaStream_t owned by the caller,
 * passed as an opaque handle; NULL = the plan's own stream). */
int heat_plan_set_stream(heat_plan* plan, void* stream);
int heat_plan_upload(heat_plan* plan, const double* host);
int heat_plan_download(heat_plan* plan, double* host);
/* Device-to-device copy of the owned points (stream-ordered on the plan's
 * stream), e.g. into a buffer of the final gather. */
int heat_plan_download_device(heat_plan* plan, void* dst_device);
/* Points [offset, offset + count) of the owned field to the host. */
int heat_plan_download_range(heat_plan* plan, size_t offset, size_t count, double* host);
/* Device IC u_i = sin(pi*i/(N-1)) with Dirichlet(0,0) ends snapped (bench only). */
int heat_plan_fill_sine(heat_plan* plan);
/* Advance the resident field by `steps` synchronous steps (no host sync). */
int heat_plan_sync_advance(heat_plan* plan, double r, int bc_kind, double c1, double c2,
                           size_t steps);
/* Advance by `steps` with the free-running async kernel on P = n/per_pe PEs
 * (delays bounded by q-1, observed delays logged in `stats`).  Each call is a
 * fresh run from the current field. */
int heat_plan_async_advance(heat_plan* plan, double r, int bc_kind, double c1, double c2,
                            size_t per_pe, size_t q, size_t steps, heat_async_stats* stats);
/* Same, deterministic: replays the DelayModel's seeded stream exactly as
 * async_run would (async_sim.cpp:77-160) for `steps` steps from step 0. */
int heat_plan_async_replay(heat_plan* plan, double r, int bc_kind, double c1, double c2,
                           size_t per_pe, size_t q, int law, size_t fixed_delay,
                           double geometric_p, uint64_t seed, size_t steps,
                           heat_async_stats* stats);
/* Blocks until the plan's stream is idle; reports strict-check / watchdog status. */
int heat_plan_synchronize(heat_plan* plan);
/* Device pointer of the current field (for peer copies / NCCL in multi-GPU). */
int heat_plan_device_ptr(heat_plan* plan, double** cur);

/* ---- multi-GPU slabs (1-D domain decomposition, no reference counterpart:
 * the reference is single-process) -------------------------
 * Rank `rank` of `world` owns n_local consecutive points of the global field.
 * Every pass of <= heat_slab_halo() steps needs fresh ghosts: pack the slab's
 * first/last H points into a 2H-double device buffer, exchange with the
 * neighbours (NCCL / peer copy), unpack the neighbours' points as ghosts.
 * Only the true global ends are pinned (rank 0 / rank world-1, Dirichlet);
 * periodic slabs wrap through the exchange. */
size_t heat_slab_halo(void);

/* ---- multi-GPU asynchronous slabs over NVLink P2P (north star (3)) ------
 * Rank r of `world` (a slab plan) runs the K5 asynchronous kernel on its
 * n_local points split into PEs of per_pe points; the PE boundaries between
 * ranks exchange edge values by P2P STORES into the neighbour's receive rings
 * (system-scope release/acquire).  With mode 1 and q = 1 every read is exact
 * and the run is the synchronous scheme; mode 0 replays a DelayModel's
 * stream (uniform/fixed) over the global PE enumeration, bit-identical to
 * async_run on the whole field.  Setup order on every rank:
 *   xlink_setup -> exchange handles (heat_xlink_handle_size() bytes; any
 *   transport) -> xlink_connect(left, right; NULL at Dirichlet ends);
 * then per run: xlink_seed -> barrier across ranks -> xlink_advance. */
size_t heat_xlink_handle_size(void);
int heat_plan_xlink_setup(heat_plan* plan, size_t per_pe, size_t q, int bc_kind, void* handle_out);
int heat_plan_xlink_connect(heat_plan* plan, const void* left_handle, const void* right_handle);
int heat_plan_xlink_seed(heat_plan* plan);
int heat_plan_xlink_advance(heat_plan* plan, double r, double c1, double c2, int mode, int law,
                            size_t fixed_delay, double geometric_p, uint64_t seed, size_t steps,
                            heat_async_stats* stats);
/* Test hook: slot 0 of the two receive rings (the neighbours' seeded values). */
int heat_plan_xlink_debug_recv(heat_plan* plan, double* out2);
int heat_plan_create_slab(heat_plan** plan, size_t n_local, int device, int rank, int world);
int heat_plan_halo_pack(heat_plan* plan, void* dst_device);
int heat_plan_halo_unpack(heat_plan* plan, const void* src_device);

#ifdef __cplusplus
}
#endif

#endif /* HEAT_B200_H */
