// sync_host.cu -- launch logic for K1 (sync_tb.cuh) and the synchronous
// C-ABI entry points: heat_sync_step / heat_sync_run / heat_sync_run_f32.
#include <algorithm>
#include <cmath>

#include "runtime.cuh"
#include "sync_tb.cuh"

namespace hb {

namespace {
constexpr int kV = 32;  // points per lane; also the maximum steps per pass

template <typename Real>
int occupancy_blocks(int sms) {
    static int cached[2] = {0, 0};
    int& slot = cached[sizeof(Real) == 8 ? 0 : 1];
    if (slot == 0) {
        using T = SyncTB<Real, kV>;
        HB_CUDA(cudaFuncSetAttribute(sync_tb_kernel<Real, kV>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, T::kSmemBytes));
        int per_sm = 0;
        HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sync_tb_kernel<Real, kV>,
                                                              T::kThreads, T::kSmemBytes));
        if (per_sm < 1) return fail(HEAT_ECUDA, "sync_tb_kernel does not fit on an SM");
        slot = per_sm;
    }
    return -slot;  // negative = ok, value = blocks per SM
}
}  // namespace

template <typename Real>
int sync_advance(int sms, Real* bufs[2], int& cur, long long n, double r, int periodic,
                 double c1, double c2, size_t steps, unsigned int* flag, cudaStream_t st) {
    using T = SyncTB<Real, kV>;
    if (steps == 0) return HEAT_OK;
    int occ = occupancy_blocks<Real>(sms);
    if (occ > 0) return occ;
    occ = -occ;
    const long long tiles = (n + T::kOut - 1) / T::kOut;
    const long long want = (tiles + T::kWarpsPerCta - 1) / T::kWarpsPerCta;
    const int grid = int(std::min<long long>(want, (long long)sms * occ));
    SyncPassArgs a{};
    a.n = n;
    a.tiles = tiles;
    a.r = r;
    if (sizeof(Real) == 8) {
        a.c = 1.0 - 2.0 * r;  // core.hpp:108: Real(1) - Real(2)*r, one rounding
    } else {
        const float rf = float(r);
        a.c = double(1.0f - 2.0f * rf);
    }
    a.c1 = c1;
    a.c2 = c2;
    a.periodic = periodic;
    a.nonfinite = flag;
    while (steps > 0) {
        const int s = int(std::min<size_t>(steps, T::kMaxSteps));
        a.src = bufs[cur];
        a.dst = bufs[cur ^ 1];
        a.nsteps = s;
        sync_tb_kernel<Real, kV><<<grid, T::kThreads, T::kSmemBytes, st>>>(a);
        HB_CUDA(cudaGetLastError());
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cur ^= 1;
        steps -= size_t(s);
    }
    return HEAT_OK;
}

template int sync_advance<double>(int, double* [2], int&, long long, double, int, double, double,
                                  size_t, unsigned int*, cudaStream_t);
template int sync_advance<float>(int, float* [2], int&, long long, double, int, double, double,
                                 size_t, unsigned int*, cudaStream_t);

namespace {

// Shared body of sync_run / sync_run_f32 (sync_solver.cpp:52-91).
template <typename Real>
int sync_run_impl(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                  size_t k_end, size_t stride, double* final_out, double* snapshots,
                  size_t* steps_out, size_t max_snapshots, size_t* n_snapshots) {
    HB_TRY(check_field(u0, n));
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    if (stride == 0) stride = default_stride(n);
    std::vector<double> start;
    HB_TRY(prepare_initial(u0, n, bc_kind, c1, c2, start));

    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(-1, &d));
    std::lock_guard<std::mutex> lock(d->mu);
    const size_t pitch = (n + 63) / 64 * 64;  // keep the second array 256-B aligned
    HB_TRY(ensure_buffers(*d, 2 * pitch * sizeof(Real)));
    Real* bufs[2] = {static_cast<Real*>(d->buf[0]), static_cast<Real*>(d->buf[0]) + pitch};
    cudaStream_t st = d->stream;

    std::vector<Real> host(n);
    for (size_t i = 0; i < n; ++i) host[i] = Real(start[i]);
    HB_CUDA(cudaMemcpyAsync(bufs[0], host.data(), n * sizeof(Real), cudaMemcpyHostToDevice, st));
    HB_CUDA(cudaMemsetAsync(d->flag, 0, 2 * sizeof(unsigned int), st));

    size_t ns = 0;
    auto record = [&](const Real* v, size_t k) {
        if (ns < max_snapshots) {
            if (snapshots)
                for (size_t i = 0; i < n; ++i) snapshots[ns * n + i] = double(v[i]);
            if (steps_out) steps_out[ns] = k;
        }
        ++ns;
    };
    record(host.data(), 0);

    const bool want_snaps = snapshots != nullptr || steps_out != nullptr;
    int cur = 0;
    size_t k = 0;
    const int periodic = bc_kind == HEAT_BC_PERIODIC;
    while (k < k_end) {
        // advance to the next recorded step (or straight to k_end)
        size_t next = want_snaps ? std::min(k_end, (k / stride + 1) * stride) : k_end;
        HB_TRY(sync_advance<Real>(d->sms, bufs, cur, (long long)n, r, periodic, c1, c2, next - k,
                                  d->flag, st));
        k = next;
        unsigned int flags[2] = {0, 0};
        HB_CUDA(cudaMemcpyAsync(flags, d->flag, sizeof flags, cudaMemcpyDeviceToHost, st));
        if (want_snaps || k == k_end)
            HB_CUDA(cudaMemcpyAsync(host.data(), bufs[cur], n * sizeof(Real),
                                    cudaMemcpyDeviceToHost, st));
        HB_CUDA(cudaStreamSynchronize(st));
        if (flags[0]) {
            if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
            return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
        }
        if (want_snaps) record(host.data(), k);
    }
    if (final_out)
        for (size_t i = 0; i < n; ++i) final_out[i] = double(host[i]);
    if (n_snapshots) *n_snapshots = ns;
    return HEAT_OK;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int heat_sync_step(const double* u, size_t n, double r, int bc_kind, double c1,
                              double c2, double* out) {
    return sync_run_impl<double>(u, n, r, bc_kind, c1, c2, 1, 1, out, nullptr, nullptr, 0,
                                 nullptr);
}

extern "C" int heat_sync_run(const double* u0, size_t n, double r, int bc_kind, double c1,
                             double c2, size_t k_end, size_t stride, double* final_out,
                             double* snapshots, size_t* steps, size_t max_snapshots,
                             size_t* n_snapshots) {
    return sync_run_impl<double>(u0, n, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                                 steps, max_snapshots, n_snapshots);
}

extern "C" int heat_sync_run_f32(const double* u0, size_t n, double r, int bc_kind, double c1,
                                 double c2, size_t k_end, size_t stride, double* final_out,
                                 double* snapshots, size_t* steps, size_t max_snapshots,
                                 size_t* n_snapshots) {
    return sync_run_impl<float>(u0, n, r, bc_kind, c1, c2, k_end, stride, final_out, snapshots,
                                steps, max_snapshots, n_snapshots);
}
