// async_host.cu -- asynchronous entry points (placeholder until K3/K4 land).
#include <cmath>

#include "common.cuh"
#include "runtime.cuh"

using namespace hb;

extern "C" {

int heat_sample_delay(size_t q, int law, size_t fixed_delay, double geometric_p, uint64_t seed,
                      uint64_t j, size_t k, size_t* delay) {
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    const size_t bound = std::min(q - 1, k);
    const uint64_t x = splitmix_draw(seed, j);
    switch (law) {
        case HEAT_DELAY_UNIFORM: *delay = size_t(x % (bound + 1)); return HEAT_OK;
        case HEAT_DELAY_FIXED:
            if (fixed_delay >= q) return fail(HEAT_EDOMAIN, "DelayModel: fixed delay must satisfy d < q");
            *delay = std::min(fixed_delay, bound);
            return HEAT_OK;
        case HEAT_DELAY_GEOMETRIC: {
            if (!(geometric_p > 0.0) || geometric_p > 1.0)
                return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
            const double u = double(x >> 11) * 0x1.0p-53;
            double g = std::floor(std::log1p(-u) / std::log1p(-geometric_p));
            if (!std::isfinite(g) || g < 0.0) g = 0.0;
            *delay = std::min(size_t(g), bound);
            return HEAT_OK;
        }
    }
    return fail(HEAT_ELOGIC, "sample_delay: unknown distribution");
}

int heat_async_run(const double*, size_t, double, int, double, double, size_t, size_t, int,
                   size_t, double, uint64_t, size_t, size_t, double*, double*, size_t*, size_t,
                   size_t*) {
    return fail(HEAT_ENODEV, "heat_async_run: not built yet");
}

int heat_exec_run(const double* u0, size_t n, double r, int bc_kind, double c1, double c2,
                  size_t per_pe, size_t workers, size_t k_end, int mode, int record_lag,
                  size_t q_free, double* field_out, uint64_t* duration_ns, heat_lag_stats* lag,
                  heat_async_stats* stats) {
    (void)record_lag;
    (void)q_free;
    (void)lag;
    (void)stats;
    // exec_run validation order (async_exec.cpp:263-272)
    HB_TRY(check_field(u0, n));
    if (per_pe == 0 || n % per_pe != 0) return fail(HEAT_EDOMAIN, "PartitionSpec: n must divide N");
    if (workers == 0 || workers != n / per_pe)
        return fail(HEAT_EINVAL, "exec_run: cfg.workers must equal part.P");
    if (k_end == 0) return fail(HEAT_EINVAL, "exec_run: k_end >= 1 required");
    if (mode != HEAT_EXEC_BARRIERED) return fail(HEAT_ENODEV, "heat_exec_run: barrier-free not built yet");
    cudaEvent_t e0, e1;
    HB_CUDA(cudaEventCreate(&e0));
    HB_CUDA(cudaEventCreate(&e1));
    int st = heat_sync_run(u0, n, r, bc_kind, c1, c2, k_end, k_end, field_out, nullptr, nullptr, 0,
                           nullptr);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (duration_ns) *duration_ns = 0;
    return st;
}

int heat_plan_async_advance(heat_plan*, double, int, double, double, size_t, size_t, size_t,
                            heat_async_stats*) {
    return fail(HEAT_ENODEV, "heat_plan_async_advance: not built yet");
}

}  // extern "C"
