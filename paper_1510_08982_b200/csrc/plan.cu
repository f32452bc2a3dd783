// plan.cu -- device-resident plans: a field that lives in HBM across calls
// (bench, multi-GPU slabs).  Two ping-pong arrays of n doubles per plan.
#include <cmath>

#include "runtime.cuh"

struct heat_plan {
    int device = 0;
    size_t n = 0;
    size_t pitch = 0;
    double* base = nullptr;
    int cur = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    unsigned int* flag = nullptr;
    int sms = 0;
    double* bufs[2] = {nullptr, nullptr};
};

namespace hb {
namespace {

__global__ void fill_sine_kernel(double* u, long long n) {
    const double pi = 3.14159265358979323846;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double v = sin(pi * double(i) / double(n - 1));
        if (i == 0 || i == n - 1) v = 0.0;  // Dirichlet(0,0) snap (sync_solver.cpp:33-34)
        u[i] = v;
    }
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" {

int heat_plan_create(heat_plan** out, size_t n, int device) {
    if (!out) return fail(HEAT_EINVAL, "null plan pointer");
    if (n < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    DevCtx* d = nullptr;
    HB_TRY(dev_ctx(device, &d));
    auto* p = new heat_plan();
    p->device = d->device;
    p->n = n;
    p->pitch = (n + 63) / 64 * 64;
    p->sms = d->sms;
    cudaError_t e = cudaMalloc(&p->base, 2 * p->pitch * sizeof(double));
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete p;
        return fail(HEAT_ENOMEM, std::string("plan cudaMalloc: ") + cudaGetErrorString(e));
    }
    p->bufs[0] = p->base;
    p->bufs[1] = p->base + p->pitch;
    HB_CUDA(cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking));
    p->stream = p->own;
    HB_CUDA(cudaMalloc(&p->flag, 4 * sizeof(unsigned int)));
    HB_CUDA(cudaMemset(p->flag, 0, 4 * sizeof(unsigned int)));
    *out = p;
    return HEAT_OK;
}

int heat_plan_destroy(heat_plan* p) {
    if (!p) return HEAT_OK;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    cudaFree(p->base);
    cudaFree(p->flag);
    cudaStreamDestroy(p->own);
    delete p;
    return HEAT_OK;
}

int heat_plan_set_stream(heat_plan* p, void* stream) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    p->stream = stream ? static_cast<cudaStream_t>(stream) : p->own;
    return HEAT_OK;
}

int heat_plan_upload(heat_plan* p, const double* host) {
    if (!p || !host) return fail(HEAT_EINVAL, "null plan or host pointer");
    HB_CUDA(cudaSetDevice(p->device));
    HB_CUDA(cudaMemcpyAsync(p->bufs[p->cur], host, p->n * sizeof(double), cudaMemcpyHostToDevice,
                            p->stream));
    return HEAT_OK;
}

int heat_plan_download(heat_plan* p, double* host) {
    if (!p || !host) return fail(HEAT_EINVAL, "null plan or host pointer");
    HB_CUDA(cudaSetDevice(p->device));
    HB_CUDA(cudaMemcpyAsync(host, p->bufs[p->cur], p->n * sizeof(double), cudaMemcpyDeviceToHost,
                            p->stream));
    HB_CUDA(cudaStreamSynchronize(p->stream));
    return HEAT_OK;
}

int heat_plan_fill_sine(heat_plan* p) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    HB_CUDA(cudaSetDevice(p->device));
    fill_sine_kernel<<<p->sms * 8, 256, 0, p->stream>>>(p->bufs[p->cur], (long long)p->n);
    HB_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return HEAT_OK;
}

int heat_plan_sync_advance(heat_plan* p, double r, int bc_kind, double c1, double c2,
                           size_t steps) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    if (bc_kind != HEAT_BC_DIRICHLET && bc_kind != HEAT_BC_PERIODIC)
        return fail(HEAT_EINVAL, "unknown boundary condition kind");
    HB_CUDA(cudaSetDevice(p->device));
    return sync_advance<double>(p->sms, p->bufs, p->cur, (long long)p->n, r,
                                bc_kind == HEAT_BC_PERIODIC, c1, c2, steps, p->flag, p->stream);
}

int heat_plan_synchronize(heat_plan* p) {
    if (!p) return fail(HEAT_EINVAL, "null plan");
    HB_CUDA(cudaSetDevice(p->device));
    unsigned int flags[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(flags, p->flag, sizeof flags, cudaMemcpyDeviceToHost, p->stream));
    HB_CUDA(cudaStreamSynchronize(p->stream));
    if (flags[1]) return fail(HEAT_ETIMEOUT, "async halo-ring wait exceeded its deadline");
    if (flags[0]) {
        HB_CUDA(cudaMemsetAsync(p->flag, 0, 2 * sizeof(unsigned int), p->stream));
        if (g_strict.load()) return fail(HEAT_EDIVERGE, "non-finite value produced by step");
        return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    }
    return HEAT_OK;
}

int heat_plan_device_ptr(heat_plan* p, double** cur) {
    if (!p || !cur) return fail(HEAT_EINVAL, "null plan or output pointer");
    *cur = p->bufs[p->cur];
    return HEAT_OK;
}

}  // extern "C"
