// plan.cu -- device-resident plans: a field that lives in HBM across calls
// (bench, multi-GPU slabs).  Two ping-pong arrays of n doubles per plan.
#include <cmath>

#include "runtime.cuh"


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
    p->pitch = (n + 2 * kSlabHalo + 63) / 64 * 64;
    p->sms = d->sms;
    cudaError_t e = cudaMalloc(&p->base, 2 * p->pitch * sizeof(double));
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete p;
        return fail(HEAT_ENOMEM, std::string("plan cudaMalloc: ") + cudaGetErrorString(e));
    }
    p->ext[0] = p->base;
    p->ext[1] = p->base + p->pitch;
    p->bufs[0] = p->ext[0] + kSlabHalo;
    p->bufs[1] = p->ext[1] + kSlabHalo;
    HB_CUDA(cudaMemset(p->base, 0, 2 * p->pitch * sizeof(double)));
    HB_CUDA(cudaStreamCreateWithFlags(&p->own, cudaStreamNonBlocking));
    p->stream = p->own;
    HB_CUDA(cudaMalloc(&p->flag, kFlagWords * sizeof(unsigned int)));
    HB_CUDA(cudaMemset(p->flag, 0, 4 * sizeof(unsigned int)));
    *out = p;
    return HEAT_OK;
}

int heat_plan_destroy(heat_plan* p) {
    if (!p) return HEAT_OK;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    xlink_release(p);
    cudaFree(p->base);
    cudaFree(p->flag);
    if (p->async_scratch) cudaFree(p->async_scratch);
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

int heat_plan_download_range(heat_plan* p, size_t offset, size_t count, double* host) {
    if (!p || !host) return fail(HEAT_EINVAL, "null plan or host pointer");
    if (offset > p->n || count > p->n - offset) return fail(HEAT_EINVAL, "range outside the plan");
    HB_CUDA(cudaSetDevice(p->device));
    HB_CUDA(cudaMemcpyAsync(host, p->bufs[p->cur] + offset, count * sizeof(double),
                            cudaMemcpyDeviceToHost, p->stream));
    HB_CUDA(cudaStreamSynchronize(p->stream));
    return HEAT_OK;
}

int heat_plan_download_device(heat_plan* p, void* dst_device) {
    if (!p || !dst_device) return fail(HEAT_EINVAL, "null plan or device pointer");
    HB_CUDA(cudaSetDevice(p->device));
    HB_CUDA(cudaMemcpyAsync(dst_device, p->bufs[p->cur], p->n * sizeof(double),
                            cudaMemcpyDeviceToDevice, p->stream));
    return HEAT_OK;  // stream-ordered on the plan's stream
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
    if (p->world == 1)
        return sync_advance<double>(p->sms, p->bufs, p->cur, (long long)p->n, r,
                                    bc_kind == HEAT_BC_PERIODIC, c1, c2, steps, p->flag,
                                    p->stream);
    if (steps > size_t(kSlabHalo))
        return fail(HEAT_EINVAL, "slab plans advance at most heat_slab_halo() steps per exchange");
    const bool dir = bc_kind == HEAT_BC_DIRICHLET;
    SlabGeom g;
    g.len = (long long)p->n + 2 * kSlabHalo;
    g.out_lo = kSlabHalo;
    g.out_hi = kSlabHalo + (long long)p->n;
    g.pin_lo = (dir && p->rank == 0) ? kSlabHalo : -1;
    g.pin_hi = (dir && p->rank == p->world - 1) ? kSlabHalo + (long long)p->n - 1 : -1;
    g.wrap = 0;
    return sync_advance_slab<double>(p->sms, p->ext, p->cur, g, r, c1, c2, steps, p->flag,
                                     p->stream, kSlabHalo);
}

size_t heat_slab_halo(void) { return size_t(kSlabHalo); }

int heat_plan_create_slab(heat_plan** out, size_t n_local, int device, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) return fail(HEAT_EINVAL, "bad rank/world");
    if (n_local < size_t(kSlabHalo))
        return fail(HEAT_EDOMAIN, "slab smaller than the halo width");
    HB_TRY(heat_plan_create(out, n_local, device));
    (*out)->rank = rank;
    (*out)->world = world;
    return HEAT_OK;
}

int heat_plan_halo_pack(heat_plan* p, void* dst) {
    if (!p || !dst) return fail(HEAT_EINVAL, "null plan or buffer");
    HB_CUDA(cudaSetDevice(p->device));
    const size_t H = kSlabHalo, b = H * sizeof(double);
    double* cur = p->bufs[p->cur];
    HB_CUDA(cudaMemcpyAsync(dst, cur, b, cudaMemcpyDeviceToDevice, p->stream));
    HB_CUDA(cudaMemcpyAsync(static_cast<double*>(dst) + H, cur + p->n - H, b,
                            cudaMemcpyDeviceToDevice, p->stream));
    return HEAT_OK;
}

int heat_plan_halo_unpack(heat_plan* p, const void* src) {
    if (!p || !src) return fail(HEAT_EINVAL, "null plan or buffer");
    HB_CUDA(cudaSetDevice(p->device));
    const size_t H = kSlabHalo, b = H * sizeof(double);
    double* ext = p->ext[p->cur];
    HB_CUDA(cudaMemcpyAsync(ext, src, b, cudaMemcpyDeviceToDevice, p->stream));
    HB_CUDA(cudaMemcpyAsync(ext + H + p->n, static_cast<const double*>(src) + H, b,
                            cudaMemcpyDeviceToDevice, p->stream));
    return HEAT_OK;
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
