// runtime.cu -- library state, per-device workspace, validation helpers and
// the small C-ABI entry points (errors, strict checks, trajectory sizing).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <memory>
#include <utility>

#include <cstring>
#include <thread>
#include <vector>

#include "runtime.cuh"

namespace hb {

std::atomic<uint64_t> g_launches{0};
std::atomic<bool> g_strict{false};

namespace {
thread_local std::string t_error;
std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevCtx>> g_ctx;
}  // namespace

void set_error(const std::string& msg) { t_error = msg; }
std::string last_error_msg() { return t_error; }

int dev_ctx(int device, DevCtx** out) {
    if (device < 0) {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            return fail(HEAT_ENODEV, std::string("no CUDA device available: ") +
                                         (e == cudaSuccess ? "count = 0" : cudaGetErrorString(e)));
        HB_CUDA(cudaGetDevice(&device));
    }
    DevCtx* d = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_ctx_mu);
        if (g_ctx.size() <= size_t(device)) g_ctx.resize(size_t(device) + 1);
        if (!g_ctx[device]) g_ctx[device] = std::make_unique<DevCtx>();
        d = g_ctx[device].get();
    }
    HB_CUDA(cudaSetDevice(device));
    if (d->device < 0) {
        std::lock_guard<std::mutex> lock(d->mu);
        if (d->device < 0) {
            cudaDeviceProp prop{};
            HB_CUDA(cudaGetDeviceProperties(&prop, device));
            if (prop.major < 10)
                return fail(HEAT_ENODEV, std::string("device ") + prop.name +
                                             " is not sm_100 (Blackwell); this build targets sm_100a only");
            d->sms = prop.multiProcessorCount;
            HB_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
            HB_CUDA(cudaStreamCreateWithFlags(&d->h2d, cudaStreamNonBlocking));
            HB_CUDA(cudaStreamCreateWithFlags(&d->d2h, cudaStreamNonBlocking));
            HB_CUDA(cudaStreamCreateWithFlags(&d->stream2, cudaStreamNonBlocking));
            HB_CUDA(cudaMalloc(&d->flag, kFlagWords * sizeof(unsigned int)));
            d->device = device;
        }
    }
    *out = d;
    return HEAT_OK;
}

int ensure_buffers(DevCtx& d, size_t bytes) {
    if (d.bytes >= bytes) return HEAT_OK;
    if (d.buf[0]) cudaFree(d.buf[0]);
    d.buf[0] = nullptr;
    d.bytes = 0;
    cudaError_t e = cudaMalloc(&d.buf[0], bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HEAT_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) +
                                     "): " + cudaGetErrorString(e));
    }
    d.bytes = bytes;
    return HEAT_OK;
}

int kernel_smem_config(const void* fn, int smem, int threads, int* per_sm) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> cache;  // (kernel, device) -> CTAs/SM
    int dev = 0;
    HB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({fn, dev});
    if (it != cache.end()) {
        *per_sm = it->second;
        return HEAT_OK;
    }
    HB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int n = 0;
    HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem));
    if (n < 1) return fail(HEAT_ECUDA, "kernel does not fit on an SM");
    cache[{fn, dev}] = n;
    *per_sm = n;
    return HEAT_OK;
}

int ensure_scratch(DevCtx& d, size_t bytes) {
    if (d.scratch_bytes >= bytes) return HEAT_OK;
    if (d.scratch) cudaFree(d.scratch);
    d.scratch = nullptr;
    d.scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&d.scratch, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HEAT_ENOMEM, std::string("cudaMalloc(scratch ") + std::to_string(bytes) +
                                     "): " + cudaGetErrorString(e));
    }
    d.scratch_bytes = bytes;
    return HEAT_OK;
}

int host_ring(DevCtx& d, unsigned char** slots) {
    if (!d.ring) {
        HB_CUDA(cudaHostAlloc(&d.ring, kRingSlots * kRingSlotBytes, cudaHostAllocDefault));
        for (auto& e : d.ring_ev) HB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (int j = 0; j < kRingSlots; ++j)
        slots[j] = static_cast<unsigned char*>(d.ring) + size_t(j) * kRingSlotBytes;
    return HEAT_OK;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
    constexpr size_t kMinPart = 8ull << 20;
    const int T = int(std::max<size_t>(1, std::min<size_t>(size_t(threads), bytes / kMinPart)));
    if (T <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(size_t(T));
    const size_t part = (bytes / size_t(T) + 63) / 64 * 64;
    for (int t = 0; t < T; ++t) {
        const size_t lo = size_t(t) * part;
        if (lo >= bytes) break;
        const size_t len = std::min(part, bytes - lo);
        pool.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, len);
        });
    }
    for (auto& th : pool) th.join();
}

bool host_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear it: an unknown pointer is ordinary host memory
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

unsigned char* host_stage(DevCtx& d, size_t bytes) {
    if (bytes > kHostStageMax) return nullptr;
    if (d.host_bytes < bytes) {
        if (d.host) cudaFreeHost(d.host);
        d.host = nullptr;
        d.host_bytes = 0;
        const size_t want = std::max<size_t>(bytes, 1u << 20);
        if (cudaMallocHost(&d.host, want) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        d.host_bytes = want;
    }
    return static_cast<unsigned char*>(d.host);
}

int check_field(const double* u, size_t n) {
    if (n < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    if (!u) return fail(HEAT_EINVAL, "null field pointer");
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(u[i])) return fail(HEAT_EDOMAIN, "TemperatureField values must be finite");
    return HEAT_OK;
}

namespace {
// The reference's unclamped geometric delay of a draw with top bits m.
double geometric_quotient(uint64_t m, double lp) {
    return std::log1p(-(double(m) * 0x1.0p-53)) / lp;
}
size_t geometric_raw(uint64_t m, double lp) {
    double g = std::floor(geometric_quotient(m, lp));
    if (!std::isfinite(g) || g < 0.0) g = 0.0;
    return size_t(g);
}
}  // namespace

int geometric_thresholds(double p, size_t q, std::vector<uint64_t>& T) {
    static std::mutex mu;
    static std::map<std::pair<uint64_t, size_t>, std::vector<uint64_t>> cache;
    uint64_t pbits;
    std::memcpy(&pbits, &p, 8);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(pbits, q);
    if (auto it = cache.find(key); it != cache.end()) {
        T = it->second;
        return HEAT_OK;
    }
    constexpr uint64_t kTop = uint64_t(1) << 53;  // m ranges over [0, 2^53)
    const double lp = std::log1p(-p);
    const double qmax = geometric_quotient(kTop - 1, lp);
    if (!std::isfinite(qmax) || qmax >= 0x1.0p62)
        return fail(HEAT_EINVAL, "geometric law: p too small for the device delay thresholds");
    T.assign(q > 0 ? q - 1 : 0, kTop);
    const double slope = std::max(1.0, std::ceil(std::fabs(lp)));
    for (size_t j = 1; j < q; ++j) {
        if (geometric_raw(kTop - 1, lp) < j) break;  // T[j-1..] stay 2^53: never reached
        uint64_t lo = 0, hi = kTop - 1;               // smallest m with raw(m) >= j
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (geometric_raw(mid, lp) >= j) hi = mid;
            else lo = mid + 1;
        }
        T[j - 1] = lo;
        // rounding can move the crossing by a few ulps of the quotient (~j ulps of
        // m per unit slope): check every m within a window far wider than that
        const uint64_t W = std::min<uint64_t>(uint64_t(64.0 * double(j) * slope) + 4096, 1u << 22);
        const uint64_t a = lo > W ? lo - W : 0, b = std::min(kTop, lo + W);
        for (uint64_t m = a; m < b; ++m)
            if ((geometric_raw(m, lp) >= j) != (m >= lo))
                return fail(HEAT_EINVAL, "geometric law: delay not monotone near a threshold");
    }
    cache.emplace(key, T);
    return HEAT_OK;
}

int prepare_initial(const double* u0, size_t n, int bc_kind, double c1, double c2,
                    std::vector<double>& out) {
    out.assign(u0, u0 + n);
    if (bc_kind == HEAT_BC_DIRICHLET) {
        constexpr double kTol = 1e-9;  // kDirichletEndTol, sync_solver.hpp:44
        if (std::abs(out.front() - c1) > kTol || std::abs(out.back() - c2) > kTol)
            return fail(HEAT_EINVAL, "Dirichlet BC inconsistent with initial end values");
        out.front() = c1;
        out.back() = c2;
    }
    return HEAT_OK;
}

}  // namespace hb

using namespace hb;

extern "C" {

const char* heat_last_error(void) { return t_error.c_str(); }

const char* heat_version(void) { return "heat_b200 0.1 (sm_100a)"; }

int heat_set_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(HEAT_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= count) return fail(HEAT_EINVAL, "heat_set_device: no such device");
    HB_CUDA(cudaSetDevice(device));
    return HEAT_OK;
}

int heat_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t heat_kernel_launches(void) { return g_launches.load(); }

void heat_set_strict_finite_checks(int enabled) { g_strict = enabled != 0; }
int heat_strict_finite_checks(void) { return g_strict ? 1 : 0; }

int heat_prepare_initial(const double* u0, size_t n, int bc_kind, double c1, double c2,
                         double* out) {
    if (!u0 || !out) return fail(HEAT_EINVAL, "null field pointer");
    if (n < 3) return fail(HEAT_EDOMAIN, "TemperatureField requires N >= 3");
    std::vector<double> v;
    HB_TRY(prepare_initial(u0, n, bc_kind, c1, c2, v));
    std::memcpy(out, v.data(), n * sizeof(double));
    return HEAT_OK;
}

int heat_geometric_thresholds(double p, size_t q, uint64_t* thresholds) {
    if (!thresholds) return fail(HEAT_EINVAL, "null output");
    if (q == 0) return fail(HEAT_EDOMAIN, "DelayModel: q >= 1 required");
    if (!(p > 0.0) || p > 1.0) return fail(HEAT_EDOMAIN, "DelayModel: geometric p must lie in (0, 1]");
    std::vector<uint64_t> T;
    HB_TRY(geometric_thresholds(p, q, T));
    std::copy(T.begin(), T.end(), thresholds);
    return HEAT_OK;
}

size_t heat_trajectory_length(size_t n, size_t k_end, size_t stride) {
    if (stride == 0) stride = default_stride(n);
    size_t count = 1 + k_end / stride;
    if (k_end % stride != 0) ++count;
    return count;
}

}  // extern "C"
