// common.cuh -- shared device helpers for the sm_100a FTCS kernels.
//
// The stencil is evaluated exactly as the reference's stencil<Real>
// (core.hpp:106-109): r*R + (1-2r)*S + r*L, left-associative, three
// separately-rounded products and two separately-rounded sums, NO FMA.
// __dmul_rn/__dadd_rn (and the float twins) forbid contraction regardless of
// -fmad, so the SASS carries DMUL/DADD only (SURVEY.md probe P6).
//
// Products r*u_j are shared between the two stencils that use them
// (u_{j-1} as its right term, u_{j+1} as its left term): IEEE multiplication
// is commutative and deterministic, so reusing the product is bit-identical
// and cuts the FP64 work to 4 instructions per update (2 DMUL + 2 DADD).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hb {

constexpr int kWarp = 32;

template <typename Real> struct Arith;
template <> struct Arith<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct Arith<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

// ((pR + c*S) + pL) with pR = r*R and pL = r*L already rounded.
template <typename Real>
__device__ __forceinline__ Real stencil_p(Real pR, Real cS, Real pL) {
    return Arith<Real>::add(Arith<Real>::add(pR, cS), pL);
}

// ---- SplitMix64 (rng.hpp:16-41), counter form -----------------------------
// The reference's stream advances state += gamma before mixing, so draw j
// (0-based) of a stream seeded with s is mix(s + (j+1)*gamma).
__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t j) {
    return splitmix_mix(seed + (j + 1) * 0x9e3779b97f4a7c15ULL);
}

// x mod m for a 32-bit m fixed per run (the uniform law's steady-state
// modulus q).  With t = 2^32 mod m, x = hi*2^32 + lo ≡ v = hi*t + lo < 2^64,
// and floor(v * floor((2^64-1)/m) / 2^64) is v's quotient or one less
// (the error is below v/2^64 < 1), so one conditional subtract finishes.
// Replaces a chain of variable 32-bit divisions on every cross-PE read.
struct ModQ {
    unsigned long long M;
    unsigned int m, t;
};
__host__ __device__ inline ModQ make_modq(unsigned int m) {
    return ModQ{~0ull / m, m, static_cast<unsigned int>((1ull << 32) % m)};
}
__device__ __forceinline__ unsigned int modq(uint64_t x, const ModQ& f) {
    const uint64_t v = uint64_t(uint32_t(x >> 32)) * f.t + uint32_t(x);
    const uint64_t r = v - __umul64hi(v, f.M) * f.m;
    return uint32_t(r >= f.m ? r - f.m : r);
}
// Uniform-law delay x mod (bound + 1), bound = min(k, q-1)
// (async_sim.cpp:57-73): the fast path for every step k >= q-1.
__device__ __forceinline__ int uniform_delay(uint64_t x, long long bound, const ModQ& fq) {
    if (bound + 1 == (long long)fq.m) return int(modq(x, fq));
    return int(x % uint64_t(bound + 1));  // the first q-1 steps only
}

// Geometric-law delay from the thresholds of geometric_thresholds()
// (runtime.cuh): T[j-1] is the first top-53-bits value whose delay is >= j.
__device__ __forceinline__ int geometric_delay(uint64_t x, const uint64_t* T, int bound) {
    const uint64_t m = x >> 11;
    int d = 0;
    while (d < bound && m >= T[d]) ++d;
    return d;
}

// ---- shared-memory / async-proxy PTX wrappers -----------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completes on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1-D bulk copy shared -> global (bulk-group completion, per issuing thread).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Order this thread's generic-proxy shared-memory accesses against later
// async-proxy (bulk copy) accesses of the same bytes, and vice versa.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- scoped acquire/release on generic addresses (rings, flags) ----------
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// system scope: words written by another GPU over NVLink (P2P stores)
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_gpu_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu_f64(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_cta_shared(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_shared(uint64_t* p, uint64_t v) {
    asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename Real>
__device__ __forceinline__ bool finite_val(Real x) {
    return isfinite(x);
}

}  // namespace hb
