// small_cluster.cuh -- the cluster plumbing shared by the small-field kernels
// K7c (sync_small.cu) and K9 (async_small.cu): each CTA of the cluster keeps
// a full copy of the field in shared memory, double-buffered; the exact
// owners write each round's results into every copy, their own with plain
// stores and the other CTAs' with st.async, whose bytes complete on the
// receiver's mbarrier for that buffer.  A round ends with one __syncthreads
// and one wait for the mbarrier phase -- no cluster barrier, no memory fence
// (a fenced barrier.cluster compiles to MEMBAR.ALL.GPU + CCTL.IVALL).  K7c
// sends only the lane groups another CTA's halo needs (HaloGeo, put_mask);
// K9 sends its whole exact chunk and history rows (put_peers8 / put_peers2).
#pragma once
#include <cstdint>

namespace hb {
namespace {

__device__ __forceinline__ uint32_t small_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void small_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// (x, y) into the same 16 bytes of every other CTA of the cluster, each
// store completing its bytes on that CTA's mbarrier `bar` (st.async: no
// fence, no cluster barrier; the receiver waits on its own mbarrier)
__device__ __forceinline__ void put_peers2(const void* p, double x, double y, uint32_t bar,
                                           int rank, int ncta) {
    const uint32_t addr = uint32_t(__cvta_generic_to_shared(p));
    for (int j = 1; j < ncta; ++j) {  // the other CTAs, no skip branch
        const int c = rank + j < ncta ? rank + j : rank + j - ncta;
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(c));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(c));
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
            "d"(x), "d"(y), "r"(rb)
            : "memory");
    }
}
// V doubles (V/2 x 16 B) into the CTAs of `mask` (bit c: CTA c)
template <int V>
__device__ __forceinline__ void put_mask(const double* p, const double (&v)[V], uint32_t bar,
                                         uint32_t mask) {
    const uint32_t addr = uint32_t(__cvta_generic_to_shared(p));
    while (mask) {
        const int c = __ffs(mask) - 1;
        mask &= mask - 1;
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(c));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(c));
#pragma unroll
        for (int i = 0; i < V; i += 2)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                    ra + 8u * i),
                "d"(v[i]), "d"(v[i + 1]), "r"(rb)
                : "memory");
    }
}
// V doubles (V/2 x 16 B) into every other CTA: one mapa pair per peer
template <int V>
__device__ __forceinline__ void put_peers8(const double* p, const double (&v)[V], uint32_t bar,
                                           int rank, int ncta) {
    const uint32_t addr = uint32_t(__cvta_generic_to_shared(p));
    for (int j = 1; j < ncta; ++j) {
        const int c = rank + j < ncta ? rank + j : rank + j - ncta;
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(c));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(c));
#pragma unroll
        for (int i = 0; i < V; i += 2)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                    ra + 8u * i),
                "d"(v[i]), "d"(v[i + 1]), "r"(rb)
                : "memory");
    }
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}

// the two round mbarriers (one arrival each: the local expect_tx), visible to
// the cluster before any st.async targets them
__device__ __forceinline__ void small_bars_init(uint32_t bar0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void small_bar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// Halo-only exchange geometry (K7c).  CTA c of a cluster owns the exact points
// [lo_c, hi_c), lo_c = c * wpc * C, hi_c = min(lo_c + wpc * C, N), C being
// a window's exact width; its windows read H points beyond each end (mod N
// when periodic, clipped to the field for Dirichlet).  A lane group of V
// points starting at g (V | H, V | C, V | N) is sent to CTA c iff it lies in
// c's halo and c does not own it; the receiver counts the same groups.
struct HaloGeo {
    int N, C, H, wpc, ncta, periodic;
    __device__ __forceinline__ int owner(int x) const { return (x / C) / wpc; }
    __device__ __forceinline__ bool needs(int c, int g) const {
        const int lo = c * wpc * C;
        if (lo >= N || owner(g) == c) return false;
        const int hi = min(lo + wpc * C, N);
        if (periodic) {
            const int dl = ((lo - g) % N + N) % N;  // g in [lo - H, lo) mod N
            const int dr = ((g - hi) % N + N) % N;  // g in [hi, hi + H) mod N
            return (dl >= 1 && dl <= H) || dr < H;
        }
        return (g >= lo - H && g < lo) || (g >= hi && g < hi + H);
    }
};
}  // namespace
}  // namespace hb
