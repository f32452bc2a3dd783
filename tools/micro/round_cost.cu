// Cost of one K7c round exchange with no stepping: each lane of lanes 8..23
// writes 64 B into the next buffer of its own CTA and (st.async) into every
// peer's, __syncthreads, the mbarrier wait, then the window reload.  Compare
// with a plain cluster barrier round.  nvcc -gencode arch=compute_100a,code=sm_100a
// -I../../paper_1510_08982_b200/csrc -o round_cost round_cost.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "small_cluster.cuh"
using namespace hb;

template <int MODE>
__global__ void rounds(int nrounds, int ncta, double* out, long long* cyc) {
    extern __shared__ double smem[];
    __shared__ __align__(8) unsigned long long sbar[2];
    const int N = 128 * int(gridDim.x) * int(blockDim.x >> 5), Np = N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = int(small_ctarank());
    const int gw = rank * int(blockDim.x >> 5) + w;
    double* su = smem;
    for (int i = threadIdx.x; i < 2 * Np; i += blockDim.x) su[i] = i;
    const long long g0 = gw * 128 - 64 + lane * 8;
    const bool lexact = lane >= 8 && lane < 24;
    const int wg0 = int(((g0 % N) + N) % N);
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&sbar[0]));
    const uint32_t incoming = uint32_t(N * 8 - __syncthreads_count(lexact) * 64);
    if (threadIdx.x == 0) small_bars_init(bar0);
    small_cluster_sync();
    double u[8];
    int par = 0;
    uint32_t phases = 0;
    long long t0 = clock64();
    for (int j = 0; j < nrounds; ++j) {
        const double* cu = su + par * Np;
        double* nu = su + (par ^ 1) * Np;
        const uint32_t nbar = bar0 + 8u * uint32_t(par ^ 1);
        if (MODE == 0 && threadIdx.x == 0) small_bar_expect(nbar, incoming);
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const double2 x = *reinterpret_cast<const double2*>(&cu[wg0 + i]);
            u[i] = x.x + 1.0;
            u[i + 1] = x.y;
        }
        if (lexact) {
#pragma unroll
            for (int i = 0; i < 8; i += 2)
                *reinterpret_cast<double2*>(&nu[g0 + i]) = make_double2(u[i], u[i + 1]);
            if (MODE == 0) put_peers8<8>(&nu[g0], u, nbar, rank, ncta);
        }
        if (MODE == 0) {
            __syncthreads();
            const int b = par ^ 1;
            mbar_wait_parity(nbar, (phases >> b) & 1u);
            phases ^= 1u << b;
        } else if (MODE == 1) {
            small_cluster_sync();
        } else {
            __syncthreads();
        }
        par ^= 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) *cyc = t1 - t0;
    if (rank == 0 && threadIdx.x < 8) out[threadIdx.x] = su[threadIdx.x];
}

template <int MODE>
void run(const char* name, int ncta, int wpc) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&cyc, 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(32 * wpc);
    cfg.dynamicSmemBytes = 2 * 128 * ncta * wpc * 8;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nr = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, rounds<MODE>, nr, ncta, out, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s ncta=%d wpc=%d: %.1f ns/round, %.0f cycles/round (%s)\n", name, ncta, wpc,
           ms * 1e6 / nr, double(c) / nr, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<0>("st.async + mbarrier", 2, 4);
    run<1>("cluster barrier", 2, 4);
    run<2>("syncthreads only (no peers)", 2, 4);
    run<0>("st.async + mbarrier", 4, 4);
    run<1>("cluster barrier", 4, 4);
    run<0>("st.async + mbarrier", 8, 4);
    return 0;
}
