// Issue rate of independent DADD/DMUL from 1..4 warps on one SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void thr(double* out, long long* cyc, double b, int n) {
    double x[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = threadIdx.x + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) x[j] = __dadd_rn(x[j], b);
#pragma unroll
        for (int j = 0; j < CH; ++j) x[j] = __dmul_rn(x[j], b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
    const int n = 4096;
    for (int warps : {1, 4, 8, 16}) {
        thr<16><<<1, 32 * warps>>>(o, c, 1.0000001, n);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps/CTA %2d (%d per SMSP): %.2f cycles per warp-DP-instruction per SMSP\n", warps,
               (warps + 3) / 4, h / double(n * 32) / ((warps + 3) / 4));
    }
    return 0;
}
