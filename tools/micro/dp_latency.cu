// Dependent-chain latency of DADD / DMUL / SHFL / LDS on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    __shared__ double sm[64];
    sm[threadIdx.x] = b;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    long long t3 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = (int)v & 31; x += v; }
    long long t4 = clock64();
    float y = float(a);
    for (int i = 0; i < n; ++i) y = __fadd_rn(y, float(b));
    long long t5 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    const int n = 4096;
    for (int rep = 0; rep < 3; ++rep) {
        lat<<<1, 32>>>(o, c, 1.0, 1e-9, n);
        long long h[5]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
        printf("per op cycles: DADD %.1f  DMUL %.1f  SHFL %.1f  LDS(+DADD) %.1f  FADD %.1f\n",
               h[0] / double(n), h[1] / double(n), h[2] / double(n), h[3] / double(n), h[4] / double(n));
    }
    return 0;
}
