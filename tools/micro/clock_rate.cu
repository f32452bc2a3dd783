// SM clock while one small kernel runs alone: clock64 vs globaltimer.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long* out, long long ns) {
    long long g0, g1, c0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); } while (g1 - g0 < ns);
    long long c1 = clock64();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = g1 - g0; }
}
int main() {
    long long* d; cudaMalloc(&d, 16);
    for (long long ns : {20000LL, 200000LL, 2000000LL, 20000000LL}) {
        spin<<<1, 32>>>(d, ns);
        long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("spin %lld ns: %.0f MHz\n", ns, h[0] * 1e3 / h[1]);
    }
    return 0;
}
