// Fixed cost of a small call on this box: an empty kernel + stream sync, the
// same with a cluster launch, a 1-step heat_async_run / heat_sync_run through
// the C-ABI, and cudaMemcpyAsync round trips.  nvcc -gencode arch=compute_100a,code=sm_100a
// -o call_floor call_floor.cu -I../../include -L../../paper_1510_08982_b200 -lheat_b200
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "heat_b200.h"

__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 1000) *p = 1;
}

template <class F>
double best_us(F f, int reps = 200) {
    double b = 1e30;
    for (int i = 0; i < reps; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        f();
        auto t1 = std::chrono::steady_clock::now();
        b = std::min(b, std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    return b;
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* dp;
    cudaMalloc(&dp, 4096);
    void* hp;
    cudaMallocHost(&hp, 1 << 20);
    empty_kernel<<<1, 32, 0, st>>>(nullptr);
    cudaStreamSynchronize(st);
    printf("empty launch+sync         %.1f us\n", best_us([&] {
               empty_kernel<<<1, 32, 0, st>>>(nullptr);
               cudaStreamSynchronize(st);
           }));
    printf("cluster(2) launch+sync    %.1f us\n", best_us([&] {
               cudaLaunchConfig_t cfg{};
               cfg.gridDim = dim3(2);
               cfg.blockDim = dim3(128);
               cfg.stream = st;
               cudaLaunchAttribute at[1];
               at[0].id = cudaLaunchAttributeClusterDimension;
               at[0].val.clusterDim.x = 2;
               at[0].val.clusterDim.y = 1;
               at[0].val.clusterDim.z = 1;
               cfg.attrs = at;
               cfg.numAttrs = 1;
               int* np = nullptr;
               void* args[] = {&np};
               cudaLaunchKernelExC(&cfg, (const void*)empty_kernel, args);
               cudaStreamSynchronize(st);
           }));
    printf("H2D 8KB pinned + sync     %.1f us\n", best_us([&] {
               cudaMemcpyAsync(dp, hp, 4096, cudaMemcpyHostToDevice, st);
               cudaStreamSynchronize(st);
           }));
    printf("memset+H2D+kern+D2H+sync  %.1f us\n", best_us([&] {
               cudaMemsetAsync(dp, 0, 16, st);
               cudaMemcpyAsync(dp, hp, 4096, cudaMemcpyHostToDevice, st);
               empty_kernel<<<1, 32, 0, st>>>(dp);
               cudaMemcpyAsync(hp, dp, 4096, cudaMemcpyDeviceToHost, st);
               cudaStreamSynchronize(st);
           }));
    const size_t N = 1024;
    std::vector<double> u(N), out(N);
    for (size_t i = 0; i < N; ++i) u[i] = std::sin(M_PI * double(i) / double(N - 1));
    u[N - 1] = 0.0;
    for (int k : {1, 1000}) {
        printf("heat_async_run k=%-5d     %.1f us\n", k, best_us([&] {
                   heat_async_run(u.data(), N, 0.25, HEAT_BC_DIRICHLET, 0.0, 0.0, N / 8, 2,
                                  HEAT_DELAY_UNIFORM, 0, 0.5, 1, size_t(k), size_t(k), out.data(),
                                  nullptr, nullptr, 0, nullptr);
               }, 100));
        printf("heat_sync_run  k=%-5d     %.1f us\n", k, best_us([&] {
                   heat_sync_run(u.data(), N, 0.25, HEAT_BC_DIRICHLET, 0.0, 0.0, size_t(k),
                                 size_t(k), out.data(), nullptr, nullptr, 0, nullptr);
               }, 100));
    }
    return 0;
}
