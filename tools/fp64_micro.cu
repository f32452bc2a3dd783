// fp64_micro.cu -- measures (1) the B200's sustained DMUL/DADD issue rate and
// (2) the FTCS step code (K1's warp_step / warp_steps_pipelined) with no
// memory traffic, i.e. the compute ceiling of the sync/async kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. tools/fp64_micro.cu
#include <cstdio>

#include "../paper_1510_08982_b200/csrc/sync_tb.cuh"

using namespace hb;

// 8 independent DMUL->DADD chains per thread (no FMA): 2 DP ops per link.
__global__ void dp_peak(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __dadd_rn(__dmul_rn(x[j], a), b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.0) out[0] = s;
}

template <int MODE>
__global__ void __launch_bounds__(128, 3) step_ceiling(double* out, int steps, double r, double c) {
    double u[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) u[i] = (threadIdx.x * 32 + i) * 1e-6;
    if (MODE == 0) {
        for (int s = 0; s < steps; ++s) warp_step<double, 32>(u, r, c);
    } else {
        warp_steps_pipelined<double, 32>(u, r, c, steps);
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += u[i];
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // warm up clocks
    for (int i = 0; i < 20; ++i) dp_peak<<<sms * 8, 256>>>(out, 20000, 0.999, 1e-3);
    cudaDeviceSynchronize();
    {
        const int iters = 20000, blocks = sms * 8, threads = 256;
        cudaEventRecord(e0);
        dp_peak<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * 8 * iters * double(blocks) * threads;
        printf("dp_peak: %.3f T DP-ops/s (%.1f ops/clk/SM at 1.965 GHz)\n", ops / (ms * 1e-3) / 1e12,
               ops / (ms * 1e-3) / sms / 1.965e9);
    }
    for (int mode = 0; mode < 2; ++mode) {
        const int steps = 2000, blocks = sms * 3, threads = 128;
        for (int w = 0; w < 3; ++w) {
            if (mode == 0) step_ceiling<0><<<blocks, threads>>>(out, steps, 0.4, 0.2);
            else step_ceiling<1><<<blocks, threads>>>(out, steps, 0.4, 0.2);
        }
        cudaEventRecord(e0);
        if (mode == 0) step_ceiling<0><<<blocks, threads>>>(out, steps, 0.4, 0.2);
        else step_ceiling<1><<<blocks, threads>>>(out, steps, 0.4, 0.2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double upd = double(blocks) * threads * 32 * steps;  // incl. halo lanes
        printf("step_ceiling %s: %.1f G point-updates/s (all lanes), %.1f GLUPS useful (30/32), "
               "%.3f T DP-ops/s\n", mode ? "pipelined" : "warp_step", upd / (ms * 1e-3) / 1e9,
               upd * 30 / 32 / (ms * 1e-3) / 1e9, 4 * upd / (ms * 1e-3) / 1e12);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
