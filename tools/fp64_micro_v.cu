// fp64_micro_v.cu -- the FTCS step code (warp_steps_pipelined) at V = 32 / 48
// / 64 points per lane with no memory traffic: does a wider lane (narrower
// relative halo) keep the FP64 pipe as busy with fewer resident warps?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/fp64_micro_v.cu
#include <cstdio>

#include "../paper_1510_08982_b200/csrc/sync_tb.cuh"

using namespace hb;

template <int V, int MINB>
__global__ void __launch_bounds__(128, MINB) step_ceiling(double* out, int steps, double r, double c) {
    double u[V];
#pragma unroll
    for (int i = 0; i < V; ++i) u[i] = (threadIdx.x * V + i) * 1e-6;
    warp_steps_pipelined<double, V>(u, r, c, steps);
    double acc = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) acc += u[i];
    if (acc == 12345.0) out[0] = acc;
}

template <int V, int MINB>
void run(int sms, double* out) {
    const int steps = 2000, blocks = sms * MINB, threads = 128;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) step_ceiling<V, MINB><<<blocks, threads>>>(out, steps, 0.4, 0.2);
    cudaEventRecord(e0);
    step_ceiling<V, MINB><<<blocks, threads>>>(out, steps, 0.4, 0.2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double upd = double(blocks) * threads * V * steps;  // all lanes
    const double exact = double(32 * V - 64) / (32 * V);        // 32-point halo per side
    printf("V=%2d CTAs/SM=%d: %.3f T DP-ops/s, %.0f GLUPS useful (exact fraction %.4f)\n", V, MINB,
           4 * upd / (ms * 1e-3) / 1e12, upd * exact / (ms * 1e-3) / 1e9, exact);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    for (int i = 0; i < 3; ++i) run<32, 3>(sms, out);  // clocks up
    run<32, 3>(sms, out);
    run<32, 2>(sms, out);
    run<48, 3>(sms, out);
    run<48, 2>(sms, out);
    run<64, 2>(sms, out);
    run<64, 3>(sms, out);
    run<64, 1>(sms, out);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
