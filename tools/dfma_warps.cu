// DFMA throughput against resident warps per scheduler and independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
    double x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(double* out, int warps_per_sm) {
    const int iters = 32768 / CH * 4, grid = 148;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k<CH><<<grid, warps_per_sm * 32>>>(out, iters, 0.9999999, 1e-9);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double inst = double(grid) * warps_per_sm * 32 * iters * CH;
    printf("{\"warps_per_scheduler\": %.2f, \"chains\": %d, \"lanes_per_clk_per_sm\": %.2f, \"cycles_per_dfma_per_scheduler\": %.2f}\n",
           warps_per_sm / 4.0, CH, inst / (best * 1e-3) / (148 * 1.965e9), (best * 1e-3 * 1.965e9) / (double(iters) * CH * warps_per_sm / 4.0));
}
int main() {
    double* out; cudaMalloc(&out, 148 * 1024 * 8);
    for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(out, w); run<2>(out, w); run<4>(out, w); run<8>(out, w); run<16>(out, w); }
    return 0;
}
