// FP64 peak microbenchmark for the roofline denominator (MEASURED_PEAKS.json has
// no FP64 entry).  Each thread runs 8 independent DFMA chains; the kernel runs
// long enough (~200 ms) for clocks to settle.  Reports DFMA-based FLOP/s
// (2 flops per DFMA) on cuda:0, best of 5 and median, plus the SM clock seen.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
    int dev = 0;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int threads = 256;
    const int blocks = prop.multiProcessorCount * 8;
    const int iters = argc > 1 ? atoi(argv[1]) : 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    std::vector<double> tf;
    for (int r = 0; r < 7; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 16 * double(iters) * threads * blocks;
        tf.push_back(flops / (ms * 1e-3) / 1e12);
    }
    std::sort(tf.begin(), tf.end());
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_mhz\": %.0f, \"fp64_dfma_tflops_best\": %.3f, "
           "\"fp64_dfma_tflops_median\": %.3f, \"err\": \"%s\"}\n",
           prop.name, prop.multiProcessorCount, clk_khz / 1e3, tf.back(), tf[tf.size() / 2],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
