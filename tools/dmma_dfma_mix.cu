// Do DMMA (FP64 tensor) and DFMA (FP64 CUDA core) share one pipe on B200?
// One kernel, 8 warps per CTA, 4 CTAs per SM: warps with (warp % 2 == 0)
// run DMMA chains, the others DFMA chains (mode 2); mode 0 = all DMMA, mode 1
// = all DFMA.  If the mixed run reaches ~the sum of the two half-rates, the
// pipes are separate and a DMMA kernel (M2L) could share SMs with a DFMA
// kernel (near field).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ void dmma_work(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    double c[8][2];
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dfma_work(double* out, int iters) {
    double x[16];
    for (int t = 0; t < 16; ++t) x[t] = 1.0 + t * 1e-7 + threadIdx.x * 1e-9;
    const double m = 0.9999999, a = 1e-9;
    for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
        for (int t = 0; t < 16; ++t) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[t]) : "d"(m), "d"(a));
    }
    double s = 0;
    for (int t = 0; t < 16; ++t) s += x[t];
    if (s == 1.2345) out[0] = s;
}

__global__ void mix(double* out, int iters, int mode, unsigned long long* cyc) {
    const int warp = threadIdx.x >> 5;
    const bool mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
    const long long t0 = clock64();
    if (mma) dmma_work(out, iters);
    else dfma_work(out, iters);
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicAdd(&cyc[mma ? 0 : 1], (unsigned long long)(t1 - t0));
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    double* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 16);
    const int threads = 256, blocks = prop.multiProcessorCount * 4, iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"all_dmma", "all_dfma", "half_half"};
    printf("[");
    for (int mode = 0; mode < 3; ++mode) {
        for (int w = 0; w < 2; ++w) mix<<<blocks, threads>>>(out, iters, mode, cyc);
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            mix<<<blocks, threads>>>(out, iters, mode, cyc);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        // per warp: DMMA 8 * iters * 512 flop; DFMA 16 * 8 * iters * 64 flop (32 lanes x 2)
        const double warps = double(threads / 32) * blocks;
        const double wm = mode == 0 ? warps : mode == 1 ? 0 : warps / 2;
        const double wf = warps - wm;
        const double fm = wm * 8.0 * iters * 512.0, ff = wf * 16.0 * 8 * iters * 64.0;
        printf("%s{\"mode\": \"%s\", \"ms\": %.4f, \"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"total_tflops\": %.3f}",
               mode ? ", " : "", names[mode], best, fm / (best * 1e-3) / 1e12, ff / (best * 1e-3) / 1e12,
               (fm + ff) / (best * 1e-3) / 1e12);
    }
    printf("]\n");
    return 0;
}
