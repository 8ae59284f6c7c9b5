// Dependent-chain latency of DFMA / DADD / LDS.64 on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
    double x = threadIdx.x * 1e-9;
    __shared__ double sm[256];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, a, b);
    }
    long long t1 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) idx = int(sm[idx & 255]) ;
    }
    long long t2 = clock64();
    double y = x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) y = y * a;
    }
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
    out[threadIdx.x] = x + idx + y;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64);
    int iters = 1000;
    chain<<<1, 32>>>(o, c, iters, 0.9999, 1e-7);
    chain<<<1, 32>>>(o, c, iters, 0.9999, 1e-7);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("{\"dfma_latency_cyc\": %.2f, \"lds_latency_cyc\": %.2f, \"dmul_latency_cyc\": %.2f}\n",
           h[0] / (16.0 * iters), h[1] / (16.0 * iters), h[2] / (16.0 * iters));
    return 0;
}
