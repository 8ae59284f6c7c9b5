// DFMA throughput against its operand pattern: does a 3-register-operand DFMA issue at
// the same rate as one whose multiplier/addend are shared (operand-reuse cache) or come
// from the constant bank?  16 independent chains per thread, 4 CTAs x 256 threads per SM.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double cc[2] = {0.9999999, 1e-9};
template <int MODE>
__global__ void __launch_bounds__(256, 4) k(double* out, int iters, double a, double b) {
    double x[16], y[16], z[16];
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 1e-9 + i; y[i] = 0.999999 + i * 1e-9; z[i] = 1e-9 * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) x[i] = fma(x[i], a, b);                   // shared multiplier and addend registers
            if (MODE == 1) x[i] = fma(x[i], y[i], z[i]);             // three distinct registers per instruction
            if (MODE == 2) x[i] = fma(x[i], cc[0], cc[1]);           // constant-bank operands
            if (MODE == 3) x[i] = fma(x[i], y[i], b);                // two distinct + shared
            if (MODE == 4) x[i] = fma(y[i], z[i], x[(i + 1) & 15]);  // 3 distinct, rotating chains
            if (MODE == 5) x[i] = x[i] + y[i];                       // DADD two registers
            if (MODE == 6) x[i] = fma(x[i], y[i], 1.0);              // two registers + immediate
        }
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += x[i] + y[i] + z[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(double* out, const char* name) {
    const int iters = 4096, grid = 148 * 4;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(a);
        k<MODE><<<grid, 256>>>(out, iters, 0.9999999, 1e-9);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double inst = double(grid) * 256 * iters * 16;
    printf("{\"mode\": \"%s\", \"ms\": %.4f, \"tflops\": %.2f, \"lanes_per_clk_per_sm\": %.2f}\n", name, best,
           2 * inst / best * 1e-9, inst / (best * 1e-3) / (148 * 1.965e9));
}
int main() {
    double* out; cudaMalloc(&out, 148 * 4 * 256 * 8);
    run<0>(out, "x=fma(x,a,b) shared regs");
    run<1>(out, "x=fma(x,y,z) three distinct regs");
    run<2>(out, "x=fma(x,c[0],c[1]) constant bank");
    run<3>(out, "x=fma(x,y,b) two distinct + shared");
    run<4>(out, "x=fma(y,z,x') three distinct rotating");
    run<5>(out, "x=x+y DADD");
    run<6>(out, "x=fma(x,y,1.0) two regs + imm");
    return 0;
}
