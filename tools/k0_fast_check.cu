// Checks k0_fast (quarter-octave fits, degree-12 series) against k0_dev
// (the reference construction, kernel.cpp:17-172) on 2M points in
// (1e-3, 745]: prints the max relative difference.
#include <cstdio>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_2203_05933_b200/csrc/k0.cuh"

__global__ void cmp(const double* x, int n, const double* tab, const double* ftab, double* rel) {
    __shared__ double ft[vpg::kK0FastIntervals * vpg::kK0FastStride];
    for (int i = threadIdx.x; i < vpg::kK0FastIntervals * vpg::kK0FastStride; i += blockDim.x) ft[i] = ftab[i];
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = vpg::k0_dev(x[i], tab), b = vpg::k0_fast(x[i], ft);
    rel[i] = a == 0.0 ? (b == 0.0 ? 0.0 : 1.0) : fabs(a - b) / fabs(a);
}

int main() {
    const int n = 2 << 20;
    std::vector<double> x(n), tab(vpg::kK0Intervals * vpg::kK0Coeffs), ft(vpg::kK0FastIntervals * vpg::kK0FastStride);
    for (int i = 0; i < n; ++i) x[i] = 1e-3 * std::pow(745.0 / 1e-3, (i + 0.5) / n);
    vpg::k0_fit_host(tab.data());
    vpg::k0_fit_fast_host(ft.data());
    double *dx, *dt, *df, *dr;
    cudaMalloc(&dx, 8 * n); cudaMalloc(&dr, 8 * n);
    cudaMalloc(&dt, 8 * tab.size()); cudaMalloc(&df, 8 * ft.size());
    cudaMemcpy(dx, x.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, tab.data(), 8 * tab.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(df, ft.data(), 8 * ft.size(), cudaMemcpyHostToDevice);
    cmp<<<(n + 255) / 256, 256>>>(dx, n, dt, df, dr);
    std::vector<double> r(n);
    cudaMemcpy(r.data(), dr, 8 * n, cudaMemcpyDeviceToHost);
    // x > 700: K0 ~ 1e-305 and below, subnormal -- no accuracy to compare
    double mx = 0, mx_small = 0; int at = 0;
    for (int i = 0; i < n; ++i) {
        if (x[i] > 700.0) continue;
        if (x[i] <= 2 && r[i] > mx_small) mx_small = r[i];
        if (r[i] > mx) { mx = r[i]; at = i; }
    }
    printf("{\"max_rel_x_le_700\": %.3e, \"at_x\": %.6g, \"max_rel_x_le_2\": %.3e, \"err\": \"%s\"}\n", mx, x[at],
           mx_small, cudaGetErrorString(cudaGetLastError()));
    return mx < 4e-15 ? 0 : 1;
}
