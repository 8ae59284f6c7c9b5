// Sweep of the symmetric pair loop's shape (csrc/sym.cuh sym_block): rows per lane R,
// step unroll U, warps per CTA W, CTAs per SM B, and the log variant (0 = fast_log as
// shipped, 2 = truncated index, see logvar_bench.cu).  Prints unordered pairs/s.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
using namespace vpg;

// trunc_log: common.cuh
// pricing only (wrong values): trunc_log with the I2F.F64 replaced by a register-pair build
__device__ __forceinline__ double trunc_log_noi2f(double x, uint32_t tab_lane) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    uint32_t idx, addr;
    asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi));
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
    const double m = __hiloint2double(mhi, lo);
    const double g = __hiloint2double((hi >> 11) + 0x40000000, lo);
    const double2 tc = lds_f64x2(addr);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}
// pricing only: the exponent word converted through FP32 (I2F.F32 + bit moves)
__device__ __forceinline__ double trunc_log_f32(double x, uint32_t tab_lane) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    uint32_t idx, addr;
    asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi));
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
    const double m = __hiloint2double(mhi, lo);
    // g = e 512 + i, |g| < 2^20: float exact; float bits -> double bits by integer ops
    const uint32_t fb = __float_as_uint(__int2float_rn((hi >> 11) - (0x3FF << 9)));
    uint32_t gh;
    asm("shr.b32 %0, %1, 3;" : "=r"(gh) : "r"(fb & 0x7FFFFFFFu));
    gh = (gh + 0x38000000u) | (fb & 0x80000000u);
    const double g = __hiloint2double(int(gh), 0);
    const double2 tc = lds_f64x2(addr);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}

template <int V, int R, int U, int W, int B>
__global__ void __launch_bounds__(W * 32, B)
pair_kernel(const double2* sxy, const double* q, int n, int tiles, const double2* gtab, double* out) {
    extern __shared__ double2 smp[];
    char* base = reinterpret_cast<char*>(smp);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kLogTableSize * kLogTableCopies; i += blockDim.x) smp[i] = gtab[i / kLogTableCopies];
    const uint32_t tab_lane = log_table_lane_addr(smp, lane & (kLogTableCopies - 1));
    double2* cxy = reinterpret_cast<double2*>(base + kLogTableBytes) + warp * 64;
    double* cq = reinterpret_cast<double*>(base + kLogTableBytes + W * 64 * 16) + warp * 64;
    __syncthreads();
    const int gw = blockIdx.x * W + warp;
    double rx[R], ry[R], rq[R], racc[R];
    for (int u = 0; u < R; ++u) {
        const int i = (gw * 32 * R + lane + 32 * u) % n;
        rx[u] = sxy[i].x; ry[u] = sxy[i].y; rq[u] = q[i]; racc[u] = 0.0;
    }
    double csum = 0.0;
    for (int ct = 0; ct < tiles; ++ct) {
        const int j = ((gw * 7 + ct) * 32 + lane) % n;
        const double2 p = sxy[j];
        const double qj = q[j];
        __syncwarp();
        cxy[lane] = p; cxy[lane + 32] = p; cq[lane] = qj; cq[lane + 32] = qj;
        __syncwarp();
        double cacc = 0.0;
#pragma unroll U
        for (int st = 0; st < 32; ++st) {
            const int c = lane + st;
            const double2 sp = cxy[c];
            const double qc = cq[c];
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const double dx = rx[u] - sp.x, dy = ry[u] - sp.y;
                const double r2 = fma(dy, dy, dx * dx);
                const double v = V == 0 ? fast_log(r2, tab_lane) : V == 2 ? trunc_log(r2, tab_lane) : V == 3 ? trunc_log_noi2f(r2, tab_lane) : trunc_log_f32(r2, tab_lane);
                racc[u] = fma(qc, v, racc[u]);
                cacc = fma(rq[u], v, cacc);
            }
            cacc = __shfl_sync(0xffffffffu, cacc, (lane + 1) & 31);
        }
        csum += cacc;
    }
    double s = csum;
    for (int u = 0; u < R; ++u) s += racc[u];
    out[size_t(gw) * 32 + lane] = s;
}

template <int V, int R, int U, int W, int B>
void run(const double2* sxy, const double* q, int n, const double2* tab, double* out) {
    const size_t smem = kLogTableBytes + W * 64 * 24;
    cudaFuncSetAttribute(pair_kernel<V, R, U, W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, pair_kernel<V, R, U, W, B>);
    const int grid = 148 * B;
    const int tiles = int(2048.0 * 4 / R * 16 / (W * B));  // equal pair count per config
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a);
        pair_kernel<V, R, U, W, B><<<grid, W * 32, smem>>>(sxy, q, n, tiles, tab, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double pairs = double(grid) * W * double(tiles) * 32 * 32 * R;
    cudaError_t e = cudaGetLastError();
    printf("{\"log\": %d, \"R\": %d, \"unroll\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, \"gpairs_s\": %.1f, \"err\": \"%s\"}\n",
           V, R, U, W, B, fa.numRegs, best, pairs / best * 1e-6, cudaGetErrorString(e));
}

// Stage-wise body: the R x U pairs of an unrolled trip advance together through the
// stages (differences, r^2, integer index work, table loads, reduction, polynomial,
// accumulation), written so that each stage is a run of independent instructions of one
// kind -- a test of whether runs of FP64 instructions from one warp use the FP64 pipe
// better than the finely interleaved schedule ptxas picks for the per-pair form.
template <int R, int U, int W, int B>
__global__ void __launch_bounds__(W * 32, B)
staged_kernel(const double2* sxy, const double* q, int n, int tiles, const double2* gtab, double* out) {
    extern __shared__ double2 smp[];
    char* base = reinterpret_cast<char*>(smp);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kLogTableSize * kLogTableCopies; i += blockDim.x) smp[i] = gtab[i / kLogTableCopies];
    const uint32_t tab_lane = log_table_lane_addr(smp, lane & (kLogTableCopies - 1));
    double2* cxy = reinterpret_cast<double2*>(base + kLogTableBytes) + warp * 64;
    double* cq = reinterpret_cast<double*>(base + kLogTableBytes + W * 64 * 16) + warp * 64;
    __syncthreads();
    const int gw = blockIdx.x * W + warp;
    double rx[R], ry[R], rq[R], racc[R];
    for (int u = 0; u < R; ++u) {
        const int i = (gw * 32 * R + lane + 32 * u) % n;
        rx[u] = sxy[i].x; ry[u] = sxy[i].y; rq[u] = q[i]; racc[u] = 0.0;
    }
    double csum = 0.0;
    constexpr int NP = R * U;
    for (int ct = 0; ct < tiles; ++ct) {
        const int j = ((gw * 7 + ct) * 32 + lane) % n;
        const double2 p = sxy[j];
        const double qj = q[j];
        __syncwarp();
        cxy[lane] = p; cxy[lane + 32] = p; cq[lane] = qj; cq[lane + 32] = qj;
        __syncwarp();
        double cacc = 0.0;
#pragma unroll 1
        for (int st = 0; st < 32; st += U) {
            double2 sp[U];
            double qc[U];
#pragma unroll
            for (int s2 = 0; s2 < U; ++s2) { sp[s2] = cxy[lane + st + s2]; qc[s2] = cq[lane + st + s2]; }
            double r2[NP];
#pragma unroll
            for (int s2 = 0; s2 < U; ++s2)
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    const double dx = rx[u] - sp[s2].x, dy = ry[u] - sp[s2].y;
                    r2[s2 * R + u] = fma(dy, dy, dx * dx);
                }
#pragma unroll
            for (int k = 0; k < NP; ++k) asm volatile("" : "+d"(r2[k]));
            double m[NP], g[NP];
            double2 tc[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const int hi = __double2hiint(r2[k]), lo = __double2loint(r2[k]);
                g[k] = __int2double_rn((hi >> 11) - (0x3FF << 9));
                int mhi;
                asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
                uint32_t idx, addr;
                asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi));
                asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
                m[k] = __hiloint2double(mhi, lo);
                tc[k] = lds_f64x2(addr);
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) asm volatile("" : "+d"(tc[k].x), "+d"(tc[k].y), "+d"(g[k]));
            double v[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const double r = fma(m[k], tc[k].x, -1.0);
                const double w = fma(g[k], c_flog[1], tc[k].y);
                double pp = fma(r, c_flog[2], c_flog[0]);
                pp = fma(r, pp, -0.5);
                pp = fma(r, pp, c_flog[3]);
                v[k] = fma(r, pp, w);
            }
#pragma unroll
            for (int s2 = 0; s2 < U; ++s2) {
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    racc[u] = fma(qc[s2], v[s2 * R + u], racc[u]);
                    cacc = fma(rq[u], v[s2 * R + u], cacc);
                }
                cacc = __shfl_sync(0xffffffffu, cacc, (lane + 1) & 31);
            }
        }
        csum += cacc;
    }
    double s = csum;
    for (int u = 0; u < R; ++u) s += racc[u];
    out[size_t(gw) * 32 + lane] = s;
}

template <int R, int U, int W, int B>
void run_staged(const double2* sxy, const double* q, int n, const double2* tab, double* out) {
    const size_t smem = kLogTableBytes + W * 64 * 24;
    cudaFuncSetAttribute(staged_kernel<R, U, W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, staged_kernel<R, U, W, B>);
    const int grid = 148 * B;
    const int tiles = int(2048.0 * 4 / R * 16 / (W * B));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(a);
        staged_kernel<R, U, W, B><<<grid, W * 32, smem>>>(sxy, q, n, tiles, tab, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double pairs = double(grid) * W * double(tiles) * 32 * 32 * R;
    printf("{\"staged\": 1, \"R\": %d, \"unroll\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, \"gpairs_s\": %.1f, \"err\": \"%s\"}\n",
           R, U, W, B, fa.numRegs, best, pairs / best * 1e-6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 1 << 16;
    std::vector<double2> xy(n);
    std::vector<double> q(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
        xy[i] = make_double2(rand() / double(RAND_MAX), rand() / double(RAND_MAX));
        q[i] = rand() / double(RAND_MAX) - 0.5;
    }
    std::vector<double2> t0(kLogTableSize), t2(kLogTableSize);
    for (int i = 0; i < kLogTableSize; ++i) {
        long double c = 1.0L + (long double)i / (kLogTableSize - 1);
        double inv = double(1.0L / c);
        t0[i] = make_double2(inv, double(-logl((long double)inv) - (long double)i * (long double)kLn2Over512));
        c = 1.0L + ((long double)i + 0.5L) / (kLogTableSize - 1);
        inv = double(1.0L / c);
        t2[i] = make_double2(inv, double(-logl((long double)inv) - (long double)i * (long double)kLn2Over512));
    }
    double2 *dxy, *dt0, *dt2; double *dq, *dout;
    cudaMalloc(&dxy, n * 16); cudaMalloc(&dq, n * 8); cudaMalloc(&dt0, t0.size() * 16); cudaMalloc(&dt2, t2.size() * 16);
    cudaMalloc(&dout, size_t(148) * 4 * 32 * 32 * 8 * 2);
    cudaMemcpy(dxy, xy.data(), n * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dt0, t0.data(), t0.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dt2, t2.data(), t2.size() * 16, cudaMemcpyHostToDevice);
#define RUN(V, R, U, W, B) run<V, R, U, W, B>(dxy, dq, n, V == 0 ? dt0 : dt2, dout)
    RUN(2, 4, 4, 12, 1);
    RUN(2, 4, 4, 8, 2);
    run_staged<4, 2, 12, 1>(dxy, dq, n, dt2, dout);
    run_staged<4, 4, 12, 1>(dxy, dq, n, dt2, dout);
    run_staged<4, 2, 8, 2>(dxy, dq, n, dt2, dout);
    run_staged<4, 2, 16, 1>(dxy, dq, n, dt2, dout);
    run_staged<8, 1, 12, 1>(dxy, dq, n, dt2, dout);
    run_staged<8, 2, 8, 1>(dxy, dq, n, dt2, dout);
    run_staged<2, 4, 8, 2>(dxy, dq, n, dt2, dout);
    run_staged<2, 4, 8, 3>(dxy, dq, n, dt2, dout);
    cudaDeviceSynchronize();
    return 0;
}
