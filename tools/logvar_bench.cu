// Micro-benchmark of the symmetric near-field pair loop (csrc/sym.cuh sym_block,
// R = 4, off-diagonal tiles) with variants of ln r^2:
//   v0  fast_log as shipped: 16-byte table entries (RN(1/c), w), 8 copies, LDS.128
//   v1  reciprocal index: j = round(1024 / m) from MUFU.RCP, 1/c = j / 1024 built by
//       integer ops (exact), 8-byte entries w_j = -ln(j / 1024), 16 copies, LDS.64
//   h0 / h1  the same with half-warp column broadcast (lanes l, l + 16 share a
//       column: column loads halve, one extra shuffle + add per 16 steps)
// Prints pairs/s per variant and the max |error| of each log against logl.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2203_05933_b200/csrc -I include
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace vpg;

constexpr int kWarps = 8;
constexpr int kRcpCopies = 16;
constexpr int kRcpSize = 513;
constexpr float kMagic = 8388608.0f;  // 2^23
static __constant__ double c_rlog[4] = {0.3333335717519124, 0.69314718055994530942, -0.25, 0.99999999999994315658};

__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// tab_lane: smem byte address of this lane's copy of entry 0, minus
// (0x4B000000 + 512) * 128 (the magic float's bits index the table directly).
__device__ __forceinline__ double rcp_log(double x, uint32_t tab_lane) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double ed = __int2double_rn((hi >> 20) - 1023);
    int mf, mhi;
    asm("lop3.b32 %0, %1, 0x007FFFF8, %2, 0xEA;" : "=r"(mf) : "r"(hi << 3), "r"(0x3F800000));
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__int_as_float(mf)));
    const uint32_t tb = __float_as_uint(fmaf(y, 1024.0f, kMagic));  // 0x4B000000 + j
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3F500000));  // m / 1024
    const double ms = __hiloint2double(mhi, lo);
    const double jd = __hiloint2double(int(tb * 2048u + 0x40700000u), 0);
    const double wj = lds_f64(tb * uint32_t(8 * kRcpCopies) + tab_lane);
    const double r = fma(ms, jd, -1.0);
    const double w = fma(ed, c_rlog[1], wj);
    double p = fma(r, c_rlog[2], c_rlog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_rlog[3]);
    return fma(r, p, w);
}


// v2: truncated index (centres 1 + (i + 1/2)/512): g = (hi >> 11) - bias is the
// exponent-and-index word without the rounding add, the mantissa word indexes the table.
__device__ __forceinline__ double trunc_log(double x, uint32_t tab_lane) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double g = __int2double_rn((hi >> 11) - (0x3FF << 9));
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    uint32_t idx, addr;
    asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi));
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
    const double m = __hiloint2double(mhi, lo);
    const double2 tc = lds_f64x2(addr);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}
// pricing only (wrong values): v2 without the I2F.F64
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
// pricing only: v0 plus two dependent dummy integer instructions per pair
__device__ __forceinline__ double fast_log_plus2(double x, uint32_t tab_lane) {
    int hi = __double2hiint(x);
    asm volatile("xor.b32 %0, %0, 0x1;" : "+r"(hi));
    asm volatile("xor.b32 %0, %0, 0x1;" : "+r"(hi));
    return fast_log(__hiloint2double(hi, __double2loint(x)), tab_lane);
}

struct V0 {
    static constexpr int kTabBytes = kLogTableBytes;
    static constexpr bool kRcp = false;
    __device__ static double f(double r2, uint32_t t) { return fast_log(r2, t); }
};
struct V2 {
    static constexpr int kTabBytes = kLogTableBytes;
    static constexpr bool kRcp = false;
    static constexpr bool kTrunc = true;
    __device__ static double f(double r2, uint32_t t) { return trunc_log(r2, t); }
};
struct V2N {
    static constexpr int kTabBytes = kLogTableBytes;
    static constexpr bool kRcp = false;
    static constexpr bool kTrunc = true;
    __device__ static double f(double r2, uint32_t t) { return trunc_log_noi2f(r2, t); }
};
struct V0P {
    static constexpr int kTabBytes = kLogTableBytes;
    static constexpr bool kRcp = false;
    __device__ static double f(double r2, uint32_t t) { return fast_log_plus2(r2, t); }
};
struct V1 {
    static constexpr int kTabBytes = kRcpSize * kRcpCopies * 8;
    static constexpr bool kRcp = true;
    __device__ static double f(double r2, uint32_t t) { return rcp_log(r2, t); }
};

template <class V, bool kHalf>
__global__ void __launch_bounds__(kWarps * 32, 2)
pair_kernel(const double2* sxy, const double* q, int n, int tiles, const double2* gtab0, const double* gtab1,
            double* out) {
    extern __shared__ double2 smp[];
    char* base = reinterpret_cast<char*>(smp);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t tab_lane;
    if (!V::kRcp) {
        for (int i = threadIdx.x; i < kLogTableSize * kLogTableCopies; i += blockDim.x) smp[i] = gtab0[i / kLogTableCopies];
        tab_lane = log_table_lane_addr(smp, lane & (kLogTableCopies - 1));
    } else {
        double* t = reinterpret_cast<double*>(base);
        for (int i = threadIdx.x; i < kRcpSize * kRcpCopies; i += blockDim.x) t[i] = gtab1[i / kRcpCopies];
        tab_lane = uint32_t(__cvta_generic_to_shared(t)) + uint32_t(lane & (kRcpCopies - 1)) * 8u -
                   (0x4B000000u + 512u) * uint32_t(8 * kRcpCopies);
    }
    double2* cxy = reinterpret_cast<double2*>(base + V::kTabBytes) + warp * 64;
    double* cq = reinterpret_cast<double*>(base + V::kTabBytes + kWarps * 64 * 16) + warp * 64;
    __syncthreads();
    constexpr int R = 4;
    const int gw = blockIdx.x * kWarps + warp;
    double rx[R], ry[R], rq[R], racc[R];
    for (int u = 0; u < R; ++u) {
        const int i = (gw * 128 + lane + 32 * u) % n;
        rx[u] = sxy[i].x;
        ry[u] = sxy[i].y;
        rq[u] = q[i];
        racc[u] = 0.0;
    }
    double csum = 0.0;
    for (int ct = 0; ct < tiles; ++ct) {
        const int j = ((gw * 7 + ct) * 32 + lane) % n;
        const double2 p = sxy[j];
        const double qj = q[j];
        __syncwarp();
        if (!kHalf) {
            cxy[lane] = p; cxy[lane + 32] = p; cq[lane] = qj; cq[lane + 32] = qj;
        } else {  // [0..15][0..15][16..31][16..31]
            const int s = (lane & 15) + (lane & 16) * 2;
            cxy[s] = p; cxy[s + 16] = p; cq[s] = qj; cq[s + 16] = qj;
        }
        __syncwarp();
        if (!kHalf) {
            double cacc = 0.0;
#pragma unroll 2
            for (int st = 0; st < 32; ++st) {
                const int c = lane + st;
                const double2 sp = cxy[c];
                const double qc = cq[c];
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    const double dx = rx[u] - sp.x, dy = ry[u] - sp.y;
                    const double r2 = fma(dy, dy, dx * dx);
                    const double v = V::f(r2, tab_lane);
                    racc[u] = fma(qc, v, racc[u]);
                    cacc = fma(rq[u], v, cacc);
                }
                cacc = __shfl_sync(0xffffffffu, cacc, (lane + 1) & 31);
            }
            csum += cacc;
        } else {
            for (int blk = 0; blk < 2; ++blk) {
                double cacc = 0.0;
                const int b0 = blk * 32 + (lane & 15);
#pragma unroll 2
                for (int st = 0; st < 16; ++st) {
                    const double2 sp = cxy[b0 + st];
                    const double qc = cq[b0 + st];
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const double dx = rx[u] - sp.x, dy = ry[u] - sp.y;
                        const double r2 = fma(dy, dy, dx * dx);
                        const double v = V::f(r2, tab_lane);
                        racc[u] = fma(qc, v, racc[u]);
                        cacc = fma(rq[u], v, cacc);
                    }
                    cacc = __shfl_sync(0xffffffffu, cacc, ((lane + 1) & 15) | (lane & 16));
                }
                cacc += __shfl_xor_sync(0xffffffffu, cacc, 16);
                csum += cacc;
            }
        }
    }
    double s = csum;
    for (int u = 0; u < R; ++u) s += racc[u];
    out[size_t(gw) * 32 + lane] = s;
}

template <class V>
__global__ void log_check(const double* x, int n, const double2* gtab0, const double* gtab1, double* y) {
    extern __shared__ double2 smp[];
    const int lane = threadIdx.x & 31;
    uint32_t tab_lane;
    if (!V::kRcp) {
        for (int i = threadIdx.x; i < kLogTableSize * kLogTableCopies; i += blockDim.x) smp[i] = gtab0[i / kLogTableCopies];
        tab_lane = log_table_lane_addr(smp, lane & (kLogTableCopies - 1));
    } else {
        double* t = reinterpret_cast<double*>(smp);
        for (int i = threadIdx.x; i < kRcpSize * kRcpCopies; i += blockDim.x) t[i] = gtab1[i / kRcpCopies];
        tab_lane = uint32_t(__cvta_generic_to_shared(t)) + uint32_t(lane & (kRcpCopies - 1)) * 8u -
                   (0x4B000000u + 512u) * uint32_t(8 * kRcpCopies);
    }
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = V::f(x[i], tab_lane);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <class V, bool kHalf>
double run(const double2* sxy, const double* q, int n, int tiles, const double2* t0, const double* t1, double* out,
           int grid, double* chk) {
    const size_t smem = V::kTabBytes + kWarps * 64 * 24;
    cudaFuncSetAttribute(pair_kernel<V, kHalf>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        pair_kernel<V, kHalf><<<grid, kWarps * 32, smem>>>(sxy, q, n, tiles, t0, t1, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    std::vector<double> h(size_t(grid) * kWarps * 32);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (double v : h) s += v;
    *chk = s;
    return best;
}

int main() {
    const int n = 1 << 16, tiles = 2048, grid = 296;
    std::vector<double2> xy(n);
    std::vector<double> q(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
        xy[i] = make_double2(rand() / double(RAND_MAX), rand() / double(RAND_MAX));
        q[i] = rand() / double(RAND_MAX) - 0.5;
    }
    std::vector<double2> t0(kLogTableSize);
    for (int i = 0; i < kLogTableSize; ++i) {
        const long double c = 1.0L + (long double)i / (kLogTableSize - 1);
        const double inv = double(1.0L / c);
        t0[i] = make_double2(inv, double(-logl((long double)inv) - (long double)i * (long double)kLn2Over512));
    }
    std::vector<double2> t2(kLogTableSize);
    for (int i = 0; i < kLogTableSize; ++i) {
        const long double c = 1.0L + ((long double)i + 0.5L) / (kLogTableSize - 1);
        const double inv = double(1.0L / c);
        t2[i] = make_double2(inv, double(-logl((long double)inv) - (long double)i * (long double)kLn2Over512));
    }
    std::vector<double> t1(kRcpSize);
    for (int i = 0; i < kRcpSize; ++i) t1[i] = double(-logl((long double)(512 + i) / 1024.0L));
    double2 *dxy, *dt0, *dt2;
    double *dq, *dt1, *dout;
    CK(cudaMalloc(&dxy, n * 16)); CK(cudaMalloc(&dq, n * 8)); CK(cudaMalloc(&dt0, t0.size() * 16));
    CK(cudaMalloc(&dt1, t1.size() * 8)); CK(cudaMalloc(&dout, size_t(grid) * kWarps * 32 * 8));
    CK(cudaMemcpy(dxy, xy.data(), n * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dq, q.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt0, t0.data(), t0.size() * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt1, t1.data(), t1.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dt2, t2.size() * 16));
    CK(cudaMemcpy(dt2, t2.data(), t2.size() * 16, cudaMemcpyHostToDevice));
    // accuracy
    const int m = 1 << 20;
    std::vector<double> x(m), y0(m), y1(m);
    for (int i = 0; i < m; ++i) {
        const double e = -60.0 + 70.0 * (rand() / double(RAND_MAX));
        x[i] = exp2(e) * (1.0 + rand() / double(RAND_MAX));
        if (i < 4096) x[i] = 1.0 + (i - 2048) * 1e-7;           // around 1
        else if (i < 8192) x[i] = ldexp(1.0, (i & 63) - 40);    // powers of two
        else if (i < 16384) x[i] = (512.5 + (i & 511)) / 1024.0 * (1.0 + ((i >> 9) - 8) * 1e-9);  // index boundaries of v0
        else if (i < 32768) x[i] = 1024.0 / (512.5 + (i & 511)) * (1.0 + (((i >> 9) & 15) - 8) * 1e-8);  // of v1
    }
    double *dx, *dy;
    CK(cudaMalloc(&dx, m * 8)); CK(cudaMalloc(&dy, m * 8));
    CK(cudaMemcpy(dx, x.data(), m * 8, cudaMemcpyHostToDevice));
    cudaFuncSetAttribute(log_check<V0>, cudaFuncAttributeMaxDynamicSharedMemorySize, V0::kTabBytes);
    cudaFuncSetAttribute(log_check<V1>, cudaFuncAttributeMaxDynamicSharedMemorySize, V1::kTabBytes);
    log_check<V0><<<148, 256, V0::kTabBytes>>>(dx, m, dt0, dt1, dy);
    CK(cudaMemcpy(y0.data(), dy, m * 8, cudaMemcpyDeviceToHost));
    log_check<V1><<<148, 256, V1::kTabBytes>>>(dx, m, dt0, dt1, dy);
    CK(cudaMemcpy(y1.data(), dy, m * 8, cudaMemcpyDeviceToHost));
    std::vector<double> y2(m);
    cudaFuncSetAttribute(log_check<V2>, cudaFuncAttributeMaxDynamicSharedMemorySize, V2::kTabBytes);
    log_check<V2><<<148, 256, V2::kTabBytes>>>(dx, m, dt2, dt1, dy);
    CK(cudaMemcpy(y2.data(), dy, m * 8, cudaMemcpyDeviceToHost));
    {
        double e2 = 0, u2 = 0;
        for (int i = 0; i < m; ++i) {
            const long double t = logl((long double)x[i]);
            const double ulp = std::fmax(std::fabs(double(t)), 1.0) * 2.220446049250313e-16;
            const double a2 = std::fabs(double((long double)y2[i] - t));
            e2 = std::fmax(e2, a2); u2 = std::fmax(u2, a2 / ulp);
        }
        printf("{\"log_check_v2\": {\"max_abs\": %.3e, \"max_rel1\": %.3f, \"ln1\": %.3e}}\n", e2, u2, y2[2048]);
    }
    double e0 = 0, e1 = 0, u0 = 0, u1 = 0;
    for (int i = 0; i < m; ++i) {
        const long double t = logl((long double)x[i]);
        const double ulp = std::fmax(std::fabs(double(t)), 1.0) * 2.220446049250313e-16;
        const double a0 = std::fabs(double((long double)y0[i] - t)), a1 = std::fabs(double((long double)y1[i] - t));
        e0 = std::fmax(e0, a0); e1 = std::fmax(e1, a1);
        u0 = std::fmax(u0, a0 / ulp); u1 = std::fmax(u1, a1 / ulp);
    }
    printf("{\"log_check\": {\"v0_max_abs\": %.3e, \"v0_max_rel1\": %.3f, \"v1_max_abs\": %.3e, \"v1_max_rel1\": %.3f, \"ln1_v1\": %.3e}}\n",
           e0, u0, e1, u1, y1[2048]);
    const double pairs = double(grid) * kWarps * double(tiles) * 32 * 128;
    double c;
    double ms;
    ms = run<V0, false>(dxy, dq, n, tiles, dt0, dt1, dout, grid, &c);
    printf("{\"variant\": \"v0\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V1, false>(dxy, dq, n, tiles, dt0, dt1, dout, grid, &c);
    printf("{\"variant\": \"v1\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V2, false>(dxy, dq, n, tiles, dt2, dt1, dout, grid, &c);
    printf("{\"variant\": \"v2_trunc\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V2N, false>(dxy, dq, n, tiles, dt2, dt1, dout, grid, &c);
    printf("{\"variant\": \"v2_noi2f(pricing)\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V0P, false>(dxy, dq, n, tiles, dt0, dt1, dout, grid, &c);
    printf("{\"variant\": \"v0_plus2alu(pricing)\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V0, true>(dxy, dq, n, tiles, dt0, dt1, dout, grid, &c);
    printf("{\"variant\": \"h0\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    ms = run<V1, true>(dxy, dq, n, tiles, dt0, dt1, dout, grid, &c);
    printf("{\"variant\": \"h1\", \"ms\": %.4f, \"gpairs_s\": %.1f, \"chk\": %.15e}\n", ms, pairs / ms * 1e-6, c);
    CK(cudaDeviceSynchronize());
    return 0;
}
