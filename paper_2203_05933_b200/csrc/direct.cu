// direct.cu -- all-pairs sums on the device: the plan's pairwise mode
// (summation.cpp:619-635, r^2 == 0 skipped) and direct_sum
// (summation.cpp:501-540, coincidence reported as the smallest (i, j)).
//
// CTA of 128 threads, TPT targets per thread; 128-source tiles staged in
// smem and read as warp broadcasts.  When the target count alone cannot
// fill the GPU, the sources are split over gridDim.y slices whose partial
// sums land in a scratch array and are reduced in slice order by a second
// kernel -- deterministic, no atomics on values.
#include <algorithm>

#include "k0.cuh"
#include "p2p.cuh"
#include "plan.cuh"

namespace vpg {
namespace {

constexpr int kDirThreads = 128;
constexpr int kDirTPT = 2;

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

template <int kFamily, bool kSkip>
__global__ void __launch_bounds__(kDirThreads)
allpairs_kernel(const double2* src, const double* q, int64_t ns,
                const double2* tgt, int64_t nt, int64_t slice, double lambda,
                const double2* gtab, const double* k0tab, double* out,
                double* partial, unsigned long long* clash) {
    extern __shared__ double2 smd[];
    double2* tab = smd;
    double2* tile = smd + (kFamily == VPG_LAPLACE ? kLogTableSize * kLogTableCopies : 0);
    if (kFamily == VPG_LAPLACE) log_table_to_smem(tab, gtab);
    const uint32_t tab_lane = log_table_lane_addr(tab, threadIdx.x & (kLogTableCopies - 1));
    const int64_t j0 = int64_t(blockIdx.y) * slice;
    const int64_t j1 = min(ns, j0 + slice);

    double tx[kDirTPT], ty[kDirTPT];
    LapAcc acc[kDirTPT];
    double kacc[kDirTPT];
    int64_t ti[kDirTPT];
#pragma unroll
    for (int u = 0; u < kDirTPT; ++u) {
        ti[u] = (int64_t(blockIdx.x) * kDirTPT + u) * kDirThreads + threadIdx.x;
        const double2 t = tgt[min(ti[u], nt - 1)];
        tx[u] = t.x;
        ty[u] = t.y;
        kacc[u] = 0.0;
    }
    for (int64_t base = j0; base < j1; base += kDirThreads) {
        const int cnt = int(min(int64_t(kDirThreads), j1 - base));
        __syncthreads();
        if (threadIdx.x < cnt) {
            tile[2 * threadIdx.x] = src[base + threadIdx.x];
            tile[2 * threadIdx.x + 1] = make_double2(q[base + threadIdx.x], 0.0);
        }
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
            const double2 sp = tile[2 * j];
            const double qj = tile[2 * j + 1].x;
#pragma unroll
            for (int u = 0; u < kDirTPT; ++u) {
                if (!kSkip) {
                    const double dx = tx[u] - sp.x, dy = ty[u] - sp.y;
                    if (fma(dy, dy, dx * dx) == 0.0 && ti[u] < nt) {
                        const unsigned long long key =
                            (static_cast<unsigned long long>(ti[u]) << 32) |
                            static_cast<unsigned long long>(base + j);
                        atomicMin(clash, key);
                    }
                }
                if (kFamily == VPG_LAPLACE)
                    lap_pair(tx[u], ty[u], sp.x, sp.y, qj, tab_lane, acc[u]);
                else
                    kacc[u] += k0_pair(tx[u], ty[u], sp.x, sp.y, qj, lambda, k0tab);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kDirTPT; ++u) {
        if (ti[u] >= nt) continue;
        const double v = kFamily == VPG_LAPLACE ? -kInv4Pi * lap_total(acc[u])
                                                : kInv2Pi * kacc[u];
        if (gridDim.y == 1)
            out[ti[u]] = v;
        else
            partial[int64_t(blockIdx.y) * nt + ti[u]] = v;
    }
}

__global__ void reduce_slices(const double* partial, int nslice, int64_t nt, double* out) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= nt) return;
    double s = 0.0;
    for (int k = 0; k < nslice; ++k) s += partial[int64_t(k) * nt + i];
    out[i] = s;
}

int sm_count() {
    int dev = 0, count = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    return count;
}

template <int kFamily, bool kSkip>
void launch_allpairs(const double2* src, const double* q, int64_t ns,
                     const double2* tgt, int64_t nt, double lambda, double* out,
                     unsigned long long* clash, cudaStream_t st) {
    if (nt <= 0) return;
    const size_t smem = (kFamily == VPG_LAPLACE ? size_t(kLogTableBytes) : 0) +
                        sizeof(double2) * 2 * kDirThreads;
    smem_optin((const void*)allpairs_kernel<kFamily, kSkip>, int(smem));
    const int64_t gx = nblk(nt, kDirThreads * kDirTPT);
    // enough CTAs for ~4 resident per SM, but slices of >= 2048 sources
    int64_t nslice = std::max<int64_t>(1, (int64_t(sm_count()) * 4 + gx - 1) / gx);
    nslice = std::min<int64_t>(nslice, std::max<int64_t>(1, ns / 2048));
    nslice = std::min<int64_t>(nslice, 65535);
    const int64_t slice = ((ns + nslice - 1) / nslice + kDirThreads - 1) / kDirThreads * kDirThreads;
    nslice = std::max<int64_t>(1, (ns + slice - 1) / std::max<int64_t>(slice, 1));
    double* partial = nullptr;
    if (nslice > 1)
        VPG_CUDA(cudaMallocAsync(&partial, sizeof(double) * size_t(nslice * nt), st));
    const dim3 grid{unsigned(gx), unsigned(nslice), 1u};
    allpairs_kernel<kFamily, kSkip><<<grid, kDirThreads, smem, st>>>(
        src, q, ns, tgt, nt, std::max<int64_t>(slice, 1), lambda,
        kFamily == VPG_LAPLACE ? lap_log_table_rn_dev() : nullptr,
        kFamily == VPG_LAPLACE ? nullptr : k0_table_dev(), out, partial, clash);
    VPG_LAUNCH_CHECK();
    if (nslice > 1) {
        reduce_slices<<<nblk(nt, 256), 256, 0, st>>>(partial, int(nslice), nt, out);
        VPG_LAUNCH_CHECK();
        VPG_CUDA(cudaFreeAsync(partial, st));
    }
}

}  // namespace

void direct_sum_device(int family, double lambda, const double2* src,
                       const double* q, int64_t ns, const double2* tgt,
                       int64_t nt, double* out, bool skip,
                       unsigned long long* clash, cudaStream_t st) {
    if (family == VPG_LAPLACE) {
        if (skip) launch_allpairs<VPG_LAPLACE, true>(src, q, ns, tgt, nt, lambda, out, clash, st);
        else launch_allpairs<VPG_LAPLACE, false>(src, q, ns, tgt, nt, lambda, out, clash, st);
    } else {
        if (skip) launch_allpairs<VPG_MODIFIED_HELMHOLTZ, true>(src, q, ns, tgt, nt, lambda, out, clash, st);
        else launch_allpairs<VPG_MODIFIED_HELMHOLTZ, false>(src, q, ns, tgt, nt, lambda, out, clash, st);
    }
}

void pairwise_apply(const Plan& pl, const double* q_dev, double* out_dev,
                    cudaStream_t st, int64_t& launches) {
    if (pl.nt == 0) return;
    if (pl.ns == 0) {
        VPG_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double) * size_t(pl.nt), st));
        return;
    }
    direct_sum_device(pl.family, pl.lambda, pl.src.p, q_dev, pl.ns, pl.tgt.p, pl.nt,
                      out_dev, true, nullptr, st);
    launches += 2;
}

}  // namespace vpg
