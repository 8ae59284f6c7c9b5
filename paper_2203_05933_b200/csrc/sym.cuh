// sym.cuh -- the symmetric near field (plan.cuh SymTask), templated on the
// pair function so the Laplace FMM (fmm.cu) and the Chebyshev
// modified-Helmholtz FMM (helm.cu) share one schedule and one kernel.
#pragma once

#include "common.cuh"
#include "plan.cuh"

namespace vpg {
namespace {

// Plans with "targets = nodes" (SymTask, plan.cuh): log r^2 of an unordered
// pair is evaluated once and feeds both targets.  A warp takes one task
// (leaf A against its flat column list: A itself, then the neighbours whose
// pairs A owns) from a ticket.  Rows are A's points, R = 1 or 2 per lane;
// columns come in 32-wide tiles staged (twice, so lane + s needs no wrap)
// in per-warp smem.  Step s pairs lane l's rows with column (l + s) mod 32:
// the row sums stay in registers, the column sum travels with its column --
// one shuffle per step hands lane l + 1's accumulator to lane l, so after 32
// steps lane c holds column c again and adds it to the column's partial
// (global, .cg, this warp is its only writer; one read-modify-write per row
// tile).  R = 1, 2, 4 or 8 rows per lane (SymTask::rows2 = log2 R).  v = ln r^2 as one double (t + e ln2 with the split constant: the
// reference's own log is a single rounded double); r^2 of (i, j) and (j, i)
// are bitwise equal, so each ordered pair sees the value the one-sided
// kernel computes.  The pair function K is the kernel: K(r2, tab_lane) =
// ln r^2 (Laplace, fmm.cu) or K0(lambda r) (modified Helmholtz, helm.cu).
// Flat column j vs row i: i <= j feeds the row, i < j the column (the self
// part: i < j both ways, i == j row only -- the Laplace coincidence list
// undoes it as in the one-sided kernel, K0 is 0 at r = 0; neighbour columns
// have j >= na > i).  Row sums are added to slot 4 of A's targets at the end
// of each row tile, after the self-column sums of the earlier tiles.
// Launch shape per pair function (K::kSymWarps warps per CTA, K::kSymMinB
// CTAs per SM; default 8 x 2).  ln r^2 runs 12 warps x 1 CTA so that R = 8
// rows per lane fit (160 registers): tools/pairloop_sweep.cu measured the
// pair loop at 1118 G pairs/s for R = 8 / unroll 2 / 12 x 1 against 1073
// for R = 4 / unroll 4 / 8 x 2 and 1025 for R = 4 / unroll 2 / 8 x 2 --
// instruction-level parallelism inside a warp beats warps per scheduler.
#ifndef VPG_SYM_WARPS
#define VPG_SYM_WARPS 8
#endif
#ifndef VPG_SYM_MINB
#define VPG_SYM_MINB 2
#endif
#ifndef VPG_SYM_UNROLL
#define VPG_SYM_UNROLL 4
#endif
constexpr int kSymUnroll4 = VPG_SYM_UNROLL;  // step unroll at R = 4
template <class K, class = void>
struct SymShape {
    static constexpr int kWarps = VPG_SYM_WARPS, kMinB = VPG_SYM_MINB;
};
template <class K>
struct SymShape<K, decltype(void(K::kSymWarps))> {
    static constexpr int kWarps = K::kSymWarps, kMinB = K::kSymMinB;
};
template <class K>
constexpr size_t sym_smem() {
    return size_t(kLogTableBytes) + size_t(SymShape<K>::kWarps) * (64 * 16 + 64 * 8 + kSymMaxRanges * sizeof(SymRange));
}

template <int R, class K>
__device__ __forceinline__ void sym_block(const K& kern, const double2* cxy, const double* cq, int lane,
                                          const double (&rx)[R], const double (&ry)[R], const double (&rq)[R],
                                          uint32_t tab_lane, double (&racc)[R], double& cacc) {
#pragma unroll(R > 4 ? 2 : R > 2 ? kSymUnroll4 : 4)
    for (int st = 0; st < 32; ++st) {
        const int c = lane + st;
        const double2 sp = cxy[c];
        const double qc = cq[c];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const double dx = rx[u] - sp.x, dy = ry[u] - sp.y;
            const double r2 = fma(dy, dy, dx * dx);
            const double v = kern(r2, tab_lane);
            racc[u] = fma(qc, v, racc[u]);
            cacc = fma(rq[u], v, cacc);
        }
        cacc = __shfl_sync(0xffffffffu, cacc, (lane + 1) & 31);
    }
}

// A column tile of A itself that meets the row tile's diagonal: the 32
// columns start at row sub-tile N - 1 of the R (j0 = i0 + 32 (N - 1)).
// Sub-tiles below N - 1 lie wholly above the diagonal (i < j: plain pairs),
// sub-tile N - 1 is the diagonal one -- row i0' + lane against column
// i0' + (lane + st) mod 32, so i <= j exactly when lane + st does not wrap
// and i < j when also st > 0 -- and the sub-tiles after it lie below the
// diagonal and are skipped (their pairs belong to the transposed tile).
template <int R, int N, class K>
__device__ __forceinline__ void sym_block_diag(const K& kern, const double2* cxy, const double* cq, int lane,
                                               const double (&rx)[R], const double (&ry)[R],
                                               const double (&rq)[R], uint32_t tab_lane, double (&racc)[R],
                                               double& cacc) {
#pragma unroll(N > 4 ? 2 : N > 2 ? kSymUnroll4 : 4)
    for (int st = 0; st < 32; ++st) {
        const int c = lane + st;
        const double2 sp = cxy[c];
        const double qc = cq[c];
#pragma unroll
        for (int u = 0; u < N - 1; ++u) {
            const double dx = rx[u] - sp.x, dy = ry[u] - sp.y;
            const double r2 = fma(dy, dy, dx * dx);
            const double v = kern(r2, tab_lane);
            racc[u] = fma(qc, v, racc[u]);
            cacc = fma(rq[u], v, cacc);
        }
        {
            const double dx = rx[N - 1] - sp.x, dy = ry[N - 1] - sp.y;
            const double r2 = fma(dy, dy, dx * dx);
            const double v = kern(r2, tab_lane);
            const bool upper = c < 32;
            racc[N - 1] = fma(upper ? qc : 0.0, v, racc[N - 1]);
            cacc = fma(upper && st > 0 ? rq[N - 1] : 0.0, v, cacc);
        }
        cacc = __shfl_sync(0xffffffffu, cacc, (lane + 1) & 31);
    }
}
template <int R, int N, class K>
__device__ __forceinline__ void sym_diag_dispatch(int ud, const K& kern, const double2* cxy, const double* cq,
                                                  int lane, const double (&rx)[R], const double (&ry)[R],
                                                  const double (&rq)[R], uint32_t tab_lane, double (&racc)[R],
                                                  double& cacc) {
    if (ud == N - 1) sym_block_diag<R, N>(kern, cxy, cq, lane, rx, ry, rq, tab_lane, racc, cacc);
    else if constexpr (N < R) sym_diag_dispatch<R, N + 1>(ud, kern, cxy, cq, lane, rx, ry, rq, tab_lane, racc, cacc);
}

// flat column j -> (range index) by a linear scan of the task's ranges
__device__ __forceinline__ int sym_range_of(const SymRange* rng, int rcount, int j) {
    int r = 0;
    for (int k = 1; k < rcount; ++k)
        if (rng[k].coff <= j) r = k;
    return r;
}

// One subtask: rows [r0, r1) of A (tiles of 32 R) x flat columns [c0, c1).
// A column's partial is stored by the group's first row tile and updated by
// the later ones (same lane: j mod 32); self columns below the group are
// never visited, their slot gets a zero.  Row partials are stored per tile.
template <int R, class K>
__device__ __forceinline__ void sym_task(const K& kern, const SymTask& T, const SymRange* rng, const double2* sxy,
                                         const double* q, double2* cxy, double* cq, uint32_t tab_lane, int lane,
                                         double* part) {
    constexpr double kFar = 1e100;
    const int ct_end = (T.c1 + 31) >> 5;
    for (int ct = T.c0 >> 5; ct < min(ct_end, T.r0 >> 5); ++ct) {
        const int j = ct * 32 + lane;
        if (j < T.c1) {
            const SymRange& g = rng[sym_range_of(rng, T.rcount, j)];
            part[g.b_part + int64_t(T.rg) * g.nb + (j - g.coff)] = 0.0;
        }
    }
    for (int r0 = T.r0; r0 < T.r1; r0 += 32 * R) {
        double rx[R], ry[R], rq[R], racc[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int i = r0 + lane + 32 * u;
            rx[u] = ry[u] = kFar;
            rq[u] = racc[u] = 0.0;
            if (i < T.r1) {
                const double2 p = sxy[T.a_src + i];
                rx[u] = p.x;
                ry[u] = p.y;
                rq[u] = q[T.a_src + i];
            }
        }
        const bool first = r0 == T.r0;
        // column tile ct + 1 is fetched into registers while tile ct is summed
        double2 p = make_double2(-kFar, -kFar);
        double qj = 0.0;
        int64_t dst = -1;
        auto fetch = [&](int ct) {
            const int j = ct * 32 + lane;
            p = make_double2(-kFar, -kFar);
            qj = 0.0;
            dst = -1;
            if (ct < ct_end && j < T.c1) {
                const SymRange& g = rng[sym_range_of(rng, T.rcount, j)];
                p = sxy[g.b_src + (j - g.coff)];
                qj = q[g.b_src + (j - g.coff)];
                dst = g.b_part + int64_t(T.rg) * g.nb + (j - g.coff);
            }
        };
        const int ct_begin = max(T.c0 >> 5, r0 >> 5);
        fetch(ct_begin);
        for (int ct = ct_begin; ct < ct_end; ++ct) {
            __syncwarp();
            cxy[lane] = p;
            cxy[lane + 32] = p;
            cq[lane] = qj;
            cq[lane + 32] = qj;
            __syncwarp();
            const int64_t dcur = dst;
            double cacc = !first && dcur >= 0 ? part[dcur] : 0.0;  // the earlier row tiles' sum, in flight under the tile
            fetch(ct + 1);
            const int ud = (ct * 32 - r0) >> 5;  // >= 0: self columns below the row tile are never visited
            if (ct * 32 < T.na && ud < R)
                sym_diag_dispatch<R, 1>(ud, kern, cxy, cq, lane, rx, ry, rq, tab_lane, racc, cacc);
            else
                sym_block<R>(kern, cxy, cq, lane, rx, ry, rq, tab_lane, racc, cacc);
            if (dcur >= 0) part[dcur] = cacc;
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int i = r0 + lane + 32 * u;
            if (i < T.r1) part[T.a_part + i] = racc[u];
        }
    }
}

template <class K>
__global__ void __launch_bounds__(SymShape<K>::kWarps * 32, SymShape<K>::kMinB)
p2p_sym_kernel(K kern, const SymTask* tasks, int64_t ntask, const SymRange* ranges, const double2* sxy,
               const double* q, const double2* gtab, int* ticket, double* part) {
    constexpr int kSymWarps = SymShape<K>::kWarps;
    extern __shared__ double2 smp[];
    double2* tab = smp;                                                   // log table
    double2* cbuf = smp + kLogTableSize * kLogTableCopies;                // [warps][64] xy
    double* qbuf = reinterpret_cast<double*>(cbuf + kSymWarps * 64);     // [warps][64]
    SymRange* rbuf = reinterpret_cast<SymRange*>(qbuf + kSymWarps * 64);  // [warps][kSymMaxRanges]
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    bulk_stage(cbuf, gtab, uint32_t(kLogTableSize) * 16u, &bar, 0);
    log_table_to_smem(tab, cbuf);
    pdl_trigger();
    pdl_wait();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab_lane = log_table_lane_addr(tab, lane & (kLogTableCopies - 1));
    double2* cxy = cbuf + warp * 64;
    double* cq = qbuf + warp * 64;
    SymRange* rng = rbuf + warp * kSymMaxRanges;
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&ticket[1], 1);
        const int64_t ti = __shfl_sync(0xffffffffu, k, 0);
        if (ti >= ntask) break;
        const SymTask T = tasks[ti];
        __syncwarp();
        if (lane < T.rcount) rng[lane] = ranges[T.rfirst + lane];
        __syncwarp();
        if (K::kSymMaxR >= 8 && T.rows2 == 3) sym_task<K::kSymMaxR >= 8 ? 8 : 2>(kern, T, rng, sxy, q, cxy, cq, tab_lane, lane, part);
        else if (K::kSymMaxR >= 4 && T.rows2 == 2) sym_task<K::kSymMaxR >= 4 ? 4 : 2>(kern, T, rng, sxy, q, cxy, cq, tab_lane, lane, part);
        else if (T.rows2) sym_task<2>(kern, T, rng, sxy, q, cxy, cq, tab_lane, lane, part);
        else sym_task<1>(kern, T, rng, sxy, q, cxy, cq, tab_lane, lane, part);
    }
}

}  // namespace
}  // namespace vpg
