// fmm.cu -- 2D Laplace FMM passes on the device (FP64):
//   P2M, M2M, M2L (factorised, batched as a dense real GEMM), L2L, and the
//   fused L2P + near-field P2P.  Follows laplace_apply (summation.cpp:224-348)
//   with the operators of build_laplace_ops (summation.cpp:150-222).
//
// Expansions are box-scaled like the reference: a box of side s centred at
// c holds multipoles in s/(z-c) and locals in (z-c)/s (summation.cpp:131-134),
// so every operator depends only on integer offsets and is shared by all
// levels.
#include <algorithm>
#include <cmath>
#include <vector>

#include "p2p.cuh"
#include "plan.cuh"

namespace vpg {

namespace {

__constant__ double c_neg_inv_k[64];  // -1/k, k = 1..63 (index k)

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

__device__ inline void box_center(double x0, double y0, double s, uint32_t id,
                                  double& cx, double& cy) {
    // summation.cpp:74-78
    cx = x0 + (squash2(id) + 0.5) * s;
    cy = y0 + (squash2(id >> 1) + 0.5) * s;
}

// ------------------------------------------------------------------ P2M --
// One CTA (64 threads) per non-empty source leaf.  Sources are processed 32
// at a time: lane t forms the running powers q*w^k of its source
// (summation.cpp:247-254) into a [32][P+1] smem panel; thread k then sums
// column k in source order, so each coefficient is reduced in the same
// order as the reference loop.  Row stride P+1 complex keeps the 128-bit
// panel accesses of each quarter-warp on distinct banks for odd P+1.
constexpr int kP2MThreads = 64;

__global__ void __launch_bounds__(kP2MThreads)
p2m_kernel(const int32_t* leaves, const int32_t* soff, const double2* sxy,
           const double* q, int P, double x0, double y0, double s,
           double2* mult_leaf) {
    extern __shared__ double2 panel[];  // [32][P+1]
    const int n = P + 1;
    const uint32_t b = uint32_t(leaves[blockIdx.x]);
    double cx, cy;
    box_center(x0, y0, s, b, cx, cy);
    const double inv_s = 1.0 / s;
    const int e0 = soff[b], e1 = soff[b + 1];
    const int k = threadIdx.x;
    double2 acc = make_double2(0.0, 0.0);
    for (int base = e0; base < e1; base += 32) {
        const int cnt = min(32, e1 - base);
        if (k < cnt) {
            const double2 p = sxy[base + k];
            const double wr = (p.x - cx) * inv_s, wi = (p.y - cy) * inv_s;
            const double qj = q[base + k];
            double2* row = panel + k * n;
            row[0] = make_double2(qj, 0.0);
            double pr = qj, pi = 0.0;
            for (int j = 1; j <= P; ++j) {
                const double nr = pr * wr - pi * wi;
                const double ni = pr * wi + pi * wr;
                pr = nr;
                pi = ni;
                const double f = c_neg_inv_k[j];
                row[j] = make_double2(f * pr, f * pi);
            }
        }
        __syncthreads();
        if (k <= P)
            for (int t = 0; t < cnt; ++t) {
                const double2 v = panel[t * n + k];
                acc.x += v.x;
                acc.y += v.y;
            }
        __syncthreads();
    }
    if (k <= P) mult_leaf[int64_t(b) * n + k] = acc;
}

// ------------------------------------------------------------ M2M / L2L --
// Shared-operator batched matvec.  A CTA takes kShiftGroup parents of one
// level; for each child index c it stages the (P+1)^2 complex operator
// (transposed, 41.6 KB at P=50) in smem and applies it to every parent of
// the group.  Upward (M2M, summation.cpp:257-267): parent = sum_c
// m2m[c] * child_c over children with src_cnt > 0, reduced in c order.
// Downward (L2L, summation.cpp:305-312): child += l2l[c] * parent for
// children with tgt_cnt > 0.  Each output vector is owned by one thread
// row, so there are no atomics.
constexpr int kShiftGroup = 8;
constexpr int kShiftThreads = 64;

template <bool kUp>
__global__ void __launch_bounds__(kShiftThreads)
shift_kernel(const int32_t* parents, int64_t nparents, const double2* ops_t,
             const int32_t* cnt_child, const double2* in_level,
             double2* out_level, double2* child_level_out, int P) {
    extern __shared__ double2 sm[];
    const int n = P + 1;
    double2* op = sm;                  // [k][r]
    double2* vec = sm + n * n;         // [g][k]
    const int64_t g0 = int64_t(blockIdx.x) * kShiftGroup;
    const int ng = int(min(int64_t(kShiftGroup), nparents - g0));
    const int r = threadIdx.x;
    double2 acc[kShiftGroup];
#pragma unroll
    for (int g = 0; g < kShiftGroup; ++g) acc[g] = make_double2(0.0, 0.0);

    if (!kUp) {
        // parents' local expansions are the input for every c
        for (int i = threadIdx.x; i < ng * n; i += blockDim.x) {
            const int g = i / n, kk = i % n;
            vec[g * n + kk] = in_level[int64_t(parents[g0 + g]) * n + kk];
        }
    }
    for (int c = 0; c < 4; ++c) {
        __syncthreads();
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) op[i] = ops_t[int64_t(c) * n * n + i];
        if (kUp) {
            for (int i = threadIdx.x; i < ng * n; i += blockDim.x) {
                const int g = i / n, kk = i % n;
                const int64_t child = (int64_t(parents[g0 + g]) << 2) | c;
                vec[g * n + kk] = cnt_child[child] > 0 ? in_level[child * n + kk]
                                                       : make_double2(0.0, 0.0);
            }
        }
        __syncthreads();
        if (r <= P) {
            double2 y[kShiftGroup];
#pragma unroll
            for (int g = 0; g < kShiftGroup; ++g) y[g] = make_double2(0.0, 0.0);
            for (int kk = 0; kk <= P; ++kk) {
                const double2 m = op[kk * n + r];
#pragma unroll
                for (int g = 0; g < kShiftGroup; ++g) {
                    const double2 x = vec[g * n + kk];
                    y[g].x = fma(m.x, x.x, fma(-m.y, x.y, y[g].x));
                    y[g].y = fma(m.x, x.y, fma(m.y, x.x, y[g].y));
                }
            }
            if (kUp) {
#pragma unroll
                for (int g = 0; g < kShiftGroup; ++g) {
                    acc[g].x += y[g].x;
                    acc[g].y += y[g].y;
                }
            } else {
                for (int g = 0; g < ng; ++g) {
                    const int64_t child = (int64_t(parents[g0 + g]) << 2) | c;
                    if (cnt_child[child] > 0) {
                        double2* dst = child_level_out + child * n + r;
                        double2 v = *dst;
                        v.x += y[g].x;
                        v.y += y[g].y;
                        *dst = v;
                    }
                }
            }
        }
    }
    if (kUp && r <= P)
        for (int g = 0; g < ng; ++g) out_level[int64_t(parents[g0 + g]) * n + r] = acc[g];
}

// ------------------------------------------------------------------ M2L --
// Factorised translation.  For offset d (in units of
// the box side) the reference operator (summation.cpp:209-218) is
//   M[l][k] = (-1)^k C(l+k-1, k-1) d^-(l+k)  (k >= 1),
//   M[l][0] = -d^-l / l (l >= 1),  M[0][0] = log(-d),
// so with a~_k = (-1)^k d^-k a_k and the real, offset-independent
// H[l][k] = C(l+k-1, k-1):
//   y = H a~,  b_0 = y_0 + log(-d) a_0,  b_l = d^-l (y_l - a_0 / l).
// A batch (<= kM2LPairs list entries of consecutive target boxes of one
// level) becomes ONE dense real GEMM Y[RP x 2*pairs] = H[RP x P] X[P x
// 2*pairs] (re and im columns), with H^T and X staged in smem and an 8x8
// register micro-tile per thread.  The epilogue applies the d^-l scaling
// and reduces each target's entries in list order, then adds the monopole
// shift qsum*log(s_l) (summation.cpp:297-301).  Executed flops per pair:
// 4 P (P+1) for the GEMM + O(P) epilogue, half of the dense 8 (P+1)^2.
constexpr int kM2LCols = 2 * kM2LPairs;  // 256
constexpr int kM2LColGroups = 32;        // 8 columns each, interleaved

__global__ void __launch_bounds__(7 * kM2LColGroups)
m2l_kernel(const M2LBatch* batches, const int32_t* tbox, const int32_t* toff,
           const int32_t* esrc, const int32_t* eoidx, const double* h_t,
           const double2* dpow, const double2* logmd, const double2* mult,
           double2* loc, const int64_t* exp_off, int P, int RP, double side) {
    extern __shared__ double smd[];
    const int n = P + 1;
    const int dp_stride = 2 * P + 1;
    double* hs = smd;                        // [P][RP]
    double* xy = hs + P * RP;                // [n][kM2LCols]
    double2* a0s = reinterpret_cast<double2*>(xy + n * kM2LCols);  // [pairs]
    int* os = reinterpret_cast<int*>(a0s + kM2LPairs);             // [pairs]

    const M2LBatch bt = batches[blockIdx.x];
    const int level = bt.level;
    const double2* mlev = mult + exp_off[level];
    double2* llev = loc + exp_off[level];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;

    for (int i = tid; i < P * RP; i += nthr) hs[i] = h_t[i];
    // X[k-1][2p | 2p+1] = (-1)^k d^-k a_k  (k = 1..P)
    for (int i = tid; i < bt.ecount * n; i += nthr) {
        const int p = i / n, k = i % n;
        const int64_t e = int64_t(bt.efirst) + p;
        const int sid = esrc[e];
        const int o = eoidx[e];
        const double2 a = mlev[int64_t(sid) * n + k];
        if (k == 0) {
            a0s[p] = a;
            os[p] = o;
        } else {
            double2 sg = dpow[o * dp_stride + k];
            if (k & 1) {
                sg.x = -sg.x;
                sg.y = -sg.y;
            }
            xy[(k - 1) * kM2LCols + 2 * p] = a.x * sg.x - a.y * sg.y;
            xy[(k - 1) * kM2LCols + 2 * p + 1] = a.x * sg.y + a.y * sg.x;
        }
    }
    __syncthreads();

    // GEMM: thread (rg, cg) owns rows rg*8..rg*8+7, columns cg + 32 j.
    const int rg = tid / kM2LColGroups, cg = tid % kM2LColGroups;
    const bool active_rows = rg * 8 < RP;
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    if (active_rows) {
        for (int k = 0; k < P; ++k) {
            const double* hrow = hs + k * RP + rg * 8;
            const double2 h01 = *reinterpret_cast<const double2*>(hrow);
            const double2 h23 = *reinterpret_cast<const double2*>(hrow + 2);
            const double2 h45 = *reinterpret_cast<const double2*>(hrow + 4);
            const double2 h67 = *reinterpret_cast<const double2*>(hrow + 6);
            const double h[8] = {h01.x, h01.y, h23.x, h23.y, h45.x, h45.y, h67.x, h67.y};
            const double* xrow = xy + k * kM2LCols + cg;
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = xrow[32 * j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(h[i], x[j], acc[i][j]);
        }
    }
    __syncthreads();
    if (active_rows) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int l = rg * 8 + i;
            if (l < n)
#pragma unroll
                for (int j = 0; j < 8; ++j) xy[l * kM2LCols + cg + 32 * j] = acc[i][j];
        }
    }
    __syncthreads();

    // Epilogue: thread -> (target t, coefficient l); t fastest so the smem
    // reads of one warp fall on different columns.
    const double logs = log(side / double(1 << level));
    for (int i = tid; i < bt.tcount * n; i += nthr) {
        const int t = i % bt.tcount, l = i / bt.tcount;
        const int64_t tg = int64_t(bt.tfirst) + t;
        const int p0 = toff[tg] - bt.efirst, p1 = toff[tg + 1] - bt.efirst;
        double sr = 0.0, si = 0.0, qsum = 0.0;
        const double inv_l = l > 0 ? c_neg_inv_k[l] : 0.0;  // -1/l
        for (int p = p0; p < p1; ++p) {
            const double yr = xy[l * kM2LCols + 2 * p];
            const double yi = xy[l * kM2LCols + 2 * p + 1];
            const double2 a0 = a0s[p];
            const int o = os[p];
            if (l == 0) {
                const double2 lg = logmd[o];
                sr += yr + (lg.x * a0.x - lg.y * a0.y);
                si += yi + (lg.x * a0.y + lg.y * a0.x);
                qsum += a0.x;
            } else {
                const double zr = fma(inv_l, a0.x, yr), zi = fma(inv_l, a0.y, yi);
                const double2 dl = dpow[o * dp_stride + l];
                sr += dl.x * zr - dl.y * zi;
                si += dl.x * zi + dl.y * zr;
            }
        }
        if (l == 0) sr += qsum * logs;
        llev[int64_t(tbox[tg]) * n + l] = make_double2(sr, si);
    }
}

// -------------------------------------------------- L2P + near-field P2P --
// A persistent grid of warps walks the target chunks (<= 32*TPT targets of
// one leaf).  Per chunk: each lane evaluates the local expansion of its
// targets by Horner in u = (t-c)/s (summation.cpp:326-329), then sums the
// 3x3 neighbour leaves (summation.cpp:330-344) in the reference order,
// staging 32 sources at a time in a per-warp smem slot (one coalesced load
// per lane, then warp-broadcast reads).  Output is scattered to the
// original target order (summation.cpp:345).
constexpr int kP2PWarps = 8;

template <int TPT>
__global__ void __launch_bounds__(kP2PWarps * 32)
l2p_p2p_kernel(const P2PChunk* chunks, int64_t nchunks, const int32_t* soff,
               const double2* sxy, const double* q, const double2* txy,
               const int32_t* tids, const double2* loc_leaf, int P, int L,
               double x0, double y0, double s, const double2* gtab, double* out) {
    extern __shared__ double2 smp[];
    double2* tab = smp;                                     // log table
    double2* sbuf = smp + kLogTableSize * kLogTableCopies;  // [warps][32][2]
    log_table_to_smem(tab, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lane8 = lane & 7;
    double2* my = sbuf + warp * 64;
    const int nb = 1 << L;
    const int n = P + 1;
    const double inv_s = 1.0 / s;

    for (int64_t ch = int64_t(blockIdx.x) * kP2PWarps + warp; ch < nchunks;
         ch += int64_t(gridDim.x) * kP2PWarps) {
        const P2PChunk c = chunks[ch];
        const uint32_t b = uint32_t(c.leaf);
        double cx, cy;
        box_center(x0, y0, s, b, cx, cy);
        double tx[TPT], ty[TPT], pot[TPT];
        LapAcc acc[TPT];
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
            const int li = min(lane + 32 * u, c.tcount - 1);
            const double2 t = txy[c.tbegin + li];
            tx[u] = t.x;
            ty[u] = t.y;
            // L2P (summation.cpp:326-329)
            const double ur = (t.x - cx) * inv_s, ui = (t.y - cy) * inv_s;
            const double2* ab = loc_leaf + int64_t(b) * n;
            double vr = ab[P].x, vi = ab[P].y;
            for (int l = P - 1; l >= 0; --l) {
                const double2 a = ab[l];
                const double nr = fma(vr, ur, fma(-vi, ui, a.x));
                const double ni = fma(vr, ui, fma(vi, ur, a.y));
                vr = nr;
                vi = ni;
            }
            pot[u] = -kInv2Pi * vr;
        }
        const int ix = int(squash2(b)), iy = int(squash2(b >> 1));
        for (int jy = max(0, iy - 1); jy <= min(nb - 1, iy + 1); ++jy) {
            for (int jx = max(0, ix - 1); jx <= min(nb - 1, ix + 1); ++jx) {
                const uint32_t sid = mort(uint32_t(jx), uint32_t(jy));
                const int f0 = soff[sid], f1 = soff[sid + 1];
                for (int base = f0; base < f1; base += 32) {
                    const int cnt = min(32, f1 - base);
                    __syncwarp();
                    if (lane < cnt) {
                        my[2 * lane] = sxy[base + lane];
                        my[2 * lane + 1] = make_double2(q[base + lane], 0.0);
                    }
                    __syncwarp();
                    for (int j = 0; j < cnt; ++j) {
                        const double2 sp = my[2 * j];
                        const double qj = my[2 * j + 1].x;
#pragma unroll
                        for (int u = 0; u < TPT; ++u)
                            lap_pair(tx[u], ty[u], sp.x, sp.y, qj, tab, lane8, acc[u]);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
            const int li = lane + 32 * u;
            if (li < c.tcount) {
                const double v = pot[u] - kInv4Pi * lap_total(acc[u]);
                out[tids[c.tbegin + li]] = v;
            }
        }
    }
}

__global__ void gather_q(const double* q, const int32_t* ids, int64_t n, double* qs) {
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e < n) qs[e] = q[ids[e]];
}


}  // namespace

// ------------------------------------------------------------- operators --
void build_laplace_ops(Plan& pl) {
    // P from epsilon (summation.cpp:155-157)
    pl.P = std::clamp(int(std::ceil(std::log(1.0 / pl.eps) / std::log(1.83))) + 4, 10, 60);
    const int P = pl.P, n = P + 1;
    pl.RP = ((n + 7) / 8) * 8;
    if (pl.RP > 56) throw Error{VPG_ERR_INVALID_ARGUMENT, "expansion order above 55"};

    // Pascal triangle to 2P (summation.cpp:160-168)
    const int nb = 2 * P + 1;
    std::vector<double> C(size_t(nb) * nb, 0.0);
    auto B = [&](int i, int j) -> double& { return C[size_t(i) * nb + j]; };
    for (int i = 0; i <= 2 * P; ++i) {
        B(i, 0) = 1.0;
        for (int j = 1; j <= i; ++j) B(i, j) = B(i - 1, j - 1) + (j <= i - 1 ? B(i - 1, j) : 0.0);
    }

    // M2M / L2L for child c at (+-1/4, +-1/4) of the parent side, bit 0 = x
    // (summation.cpp:170-197); stored transposed ([k][r]) for the kernels.
    std::vector<cplx> up_t(size_t(4) * n * n, cplx{0, 0}), dn_t(size_t(4) * n * n, cplx{0, 0});
    for (int c = 0; c < 4; ++c) {
        const cplx t{(c & 1) ? 0.25 : -0.25, (c & 2) ? 0.25 : -0.25};
        std::vector<cplx> tp(size_t(2 * P + 1));
        tp[0] = {1.0, 0.0};
        for (int j = 1; j <= 2 * P; ++j) tp[size_t(j)] = cmul(tp[size_t(j - 1)], t);
        cplx* U = up_t.data() + size_t(c) * n * n;
        cplx* D = dn_t.data() + size_t(c) * n * n;
        U[0] = {1.0, 0.0};
        double sig = 1.0;
        std::vector<double> sg(static_cast<size_t>(n));
        for (int k = 0; k <= P; ++k, sig *= 0.5) sg[size_t(k)] = sig;
        for (int l = 1; l <= P; ++l) {
            const double f = -1.0 / l;
            U[size_t(0) * n + l] = {f * tp[size_t(l)].re, f * tp[size_t(l)].im};  // [k=0][r=l]
            for (int k = 1; k <= l; ++k) {
                const double w = sg[size_t(k)] * B(l - 1, k - 1);
                U[size_t(k) * n + l] = {w * tp[size_t(l - k)].re, w * tp[size_t(l - k)].im};
            }
        }
        double half = 1.0;
        for (int m = 0; m <= P; ++m, half *= 0.5)
            for (int l = m; l <= P; ++l) {
                const double w = half * B(l, m);
                D[size_t(l) * n + m] = {w * tp[size_t(l - m)].re, w * tp[size_t(l - m)].im};
            }
    }

    // M2L factors: H^T[k-1][l] = C(l+k-1, k-1); d^-j and log(-d) per offset
    // (summation.cpp:199-220).
    std::vector<double> ht(size_t(P) * pl.RP, 0.0);
    for (int k = 1; k <= P; ++k)
        for (int l = 0; l <= P; ++l) ht[size_t(k - 1) * pl.RP + l] = B(l + k - 1, k - 1);
    const int dps = 2 * P + 1;
    std::vector<cplx> dpw(size_t(49) * dps, cplx{0, 0});
    std::vector<cplx> lg(49, cplx{0, 0});
    for (int dy = -3; dy <= 3; ++dy)
        for (int dx = -3; dx <= 3; ++dx) {
            if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
            const int o = (dx + 3) + 7 * (dy + 3);
            const double m2 = double(dx) * dx + double(dy) * dy;
            const cplx dinv{dx / m2, -dy / m2};
            cplx* dp = dpw.data() + size_t(o) * dps;
            dp[0] = {1.0, 0.0};
            for (int j = 1; j <= 2 * P; ++j) dp[j] = cmul(dp[j - 1], dinv);
            lg[size_t(o)] = {0.5 * std::log(m2), std::atan2(double(-dy), double(-dx))};
        }

    cudaStream_t st = 0;
    pl.m2m_ops.alloc(size_t(4) * n * n * 2);
    pl.l2l_ops.alloc(size_t(4) * n * n * 2);
    pl.h_t.alloc(ht.size());
    pl.dpow.alloc(dpw.size());
    pl.logmd.alloc(lg.size());
    VPG_CUDA(cudaMemcpyAsync(pl.m2m_ops.p, up_t.data(), pl.m2m_ops.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.l2l_ops.p, dn_t.data(), pl.l2l_ops.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.h_t.p, ht.data(), pl.h_t.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.dpow.p, dpw.data(), pl.dpow.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.logmd.p, lg.data(), pl.logmd.bytes(), cudaMemcpyHostToDevice, st));
    double nik[64] = {0.0};
    for (int k = 1; k < 64; ++k) nik[k] = -1.0 / k;
    VPG_CUDA(cudaMemcpyToSymbol(c_neg_inv_k, nik, sizeof(nik)));
    VPG_CUDA(cudaStreamSynchronize(st));

    // expansion layout: levels 2..L, 4^l boxes x (P+1) complex each
    pl.exp_off.assign(size_t(pl.L + 1), 0);
    int64_t off = 0;
    for (int l = 2; l <= pl.L; ++l) {
        pl.exp_off[size_t(l)] = off;
        off += (int64_t(1) << (2 * l)) * n;
    }
    pl.exp_total = off;
    pl.exp_off_dev.alloc(pl.exp_off.size());
    VPG_CUDA(cudaMemcpy(pl.exp_off_dev.p, pl.exp_off.data(), pl.exp_off_dev.bytes(),
                        cudaMemcpyHostToDevice));

    smem_optin((const void*)m2l_kernel, 200 * 1024);
    smem_optin((const void*)shift_kernel<true>, 100 * 1024);
    smem_optin((const void*)shift_kernel<false>, 100 * 1024);
    smem_optin((const void*)l2p_p2p_kernel<1>, 64 * 1024);
    smem_optin((const void*)l2p_p2p_kernel<2>, 64 * 1024);
}

// ----------------------------------------------------------------- apply --
void laplace_apply(const Plan& pl, const double* q_dev, double* out_dev,
                   cudaStream_t st, cudaEvent_t* ev, int64_t& launches) {
    const int P = pl.P, n = P + 1, L = pl.L;
    auto mark = [&](int i) {
        if (ev) VPG_CUDA(cudaEventRecord(ev[i], st));
    };
    // scratch: sorted charges, then mult and loc expansions (stream-ordered)
    double* qs = nullptr;
    double2* mult = nullptr;
    double2* loc = nullptr;
    VPG_CUDA(cudaMallocAsync(&qs, sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1)), st));
    VPG_CUDA(cudaMallocAsync(&mult, sizeof(double2) * size_t(pl.exp_total), st));
    VPG_CUDA(cudaMallocAsync(&loc, sizeof(double2) * size_t(pl.exp_total), st));
    struct Free {
        void* p[3];
        cudaStream_t s;
        ~Free() {
            for (void* x : p)
                if (x) cudaFreeAsync(x, s);
        }
    } fr{{qs, mult, loc}, st};
    const int64_t* exp_off_d = pl.exp_off_dev.p;

    mark(0);
    gather_q<<<nblk(pl.ns, 256), 256, 0, st>>>(q_dev, pl.src_ids.p, pl.ns, qs);
    VPG_LAUNCH_CHECK();
    ++launches;
    mark(1);

    const double sL = pl.side / double(1 << L);
    if (pl.n_p2m_leaves > 0) {
        p2m_kernel<<<unsigned(pl.n_p2m_leaves), kP2MThreads, 32 * n * sizeof(double2), st>>>(
            pl.p2m_leaves.p, pl.src_off.p, pl.src_sorted.p, qs, P, pl.x0, pl.y0, sL,
            mult + pl.exp_off[size_t(L)]);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(2);
    const size_t shift_smem = sizeof(double2) * size_t(n * n + kShiftGroup * n);
    for (int l = L - 1; l >= 2; --l) {
        const int64_t np = pl.m2m_count[size_t(l)];
        if (!np) continue;
        shift_kernel<true><<<nblk(np, kShiftGroup), kShiftThreads, shift_smem, st>>>(
            pl.updown_boxes.p + pl.m2m_first[size_t(l)], np,
            reinterpret_cast<const double2*>(pl.m2m_ops.p),
            pl.src_cnt.p + lvl_base(l + 1), mult + pl.exp_off[size_t(l + 1)],
            mult + pl.exp_off[size_t(l)], nullptr, P);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(3);
    if (pl.n_m2l_batches > 0) {
        const size_t smem = sizeof(double) * (size_t(P) * pl.RP + size_t(n) * kM2LCols) +
                            sizeof(double2) * kM2LPairs + sizeof(int) * kM2LPairs;
        const int threads = (pl.RP / 8) * kM2LColGroups;
        m2l_kernel<<<unsigned(pl.n_m2l_batches), threads, smem, st>>>(
            pl.m2l_batches.p, pl.m2l_tbox.p, pl.m2l_toff.p, pl.m2l_src.p, pl.m2l_oidx.p,
            pl.h_t.p, pl.dpow.p, pl.logmd.p, mult, loc, exp_off_d, P, pl.RP, pl.side);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(4);
    for (int l = 2; l < L; ++l) {
        const int64_t np = pl.l2l_count[size_t(l)];
        if (!np) continue;
        shift_kernel<false><<<nblk(np, kShiftGroup), kShiftThreads, shift_smem, st>>>(
            pl.updown_boxes.p + pl.l2l_first[size_t(l)], np,
            reinterpret_cast<const double2*>(pl.l2l_ops.p),
            pl.tgt_cnt.p + lvl_base(l + 1), loc + pl.exp_off[size_t(l)], nullptr,
            loc + pl.exp_off[size_t(l + 1)], P);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(5);
    if (pl.n_p2p_chunks > 0) {
        const size_t smem = size_t(kLogTableBytes) + sizeof(double2) * 64 * kP2PWarps;
        const int per_sm = 2;
        const int64_t want = (pl.n_p2p_chunks + kP2PWarps - 1) / kP2PWarps;
        const unsigned grid = unsigned(std::min<int64_t>(want, int64_t(pl.sm_count) * per_sm));
        if (pl.p2p_tpt == 2)
            l2p_p2p_kernel<2><<<grid, kP2PWarps * 32, smem, st>>>(
                pl.p2p_chunks.p, pl.n_p2p_chunks, pl.src_off.p, pl.src_sorted.p, qs,
                pl.tgt_sorted.p, pl.tgt_ids.p, loc + pl.exp_off[size_t(L)], P, L, pl.x0,
                pl.y0, sL, log_table_dev(), out_dev);
        else
            l2p_p2p_kernel<1><<<grid, kP2PWarps * 32, smem, st>>>(
                pl.p2p_chunks.p, pl.n_p2p_chunks, pl.src_off.p, pl.src_sorted.p, qs,
                pl.tgt_sorted.p, pl.tgt_ids.p, loc + pl.exp_off[size_t(L)], P, L, pl.x0,
                pl.y0, sL, log_table_dev(), out_dev);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(6);
}

}  // namespace vpg
