// fmm.cu -- 2D Laplace FMM passes on the device (FP64):
//   P2M, M2M, M2L (factorised, batched as a dense real GEMM), L2L, and the
//   fused L2P + near-field P2P.  Follows laplace_apply (summation.cpp:224-348)
//   with the operators of build_laplace_ops (summation.cpp:150-222).
//
// Expansions are box-scaled like the reference: a box of side s centred at
// c holds multipoles in s/(z-c) and locals in (z-c)/s (summation.cpp:131-134),
// so every operator depends only on integer offsets and is shared by all
// levels.
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>

#include "p2p.cuh"
#include "plan.cuh"
#include "sym.cuh"

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
// One warp per work item = (level, box, source range).  Lane 4 j + h:
// source stream j (0..7: the item's sources j, j + 8, ...) and quarter h of
// the powers, k in (h KQ, (h + 1) KQ].  Every lane keeps the sums of q w^k
// over its stream's sources for its KQ powers IN REGISTERS (summation.cpp:
// 247-254 with the sums reassociated: per stream, then across the 8 streams
// by shuffles, once per item); quarter h of a source runs one step after
// quarter h - 1 and takes over its running power q w^(h KQ) and w by a
// shuffle from the neighbouring lane, so no power is formed twice and
// nothing goes through shared memory -- the per-source smem panel of the
// first version (25 STS.128 + 32 LDS.128 per 16 sources and warp) capped
// P2M at the shared-memory pipe: cfg4 0.276 ms against 0.08 ms of FP64 work.
// The factors -1/k are applied to the sums, not to the powers.  Leaf items
// cover the reference P2M; in the multilevel upward pass (small problems, see
// laplace_apply) every level's boxes are items too and boxes split into
// several items are summed in item order by p2m_reduce_kernel.
constexpr int kP2MWarps = 4;
constexpr int kP2MSrc = 16;  // p2l_kernel's panel rows
#ifndef VPG_P2M_ILP
#define VPG_P2M_ILP 1
#endif

template <int KQ>
__global__ void __launch_bounds__(kP2MWarps * 32)
p2m_kernel(const P2MItem* items, int64_t nitems, const double2* sxy, const double* q, int P, double x0,
           double y0, double side, double2* mult, double2* partial) {
    pdl_trigger();
    pdl_wait();
    const int n = P + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t li = int64_t(blockIdx.x) * kP2MWarps + warp;
    if (li >= nitems) return;
    const P2MItem it = items[li];
    const double s = side / double(1 << it.level);
    double cx, cy;
    box_center(x0, y0, s, uint32_t(it.box), cx, cy);
    const double inv_s = 1.0 / s;
    const int e0 = it.e0, e1 = it.e1;
    const int j = lane >> 2, h = lane & 3;
    // S sources of the stream per step (2 S independent multiply chains per lane; S = 2
    // measured slower: cfg4 0.140 -> 0.177 ms, one more fill/drain step in three and 118 registers)
    constexpr int S = VPG_P2M_ILP;
    const int nstep = (e1 - e0 + 8 * S - 1) / (8 * S) + 3;  // + 3: the last sources' upper quarters
    double ar[KQ], ai[KQ];
#pragma unroll
    for (int t = 0; t < KQ; ++t) ar[t] = ai[t] = 0.0;
    double a0 = 0.0;  // sum q (lanes h = 0)
    double pr[S], pi[S], wr[S], wi[S];  // running powers q w^k and w of the lane's current sources
    double2 pn[S];                      // quarter 0 loads one step ahead
    double qn[S];
#pragma unroll
    for (int u = 0; u < S; ++u) {
        pr[u] = pi[u] = wr[u] = wi[u] = 0.0;
        pn[u] = make_double2(cx, cy);
        qn[u] = 0.0;
        const int i0 = e0 + j + 8 * u;
        if (h == 0 && i0 < e1) {
            pn[u] = sxy[i0];
            qn[u] = q[i0];
        }
    }
    for (int st = 0; st < nstep; ++st) {
#pragma unroll
        for (int u = 0; u < S; ++u) {
            // the neighbouring quarter's state after its previous step
            const double tpr = __shfl_up_sync(0xffffffffu, pr[u], 1), tpi = __shfl_up_sync(0xffffffffu, pi[u], 1);
            const double twr = __shfl_up_sync(0xffffffffu, wr[u], 1), twi = __shfl_up_sync(0xffffffffu, wi[u], 1);
            if (h == 0) {
                wr[u] = (pn[u].x - cx) * inv_s;
                wi[u] = (pn[u].y - cy) * inv_s;
                pr[u] = qn[u];
                pi[u] = 0.0;
                a0 += qn[u];
                const int nx = e0 + j + 8 * (S * (st + 1) + u);
                pn[u] = make_double2(cx, cy);
                qn[u] = 0.0;
                if (nx < e1) {
                    pn[u] = sxy[nx];
                    qn[u] = q[nx];
                }
            } else {
                pr[u] = tpr;
                pi[u] = tpi;
                wr[u] = twr;
                wi[u] = twi;
            }
        }
#pragma unroll
        for (int t = 0; t < KQ; ++t) {
#pragma unroll
            for (int u = 0; u < S; ++u) {
                const double nr = fma(pr[u], wr[u], -(pi[u] * wi[u]));
                const double ni = fma(pr[u], wi[u], pi[u] * wr[u]);
                pr[u] = nr;
                pi[u] = ni;
            }
            if (S == 2) {
                ar[t] += pr[0] + pr[S - 1];
                ai[t] += pi[0] + pi[S - 1];
            } else {
                ar[t] += pr[0];
                ai[t] += pi[0];
            }
        }
    }
    // the 8 streams' sums (lane bits 2..4) by recursive halving: at each of
    // the three stages a lane keeps one half of its slots and receives the
    // partner's copy of that half, so 14 + 14 values cross the warp instead
    // of 3 x 2 KQ; stream j ends with the slots 8 j0 + 4 j1 + 2 j2 + {0, 1}
    constexpr int KH = 16;
    double vr[KH], vi[KH];
#pragma unroll
    for (int t = 0; t < KH; ++t) {
        vr[t] = t < KQ ? ar[t] : 0.0;
        vi[t] = t < KQ ? ai[t] : 0.0;
    }
#pragma unroll
    for (int stage = 0; stage < 3; ++stage) {
        const int off = 4 << stage, half = KH >> (stage + 1);
        const bool up = lane & off;
        a0 += __shfl_xor_sync(0xffffffffu, a0, off);
#pragma unroll
        for (int t = 0; t < half; ++t) {
            const double sr = up ? vr[t] : vr[t + half], si = up ? vi[t] : vi[t + half];
            const double kr = up ? vr[t + half] : vr[t], ki = up ? vi[t + half] : vi[t];
            vr[t] = kr + __shfl_xor_sync(0xffffffffu, sr, off);
            vi[t] = ki + __shfl_xor_sync(0xffffffffu, si, off);
        }
    }
    double2* dst = it.direct ? mult + int64_t(it.row) * n : partial + li * n;
    if (lane == 0) dst[0] = make_double2(a0, 0.0);
    const int slot0 = 8 * (j & 1) + 4 * ((j >> 1) & 1) + 2 * (j >> 2);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int slot = slot0 + t, k = h * KQ + slot + 1;
        if (slot < KQ && k <= P) {
            const double f = c_neg_inv_k[k];
            dst[k] = make_double2(f * vr[t], f * vi[t]);
        }
    }
}

// Boxes split over several P2M items: sum the item partials in item order.
// One CTA per split row: kRedGroups groups of 64 threads stride over the
// pieces (coefficient k on thread k of a group), then the group partials are
// added in group order -- a fixed order, so results are run-to-run
// identical.  (Level-2 rows of a million-point tree have ~10^3 pieces; a
// serial walk per coefficient was latency bound.)
constexpr int kRedGroups = 8;

__global__ void __launch_bounds__(kRedGroups * 64)
p2m_reduce_kernel(const P2MSplit* splits, const double2* partial, int P, double2* mult) {
    __shared__ double2 part[kRedGroups][64];
    pdl_trigger();
    pdl_wait();
    const int n = P + 1;
    const P2MSplit b = splits[blockIdx.x];
    const int k = threadIdx.x & 63, g = threadIdx.x >> 6;
    double2 acc = make_double2(0.0, 0.0);
    if (k < n) {
#pragma unroll 4
        for (int t = g; t < b.count; t += kRedGroups) {
            const double2 v = partial[int64_t(b.first + t) * n + k];
            acc.x += v.x;
            acc.y += v.y;
        }
    }
    part[g][k] = acc;
    __syncthreads();
    if (g == 0 && k < n) {
        for (int i = 1; i < kRedGroups; ++i) {
            acc.x += part[i][k].x;
            acc.y += part[i][k].y;
        }
        mult[int64_t(b.row) * n + k] = acc;
    }
}

// ------------------------------------------------------------ M2M / L2L --
// Factorised shifts.  With the child centre at t = (+-1/4, +-1/4) parent
// sides, the reference operators (summation.cpp:170-197) are, up to
// diagonal factors, real binomial triangles:
//   M2M  b_l = t^l ( sum_{k=1..l} C(l-1,k-1) (2t)^-k a_k - a_0 / l ),  b_0 = a_0
//   L2L  b'_m = (2t)^-m sum_{l>=m} C(l,m) t^l b_l
// (|t| = 0.35, |2t| = 0.71: every factor stays within 1e+-23 at P = 55).
// Per parent the four children's (re, im) columns form exactly one DMMA
// n-tile: Y[n x 8] = B[n x P] X[P x 8] on the FP64 tensor cores, B (the
// binomial triangle, transposed) resident in smem, only the k-steps that
// meet the triangle issued.  A warp per parent: each lane builds its B
// fragment (scaled child or parent coefficient) in registers; the
// epilogue applies the output diagonal on the accumulators (a lane holds
// re and im of one (row, child)):
//   M2M: the four children are added in quadrant order (shuffles) and the
//        parent row written (one writer per row);
//   L2L: child_c[m] += b'_m (one writer per child element).
// One cooperative launch covers all levels (bottom-up / top-down) with a
// grid-wide barrier between them; cross-level reads use ld.global.cg.
// Flops per child: 2 P^2 (one triangle, re and im) vs the dense 8 (P+1)^2.
constexpr int kShiftWarps = 8;
constexpr int kMaxShiftLevels = 16;
constexpr int kM2LHS = 60;  // row stride of the transposed operator tiles (== 12 mod 16)

struct ShiftLevels {
    int nlev;                                 // levels processed, in order
    const int32_t* parents[kMaxShiftLevels];  // parent rows
    const int4* kids[kMaxShiftLevels];        // child rows per quadrant (-1: none)
    int64_t nparents[kMaxShiftLevels];
};

// Grid-wide barrier for a cooperative launch (all CTAs co-resident):
// monotonic arrival counter, zeroed by the previous kernel of the apply.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(count, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
            if (v < target) __nanosleep(64);
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ int quad(const int4& v, int c) {
    return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}

template <bool kUp, int MT>
__global__ void __launch_bounds__(kShiftWarps * 32)
shift_kernel(ShiftLevels lv, const double* bmat_t, const double2* tab_g, int P, int KP, double2* ex,
             unsigned* gbar) {
    extern __shared__ __align__(16) double smb[];
    const int n = P + 1;
    double* bs = smb;                                            // [KP][kM2LHS]
    double2* tpow = reinterpret_cast<double2*>(bs + KP * kM2LHS);  // [4][n]  t_c^j
    double2* tinv = tpow + 4 * n;                                // [4][n]  (2 t_c)^-j
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    for (int i = threadIdx.x; i < 8 * n; i += blockDim.x) tpow[i] = tab_g[i];
    __syncthreads();
    bulk_stage(bs, bmat_t, uint32_t(KP * kM2LHS) * 8u, &bar, 0);
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    const int cb = rq >> 1;    // child of this lane's B-fragment column
    const bool im = rq & 1;
    const int ce = lane & 3;   // child of this lane's accumulator columns
    const double* acol = bs + kq * kM2LHS + rq;
    unsigned target = 0;
    for (int li = 0; li < lv.nlev; ++li) {
        const int32_t* parents = lv.parents[li];
        const int4* kids = lv.kids[li];
        const int64_t np = lv.nparents[li];
        for (int64_t pi = int64_t(blockIdx.x) * kShiftWarps + warp; pi < np;
             pi += int64_t(gridDim.x) * kShiftWarps) {
            const int64_t prow = parents[pi];
            const int4 kd = kids[pi];
            const int kb = quad(kd, cb), kc = quad(kd, ce);
            double acc[MT][2];
#pragma unroll
            for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = 0.0;
            // B rows: M2M k = k4 + kq + 1 (x_k = (2t)^-k a_k of the child),
            //         L2L l = k4 + kq     (x_l = t^l b_l of the parent)
            const double2* src = kUp ? ex + int64_t(max(kb, 0)) * n : ex + prow * n;
            const double2* dtab = (kUp ? tinv : tpow) + cb * n;
            const int off = kUp ? 1 : 0;
            // all of this lane's coefficients in flight at once (KP <= 8 MT)
            double2 av[2 * MT];
#pragma unroll
            for (int j = 0; j < 2 * MT; ++j)
                av[j] = 4 * j < KP ? __ldcg(src + min(4 * j + kq + off, P)) : make_double2(0.0, 0.0);
            const double2 a0 = (kUp && kc >= 0) ? __ldcg(ex + int64_t(kc) * n) : make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 2 * MT; ++j) {
                const int k4 = 4 * j;
                if (k4 >= KP) break;
                const int k = k4 + kq + off;
                const double2 d = dtab[min(k, P)];
                const double2 a = av[j];
                const double v = im ? fma(a.x, d.y, a.y * d.x) : fma(a.x, d.x, -(a.y * d.y));
                const double bfr = (kb >= 0 && k <= P) ? v : 0.0;
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    // triangle: M2M rows 8i.. need k <= l; L2L rows 8i.. need l >= m
                    if (kUp ? (k4 < 8 * i + 8) : (k4 >= 8 * i))
                        dmma_884(acc[i][0], acc[i][1], acol[k4 * kM2LHS + 8 * i], bfr);
                }
            }
            if (kUp) {
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int l = 8 * i + rq;
                    double2 b = a0;
                    if (l > 0 && l <= P) {
                        const double inv_l = c_neg_inv_k[l];  // -1/l
                        b = cmul2(tpow[ce * n + l], make_double2(fma(inv_l, a0.x, acc[i][0]),
                                                                 fma(inv_l, a0.y, acc[i][1])));
                    }
                    // children in quadrant order (summation.cpp:257-267)
                    double2 sum = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const double bx = __shfl_sync(0xffffffffu, b.x, (lane & ~3) | c);
                        const double by = __shfl_sync(0xffffffffu, b.y, (lane & ~3) | c);
                        sum.x += bx;
                        sum.y += by;
                    }
                    if (ce == 0 && l <= P) ex[prow * n + l] = sum;
                }
            } else if (kc >= 0) {
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int m = 8 * i + rq;
                    if (m <= P) {
                        const double2 b = cmul2(tinv[ce * n + m], make_double2(acc[i][0], acc[i][1]));
                        double2* dst = ex + int64_t(kc) * n + m;
                        double2 d = __ldcg(dst);
                        d.x += b.x;
                        d.y += b.y;
                        *dst = d;
                    }
                }
            }
        }
        if (li + 1 < lv.nlev) grid_barrier(gbar, target);
    }
}

using ShiftKernel = void (*)(ShiftLevels, const double*, const double2*, int, int, double2*, unsigned*);

template <bool kUp>
ShiftKernel shift_kernel_for(int mt) {
    switch (mt) {
        case 2: return shift_kernel<kUp, 2>;
        case 3: return shift_kernel<kUp, 3>;
        case 4: return shift_kernel<kUp, 4>;
        case 5: return shift_kernel<kUp, 5>;
        case 6: return shift_kernel<kUp, 6>;
        default: return shift_kernel<kUp, 7>;
    }
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
// 2*pairs] (re and im columns).  Persistent CTAs keep H^T and the canonical
// offset power table c^-j (j <= P, 7 offsets up to the square's symmetry)
// resident in smem; two batch groups of six warps per CTA, each:
//   0. the NEXT batch's source rows arrive by 1-D TMA bulk copies
//      (cp.async.bulk, mbarrier completion) while this batch computes;
//   1. X build: warp per list entry, lane per coefficient;
//   2. GEMM on the FP64 tensor cores: mma.sync m8n8k4 f64 (DMMA), warp w
//      owns column tiles w, w+6, w+12, all row tiles in registers;
//   3. epilogue in two passes: b = D'(y ...) per (entry, l) in place, then
//      each target box sums its entries in list order and adds the monopole
//      shift qsum*log(s_l) (summation.cpp:297-301).
// Executed flops per pair: 4 P (P+1) for the GEMM + O(P), half the dense
// 8 (P+1)^2 of the reference matvec.
constexpr int kM2LCols = 2 * kM2LPairs;          // 108 used columns
static_assert((kM2LCols + 7) / 8 <= 14, "14 column tiles");
constexpr int kM2LXS = 116;                      // X/Y row stride (== 4 mod 16: conflict-free fragments)
constexpr int kM2LCanon = 7;                     // offsets up to the square's symmetry
constexpr int kM2LMaxMT = 7;                     // RP <= 56

// Offset powers through the symmetry of the square: every interaction offset
// d is u * conj^s(c) for a canonical c in {(2,0),(2,1),(2,2),(3,0),(3,1),
// (3,2),(3,3)} and u = i^m', so d^-j = i^(m j) conj^s(c^-j) (m = -m' mod 4).
// The table c^-j (7 x (P+1) complex, 5.7 KB at P=50) lives in smem; the
// conjugation and the quarter turn i^r are sign flips and a swap done on
// the integer words (no FP64 instructions).
__device__ __forceinline__ double2 turn(double2 v, int r, int sconj) {
    int xh = __double2hiint(v.x), xl = __double2loint(v.x);
    int yh = __double2hiint(v.y) ^ (sconj << 31), yl = __double2loint(v.y);
    const bool sw = r & 1;
    int ah = sw ? yh : xh, al = sw ? yl : xl;
    int bh = sw ? xh : yh, bl = sw ? xl : yl;
    ah ^= ((r + 1) & 2) << 30;  // new re negated for r = 1, 2
    bh ^= (r & 2) << 30;        // new im negated for r = 2, 3
    return make_double2(__hiloint2double(ah, al), __hiloint2double(bh, bl));
}

struct M2LStage {
    int32_t src[kM2LPairs];
    int32_t omap[kM2LPairs];
    int32_t oidx[kM2LPairs];
    int32_t ecount;
};



// The producer warp stages a batch in two steps, one batch apart: the list
// metadata into its ring slot (global loads whose latency then hides behind
// the previous batch's GEMM), and later the source rows by 1-D TMA bulk
// copies completing on the batch's mbarrier.
__device__ __forceinline__ void m2l_stage_meta(const M2LBatch& bt, const int32_t* esrc,
                                               const int32_t* eoidx, const int32_t* omap_s,
                                               M2LStage* stg, int lane) {
    for (int e = lane; e < bt.ecount; e += 32) {
        const int64_t g = int64_t(bt.efirst) + e;
        const int o = eoidx[g];
        stg->src[e] = esrc[g];
        stg->oidx[e] = o;
        stg->omap[e] = omap_s[o];
    }
    if (lane == 0) stg->ecount = bt.ecount;
    __syncwarp();
}

__device__ __forceinline__ void m2l_issue_rows(const M2LStage* stg, const double2* mult, int n,
                                               double2* raw, uint64_t* bar, int lane) {
    const int ecount = stg->ecount;
    if (lane == 0) mbar_arrive_expect_tx(bar, uint32_t(ecount) * uint32_t(n) * 16u);
    __syncwarp();
    for (int e = lane; e < ecount; e += 32)
        tma_load_1d(raw + e * n, mult + int64_t(stg->src[e]) * n, uint32_t(n) * 16u, bar);
}

// Factorised M2L (see the block comment above): per batch one dense real
// GEMM Y = H X on the FP64 tensor cores (mma.sync m8n8k4, DMMA: 256 FMA per
// warp instruction, measured 36.9 TFLOP/s on this B200 vs 34.2 for DFMA).
// Warp-specialised, one CTA per SM, pipelined over the CTA's batches:
//   warp 0      TMA producer: the source rows of batch i+2 are copied into
//               staging buffer i%2 as soon as batch i has consumed it;
//   warps 1-14  MMA: warp w owns column tile w-1 (entries 4(w-1) .. +3).
//               X is never materialised: each lane builds its B fragment
//               (-1)^k d^-k a_k straight from the staged row, and the
//               diagonal epilogue b_l = d^-l (y_l - a0/l) runs on the
//               accumulators in registers (a lane holds re and im of one
//               (l, entry)); b goes to the Y buffer i%2;
//   warps 15-18 reduction: per target box and l, the entries' b in list
//               order plus the monopole shift; frees Y buffer i%2.
// The MMA warps only wait for the Y buffer right before their register
// epilogue, so batch i+1's GEMM overlaps batch i's reduction.  One column
// tile per MMA warp keeps ~3 MMA warps per SM sub-partition for typical
// batches (measured: 2 tiles per warp was 14% slower on cfg2).
#ifndef VPG_M2L_TPW
#define VPG_M2L_TPW 1
#endif
constexpr int kWSTPW = VPG_M2L_TPW;          // column tiles per MMA warp
constexpr int kWSMMAWarps = 14 / kWSTPW;     // 14 column tiles
constexpr int kWSRedThreads = 128;
constexpr int kWSThreads = 32 * (1 + kWSMMAWarps) + kWSRedThreads;
#ifndef VPG_M2L_DEEP
#define VPG_M2L_DEEP 0
#endif
// source-row ring depth and Y buffers: 3 / 1 (rows of two batches ahead in
// flight, one Y buffer drained by the reduction during the next k-loop) or 2 / 2
constexpr int kM2LRaw = VPG_M2L_DEEP ? 3 : 2;
constexpr int kM2LYs = VPG_M2L_DEEP ? 1 : 2;
constexpr int kWSStages = 5;                 // batch metadata ring (kM2LRaw + 2 live batches)
#ifndef VPG_M2L_KUNROLL
#define VPG_M2L_KUNROLL 2
#endif
constexpr int kM2LKUnroll = VPG_M2L_KUNROLL;  // k-loop unroll of the MMA warps
// Timing ablations (tools/ab_m2l_abl.sh; wrong results, never in a shipped
// build): 1 no DMMA, 2 no B-fragment build, 4 no A-fragment loads, 8 no
// reduction sums, 16 no epilogue, 32 source rows fetched once only.
#ifndef VPG_M2L_ABL
#define VPG_M2L_ABL 0
#endif

// Ping-pong of the MMA warps' k-loops (VPG_M2L_PINGPONG, measured and left
// off: cfg2 M2L 0.203 -> 0.213 ms, cfg4 0.353 -> 0.364 ms).  The
// 14 MMA warps of a batch all run k-loop, register epilogue, k-loop, ... in
// lock step (the batch barriers keep them together), so the FP64 tensor pipe
// idles through every epilogue and every wait for the next rows: the timing
// ablations give 0.126 ms for the kernel without its DMMAs and 0.110 ms for
// the DMMAs alone against 0.203 ms together (cfg2).  With the token the
// warps of column tiles 0-6 and 7-13 take turns: one half runs its k-loop at
// the pipe's full rate (7 warps saturate it, tools/dmma_sweep.cu) while the
// other half does its epilogue, hands its rows back and waits for the next
// batch's.  Two named barriers pass the token (the CUTLASS ordered-sequence
// form): a half syncs on its own barrier before the k-loop and arrives on
// the other half's after it.  It did not pay: a half's 7 warps sit 2/2/2/1 on
// the four schedulers, each of which owns a quarter of the DMMA rate
// (tools/dmma_sweep.cu: 1 warp per SM 9.0 TFLOP/s, 4 warps 36.3, 7 warps
// 32.1, 14 warps 32.3), so a half's k-loop takes as long as half of the
// lock-step one and the hand-offs come on top.
// VPG_M2L_PREBUILD (also off: 0.203 -> 0.210 ms) builds all B fragments of a
// batch before a DMMA-only k-loop, after tools/dmma_with_dfma.cu showed that
// an FP64 CUDA-core instruction issued among DMMAs costs ~9 pipe cycles.
#ifndef VPG_M2L_PINGPONG
#define VPG_M2L_PINGPONG 0
#endif
#ifndef VPG_M2L_PREBUILD
#define VPG_M2L_PREBUILD 0
#endif
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MT, int NK>  // row tiles: RP / 8; k-steps KP / 4 when fixed at compile time (0: runtime KP)
__global__ void __launch_bounds__(kWSThreads, 1)
m2l_kernel(const M2LBatch* batches, int64_t nbatch, const int32_t* tbox,
           const int32_t* toff, const int32_t* esrc, const int32_t* eoidx,
           const double* h_t, const double2* canon_g, const int32_t* omap_g,
           const double2* logmd_g, const double2* mult, double2* loc, int P, int RP, int KP,
           double side) {
    extern __shared__ __align__(16) double smd[];
    const int n = P + 1;
    double* hs = smd;                                               // [KP][kM2LHS]
    double2* canon = reinterpret_cast<double2*>(hs + KP * kM2LHS);  // [7][n]
    double2* logmd = canon + kM2LCanon * n;                         // [49]
    int32_t* omap_s = reinterpret_cast<int32_t*>(logmd + 49);       // [49] (+pad)
    double2* raw0 = reinterpret_cast<double2*>(omap_s + 52);        // [kM2LRaw][kM2LPairs][n]
    double* yb0 = reinterpret_cast<double*>(raw0 + kM2LRaw * kM2LPairs * n);  // [kM2LYs][n][kM2LXS]
    double2* a0s0 = reinterpret_cast<double2*>(yb0 + kM2LYs * n * kM2LXS);    // [kM2LYs][kM2LPairs]
    M2LStage* stg = reinterpret_cast<M2LStage*>(a0s0 + kM2LYs * kM2LPairs);   // [kWSStages]
    __shared__ __align__(8) uint64_t bars[1 + 2 * kM2LRaw + 2 * kM2LYs];
    __shared__ double ninv[64];    // -1/l (the epilogue's per-lane rows; no divergent LDC)
    uint64_t* full = bars + 1;                 // [kM2LRaw] source rows landed (TMA tx count)
    uint64_t* rawfree = full + kM2LRaw;        // [kM2LRaw] rows consumed (MMA warps)
    uint64_t* ydone = rawfree + kM2LRaw;       // [kM2LYs] Y written (MMA warps)
    uint64_t* yfree = ydone + kM2LYs;          // [kM2LYs] Y consumed (reduction warps)

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        for (int j = 0; j < kM2LRaw; ++j) {
            mbar_init(&full[j], 1);
            mbar_init(&rawfree[j], 32 * kWSMMAWarps);
        }
        for (int j = 0; j < kM2LYs; ++j) {
            mbar_init(&ydone[j], 32 * kWSMMAWarps);
            mbar_init(&yfree[j], kWSRedThreads);
        }
    }
    for (int i = tid; i < kM2LCanon * n; i += blockDim.x) canon[i] = canon_g[i];
    for (int i = tid; i < 49; i += blockDim.x) {
        logmd[i] = logmd_g[i];
        omap_s[i] = omap_g[i];
    }
    for (int i = tid; i < 64; i += blockDim.x) ninv[i] = c_neg_inv_k[i];
    __syncthreads();
    bulk_stage(hs, h_t, uint32_t(KP * kM2LHS) * 8u, &bars[0], 0);
    __syncthreads();
    pdl_trigger();
    pdl_wait();

    const int64_t stride = gridDim.x;
    if (warp == 0) {
        // ------------------------------------------------- TMA producer
        // metadata of batches 0..R, rows of batches 0..R-1 (R = kM2LRaw);
        // then per consumed batch it: rows of it + R into its slot (metadata
        // already staged), metadata of it + R + 1
        for (int j = 0; j <= kM2LRaw; ++j) {
            const int64_t bi = blockIdx.x + j * stride;
            if (bi < nbatch) m2l_stage_meta(batches[bi], esrc, eoidx, omap_s, &stg[j % kWSStages], lane);
        }
        for (int j = 0; j < kM2LRaw; ++j)
            if (blockIdx.x + j * stride < nbatch)
                m2l_issue_rows(&stg[j % kWSStages], mult, n, raw0 + j * kM2LPairs * n, &full[j], lane);
        for (int it = 0;; ++it) {
            const int64_t bn = blockIdx.x + (it + kM2LRaw) * stride;
            if (bn >= nbatch) break;
            const int j = it % kM2LRaw;
            mbar_wait(&rawfree[j], uint32_t(it / kM2LRaw) & 1u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (VPG_M2L_ABL & 32) {
                if (lane == 0) mbar_arrive(&full[j]);
                continue;
            }
            m2l_issue_rows(&stg[(it + kM2LRaw) % kWSStages], mult, n, raw0 + j * kM2LPairs * n, &full[j], lane);
            const int64_t bm = bn + stride;
            if (bm < nbatch)
                m2l_stage_meta(batches[bm], esrc, eoidx, omap_s, &stg[(it + kM2LRaw + 1) % kWSStages], lane);
        }
    } else if (warp <= kWSMMAWarps) {
        // ---------------------------------------------------------- MMA
        const int w = warp - 1;
        const int kq = lane & 3, rq = lane >> 2;
        // the next batch's descriptor is loaded one batch ahead (its global
        // latency otherwise sits in front of every batch)
        M2LBatch bt_next{};
        if (blockIdx.x < nbatch) bt_next = batches[blockIdx.x];
        constexpr bool kPing = VPG_M2L_PINGPONG && kWSMMAWarps % 2 == 0;
        constexpr int kTokThreads = 32 * kWSMMAWarps;
        const int half = w >= kWSMMAWarps / 2;  // named barrier 1 + half: this half may run its k-loop
        if (kPing && half == 1 && blockIdx.x < nbatch) named_bar_arrive(1, kTokThreads);  // half 0 goes first
        for (int it = 0;; ++it) {
            const int64_t bi = blockIdx.x + it * stride;
            if (bi >= nbatch) break;
            const int j = it % kM2LRaw;
            const M2LBatch bt = bt_next;
            if (bi + stride < nbatch) bt_next = batches[bi + stride];
            const M2LStage& sg = stg[it % kWSStages];
            const double2* raw = raw0 + j * kM2LPairs * n;
            mbar_wait(&full[j], uint32_t(it / kM2LRaw) & 1u);
            if (kPing) named_bar_sync(1 + half, kTokThreads);
            // B-fragment sources: tile TPW w + t, column 8(TPW w + t) + rq ->
            // entry 4(TPW w + t) + rq/2, part rq&1; row k4 + kq <-> k = k4 + kq + 1
            const double2* brow[kWSTPW];
            const double2* bcan[kWSTPW];
            int bm2[kWSTPW], bsc[kWSTPW];
            bool blive[kWSTPW];
#pragma unroll
            for (int t = 0; t < kWSTPW; ++t) {
                const int p = 4 * (kWSTPW * w + t) + (rq >> 1);
                blive[t] = p < bt.ecount;
                const int pp = blive[t] ? p : 0;
                const int om = sg.omap[pp];
                brow[t] = raw + pp * n;
                bcan[t] = canon + (om & 7) * n;
                bsc[t] = (om >> 3) & 1;
                bm2[t] = ((om >> 4) & 3) + 2;
            }
            const bool im = rq & 1;
            double acc[MT][kWSTPW][2];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int t = 0; t < kWSTPW; ++t) acc[i][t][0] = acc[i][t][1] = 0.0;
            const double* hcol = hs + kq * kM2LHS + rq;
            if (4 * kWSTPW * w < bt.ecount) {  // warp-uniform: the warp's first tile is in use
                auto kstep = [&](int k4) {
                    double afr[MT];
#pragma unroll
                    for (int i = 0; i < MT; ++i)
                        afr[i] = (VPG_M2L_ABL & 4) ? double(k4 + i) : hcol[k4 * kM2LHS + 8 * i];
                    // branch-free B fragments (mma.sync needs a converged warp)
                    const int k = k4 + kq + 1;
                    const int kc = min(k, P);
                    double bfr[kWSTPW];
#pragma unroll
                    for (int t = 0; t < kWSTPW; ++t) {
                        if (VPG_M2L_ABL & 2) {
                            bfr[t] = double(kc);
                            continue;
                        }
                        const double2 a = brow[t][kc];
                        const double2 d = turn(bcan[t][kc], (bm2[t] * kc) & 3, bsc[t]);
                        const double v = im ? fma(a.x, d.y, a.y * d.x) : fma(a.x, d.x, -(a.y * d.y));
                        bfr[t] = (blive[t] && k <= P) ? v : 0.0;
                    }
#pragma unroll
                    for (int i = 0; i < MT; ++i)
#pragma unroll
                        for (int t = 0; t < kWSTPW; ++t) {
                            if (VPG_M2L_ABL & 1)
                                asm volatile("" : "+d"(acc[i][t][0]) : "d"(afr[i]), "d"(bfr[t]));
                            else
                                dmma_884(acc[i][t][0], acc[i][t][1], afr[i], bfr[t]);
                        }
                };
                if constexpr (NK > 0 && VPG_M2L_PREBUILD && kWSTPW == 1) {
                    // All B fragments of the batch first, then a k-loop of
                    // DMMAs only.  An FP64 CUDA-core instruction issued among
                    // DMMAs costs ~9 cycles of the shared FP64 pipe, not 2
                    // (tools/dmma_with_dfma.cu); the MMA warps wake together
                    // on the rows' barrier, so their builds coincide and the
                    // pipe then sees DMMAs only.  The empty volatile asm pins
                    // every fragment ahead of the first (volatile) DMMA.
                    double ball[NK];
#pragma unroll
                    for (int s4 = 0; s4 < NK; ++s4) {
                        const int k = 4 * s4 + kq + 1;
                        const int kc = min(k, P);
                        const double2 a = brow[0][kc];
                        const double2 d = turn(bcan[0][kc], (bm2[0] * kc) & 3, bsc[0]);
                        const double v = im ? fma(a.x, d.y, a.y * d.x) : fma(a.x, d.x, -(a.y * d.y));
                        ball[s4] = (blive[0] && k <= P) ? v : 0.0;
                    }
#pragma unroll
                    for (int s4 = 0; s4 < NK; ++s4) asm volatile("" : "+d"(ball[s4]));
#pragma unroll
                    for (int s4 = 0; s4 < NK; ++s4) {
                        double afr[MT];
#pragma unroll
                        for (int i = 0; i < MT; ++i) afr[i] = hcol[4 * s4 * kM2LHS + 8 * i];
#pragma unroll
                        for (int i = 0; i < MT; ++i) dmma_884(acc[i][0][0], acc[i][0][1], afr[i], ball[s4]);
                    }
                } else if constexpr (NK > 0) {
                    // the plan's k-step count is known at compile time: the
                    // whole k-loop unrolls (13 steps at P = 50: M2L -7%)
#pragma unroll
                    for (int s4 = 0; s4 < NK; ++s4) kstep(4 * s4);
                } else {
#pragma unroll kM2LKUnroll
                    for (int k4 = 0; k4 < KP; k4 += 4) kstep(k4);
                }
            }
            // the token goes to the other half (the last batch's second half keeps it)
            if (kPing && (half == 0 || bi + stride < nbatch)) named_bar_arrive(2 - half, kTokThreads);
            // register epilogue: lane holds (re, im) of row l = 8i + rq,
            // entry p = 4(2w+t) + kq.  The entries' a_0 are read before the
            // rows' slot is released to the producer.
            double2 a0r[kWSTPW];
#pragma unroll
            for (int t = 0; t < kWSTPW; ++t) {
                const int p = 4 * (kWSTPW * w + t) + kq;
                a0r[t] = p < bt.ecount ? raw[p * n] : make_double2(0.0, 0.0);
            }
            mbar_arrive(&rawfree[j]);
            const int ys = it % kM2LYs;
            if (it >= kM2LYs) mbar_wait(&yfree[ys], uint32_t(it / kM2LYs - 1) & 1u);
            double* yb = yb0 + ys * n * kM2LXS;
            double2* a0s = a0s0 + ys * kM2LPairs;
#pragma unroll
            for (int t = 0; t < kWSTPW; ++t) {
                const int p = 4 * (kWSTPW * w + t) + kq;
                if ((VPG_M2L_ABL & 16) && acc[0][t][0] != 1.2345) continue;
                if (p < bt.ecount) {
                    const double2 a0 = a0r[t];
                    const int om = sg.omap[p];
                    const int ci = om & 7, sc = (om >> 3) & 1, m = (om >> 4) & 3;
                    if (rq == 0) a0s[p] = a0;
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int l = 8 * i + rq;
                        if (l <= P) {
                            const double yr = acc[i][t][0], yi = acc[i][t][1];
                            double br, bim;
                            if (l == 0) {
                                const double2 lg = logmd[sg.oidx[p]];
                                br = yr + (lg.x * a0.x - lg.y * a0.y);
                                bim = yi + (lg.x * a0.y + lg.y * a0.x);
                            } else {
                                const double inv_l = ninv[l];  // -1/l
                                const double zr = fma(inv_l, a0.x, yr), zi = fma(inv_l, a0.y, yi);
                                const double2 dl = turn(canon[ci * n + l], (m * l) & 3, sc);
                                br = dl.x * zr - dl.y * zi;
                                bim = dl.x * zi + dl.y * zr;
                            }
                            *reinterpret_cast<double2*>(yb + l * kM2LXS + 2 * p) = make_double2(br, bim);
                        }
                    }
                }
            }
            mbar_arrive(&ydone[ys]);
        }
    } else {
        // ---------------------------------------------------- reduction
        const int rtid = tid - 32 * (1 + kWSMMAWarps);
        M2LBatch bt_next{};
        if (blockIdx.x < nbatch) bt_next = batches[blockIdx.x];
        for (int it = 0;; ++it) {
            const int64_t bi = blockIdx.x + it * stride;
            if (bi >= nbatch) break;
            const int ys = it % kM2LYs;
            const M2LBatch bt = bt_next;
            if (bi + stride < nbatch) bt_next = batches[bi + stride];
            const double* yb = yb0 + ys * n * kM2LXS;
            const double2* a0s = a0s0 + ys * kM2LPairs;
            mbar_wait(&ydone[ys], uint32_t(it / kM2LYs) & 1u);
            // per (target t, row l): entries summed in list order, plus the
            // monopole shift (summation.cpp:297-301)
            const double logs = log(side / double(1 << bt.level));
            const int l = rtid & 63;
            if (l <= P && !((VPG_M2L_ABL & 8) && it > 0))
                for (int t = rtid >> 6; t < bt.tcount; t += kWSRedThreads >> 6) {
                    const int64_t tg = int64_t(bt.tfirst) + t;
                    // the batch's entries are contiguous; its last box ends at the
                    // batch end (toff[tg + 1] may start a non-adjacent box: shards)
                    const int p0 = toff[tg] - bt.efirst;
                    const int p1 = t + 1 < bt.tcount ? toff[tg + 1] - bt.efirst : bt.ecount;
                    const double* yrow = yb + l * kM2LXS;
                    double sr = 0.0, si = 0.0, qsum = 0.0;
#pragma unroll 4
                    for (int p = p0; p < p1; ++p) {
                        sr += yrow[2 * p];
                        si += yrow[2 * p + 1];
                        if (l == 0) qsum += a0s[p].x;
                    }
                    if (l == 0) sr += qsum * logs;
                    loc[int64_t(tbox[tg]) * n + l] = make_double2(sr, si);
                }
            mbar_arrive(&yfree[ys]);
        }
    }
}

using M2LKernel = void (*)(const M2LBatch*, int64_t, const int32_t*, const int32_t*, const int32_t*,
                          const int32_t*, const double*, const double2*, const int32_t*, const double2*,
                          const double2*, double2*, int, int, int, double);

M2LKernel m2l_kernel_for(int mt, int kp) {
    // the sweep's tolerances 1e-12 / 1e-9 / 1e-6 give P = 50 / 39 / 27: KP = 52 / 40 / 28
    if (mt == 7 && kp == 52) return m2l_kernel<7, 13>;
    if (mt == 5 && kp == 40) return m2l_kernel<5, 10>;
    if (mt == 4 && kp == 28) return m2l_kernel<4, 7>;
    switch (mt) {
        case 2: return m2l_kernel<2, 0>;
        case 3: return m2l_kernel<3, 0>;
        case 4: return m2l_kernel<4, 0>;
        case 5: return m2l_kernel<5, 0>;
        case 6: return m2l_kernel<6, 0>;
        default: return m2l_kernel<7, 0>;
    }
}

// ------------------------------------------------------------------ L2P --
// Warp per near-field chunk (<= 64 targets of one leaf, two per lane):
// Horner of every local expansion on the leaf's L2P chain (the leaf after
// the L2L pass, summation.cpp:323-329; in the multilevel / hybrid downward
// passes also the ancestors whose locals were not pushed down), summed in
// chain order, pot = -(1/2pi) Re.  A row is staged through a per-warp smem
// slot with coalesced loads while the next row's coefficients are already
// in flight (register prefetch).  Zeroes the near-field tickets.
constexpr int kL2PWarps = 8;

__global__ void __launch_bounds__(kL2PWarps * 32)
l2p_kernel(const P2PChunk* chunks, int64_t nchunks, const int32_t* lrows, const double2* txy,
           const double2* loc, const int32_t* row_level, const int32_t* row_morton, int P,
           double x0, double y0, double side, const int32_t* tids, double* out, int assign) {
    __shared__ double2 rowbuf[kL2PWarps][64];
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = P + 1;
    double2* buf = rowbuf[warp];
    for (int64_t ci = int64_t(blockIdx.x) * kL2PWarps + warp; ci < nchunks;
         ci += int64_t(gridDim.x) * kL2PWarps) {
        const P2PChunk c = chunks[ci];
        if (c.part != 0) continue;  // split chunks: evaluated once
        const int myrow = lane < c.lcount ? lrows[c.lfirst + lane] : 0;
        const double2 t0 = txy[c.tbegin + min(lane, c.tcount - 1)];
        const double2 t1 = txy[c.tbegin + min(lane + 32, c.tcount - 1)];
        double s0 = 0.0, s1 = 0.0;
        int r = __shfl_sync(0xffffffffu, myrow, 0);
        double2 v0 = lane < n ? loc[int64_t(r) * n + lane] : make_double2(0.0, 0.0);
        double2 v1 = lane + 32 < n ? loc[int64_t(r) * n + lane + 32] : make_double2(0.0, 0.0);
        for (int q = 0; q < c.lcount; ++q) {
            buf[lane] = v0;
            buf[lane + 32] = v1;
            __syncwarp();
            const int rc = r;
            if (q + 1 < c.lcount) {  // prefetch the next row under this row's Horner
                r = __shfl_sync(0xffffffffu, myrow, q + 1);
                v0 = lane < n ? loc[int64_t(r) * n + lane] : make_double2(0.0, 0.0);
                v1 = lane + 32 < n ? loc[int64_t(r) * n + lane + 32] : make_double2(0.0, 0.0);
            }
            const double s = side / double(1 << row_level[rc]);
            double cx, cy;
            box_center(x0, y0, s, uint32_t(row_morton[rc]), cx, cy);
            const double inv_s = 1.0 / s;
            const double u0r = (t0.x - cx) * inv_s, u0i = (t0.y - cy) * inv_s;
            const double u1r = (t1.x - cx) * inv_s, u1i = (t1.y - cy) * inv_s;
            double ar = buf[P].x, ai = buf[P].y, br = ar, bi = ai;
            if (c.tcount > 32) {  // two targets per lane
                for (int k = P - 1; k >= 0; --k) {
                    const double2 a = buf[k];
                    const double nar = fma(ar, u0r, fma(-ai, u0i, a.x));
                    const double nai = fma(ar, u0i, fma(ai, u0r, a.y));
                    const double nbr = fma(br, u1r, fma(-bi, u1i, a.x));
                    const double nbi = fma(br, u1i, fma(bi, u1r, a.y));
                    ar = nar;
                    ai = nai;
                    br = nbr;
                    bi = nbi;
                }
            } else {  // warp-uniform: one target per lane, half the FP64 work
                for (int k = P - 1; k >= 0; --k) {
                    const double2 a = buf[k];
                    const double nar = fma(ar, u0r, fma(-ai, u0i, a.x));
                    const double nai = fma(ar, u0i, fma(ai, u0r, a.y));
                    ar = nar;
                    ai = nai;
                }
            }
            s0 += ar;
            s1 += br;
            __syncwarp();
        }
        // the near field is already in out (l2p_p2p_kernel): out += far
        // assign: the far field goes in first (the symmetric near field adds
        // on top later); otherwise it adds to the near field already there
        if (lane < c.tcount) {
            double& o = out[tids[c.tbegin + lane]];
            o = assign ? -kInv2Pi * s0 : o + -kInv2Pi * s0;
        }
        if (lane + 32 < c.tcount) {
            double& o = out[tids[c.tbegin + lane + 32]];
            o = assign ? -kInv2Pi * s1 : o + -kInv2Pi * s1;
        }
    }
}

// ------------------------------------------------------- near-field P2P --
// Persistent CTAs over target chunks (<= 64 targets of one leaf, sorted
// costliest first at plan time).  For a chunk, the 3x3 neighbour leaves
// (summation.cpp:330-334, reference order jy outer, jx inner) are flattened
// into one virtual source list -- lanes 0..8 own one neighbour range each, a
// shuffle scan gives the flat offsets -- and streamed through a per-warp
// smem slot kP2PBatch sources at a time (coalesced loads, broadcast reads).
// Every lane holds two targets, so one source fetch feeds two pairs.  The
// hot loop has no zero test: the pairs with r^2 zero or subnormal (only
// possible within the centre leaf) are listed once per plan
// (build_coincidences) and undone / redone with the reference skip rule in
// the chunk epilogue (coin_correction).
// Every task is one warp, drawn from a ticket counter (zeroed by
// l2p_kernel) in plan-time cost order:
//   split chunks (large neighbourhoods, see schedule_near_chunks): part i of
//   n takes the i-th contiguous share of the flat source list for all the
//   chunk's targets, writes 64 partial sums, and the last of the n warps to
//   finish (completion counter) adds the parts in part order -- no CTA
//   barriers, so no warp idles behind a slower sibling;
//   whole chunks (small leaves, cfg1/cfg2 interior): to keep lanes busy with
//   ~15-target leaves the warp splits into S = 32 / ceil(nT/2) groups taking
//   every S-th source, partials added in group order.
// Every sum has a fixed order, so results are run-to-run identical.  Output:
// far field (l2p_kernel) + near field, scattered to the original target
// order (summation.cpp:345).
// 16 warps x 1 CTA per SM, 4 sources per hot-loop trip (A/B with the truncated-index log:
// 8 x 2 / unroll 2 -> 16 x 1 / unroll 4: op_star near field 7.39 -> 7.13 ms, cfg2 0.195 -> 0.192 ms)
#ifndef VPG_P2P_WARPS
#define VPG_P2P_WARPS 16
#endif
constexpr int kP2PWarps = VPG_P2P_WARPS;
constexpr int kP2PBatch = 64;
constexpr int kP2PChunk = 64;
#ifndef VPG_P2P_MIN_BLOCKS
#define VPG_P2P_MIN_BLOCKS 1
#endif
constexpr int kP2PMinBlocks = VPG_P2P_MIN_BLOCKS;
#ifndef VPG_P2P_UNROLL
#define VPG_P2P_UNROLL 4
#endif
constexpr int kP2PUnroll = VPG_P2P_UNROLL;  // sources per hot-loop iteration

// The near sources of a chunk: up to kMaxNearRanges leaf ranges (the 3x3
// neighbourhood in uniform trees, the U list in adaptive ones) flattened
// into one virtual list.  Range starts and prefix offsets live in a per-warp
// smem slot; a flat index maps to its source by binary search.
struct NearList {
    int total;
    int nr;
    const int* pre;     // [nr] prefix offsets (smem)
    const int* st;      // [nr] first sorted source (smem)
};

__device__ __forceinline__ NearList near_list(const int2* ranges, int rfirst, int rcount, int rself,
                                              int lane, int* pre_s, int* st_s) {
    __syncwarp();
    int2 r0 = make_int2(0, 0), r1 = make_int2(0, 0);
    if (lane < rcount) r0 = ranges[rfirst + lane];
    if (lane + 32 < rcount) r1 = ranges[rfirst + lane + 32];
    int i0 = r0.y, i1 = r1.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v0 = __shfl_up_sync(0xffffffffu, i0, o);
        const int v1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= o) {
            i0 += v0;
            i1 += v1;
        }
    }
    const int tot0 = __shfl_sync(0xffffffffu, i0, 31);
    pre_s[lane] = i0 - r0.y;
    st_s[lane] = r0.x;
    pre_s[lane + 32] = tot0 + i1 - r1.y;
    st_s[lane + 32] = r1.x;
    NearList nl;
    nl.total = tot0 + __shfl_sync(0xffffffffu, i1, 31);
    nl.nr = rcount;
    __syncwarp();
    nl.pre = pre_s;
    nl.st = st_s;
    return nl;
}

// One batch [base, base+cnt) of the flat list, software-pipelined: the
// sources of batch b+1 are fetched (global -> registers) while batch b is
// evaluated from smem, so the L2 latency of the staging loads hides behind
// the pair loop (small leaves have only ~2-3 batches per chunk).
struct NearRegs {
    double2 xy[kP2PBatch / 32];
    double q[kP2PBatch / 32];
};

__device__ __forceinline__ void near_fetch(const NearList& nl, int base, int cnt, int lane,
                                           const double2* sxy, const double* q, NearRegs& r) {
#pragma unroll
    for (int h = 0; h < kP2PBatch / 32; ++h) {
        const int f = h * 32 + lane;
        if (f < cnt) {
            const int ff = base + f;
            // last range with pre <= ff (empty ranges share the next start)
            int lo = 0, hi = nl.nr - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (nl.pre[mid] <= ff) lo = mid; else hi = mid - 1;
            }
            const int src = nl.st[lo] + (ff - nl.pre[lo]);
            r.xy[h] = sxy[src];
            r.q[h] = q[src];
        }
    }
}

// evaluate (sources f == grp mod S) from the staged batch
__device__ __forceinline__ void near_batch(const NearRegs& r, int base, int cnt, int grp, int S,
                                           bool active, int lane, double2* mxy, double* mq,
                                           uint32_t tab_lane, const double (&tx)[2],
                                           const double (&ty)[2], LapAcc (&acc)[2]) {
    __syncwarp();
#pragma unroll
    for (int h = 0; h < kP2PBatch / 32; ++h) {
        const int f = h * 32 + lane;
        if (f < cnt) {
            mxy[f] = r.xy[h];
            mq[f] = r.q[h];
        }
    }
    __syncwarp();
    if (!active) return;
    int j = grp - base % S;
    if (j < 0) j += S;
#pragma unroll kP2PUnroll
    for (; j < cnt; j += S) {
        const double2 sp = mxy[j];
        const double qj = mq[j];
        lap_pair_fast(tx[0], ty[0], sp.x, sp.y, qj, tab_lane, acc[0]);
        lap_pair_fast(tx[1], ty[1], sp.x, sp.y, qj, tab_lane, acc[1]);
    }
}

// all batches of [f0, f1): fetch b+1 while b is evaluated
__device__ __forceinline__ void near_range(const NearList& nl, int f0, int f1, int grp, int S,
                                           bool active, int lane, const double2* sxy, const double* q,
                                           double2* mxy, double* mq, uint32_t tab_lane,
                                           const double (&tx)[2], const double (&ty)[2],
                                           LapAcc (&acc)[2]) {
    if (f0 >= f1) return;
    NearRegs r;
    near_fetch(nl, f0, min(kP2PBatch, f1 - f0), lane, sxy, q, r);
    for (int base = f0; base < f1; base += kP2PBatch) {
        const int cnt = min(kP2PBatch, f1 - base);
        NearRegs cur = r;
        if (base + kP2PBatch < f1)
            near_fetch(nl, base + kP2PBatch, min(kP2PBatch, f1 - base - kP2PBatch), lane, sxy, q, r);
        near_batch(cur, base, cnt, grp, S, active, lane, mxy, mq, tab_lane, tx, ty, acc);
    }
}

// The coincidence correction of one target (sorted index ti): the listed
// pairs undone and redone with the reference rule (lap_pair_fixup), as a
// separate sum added to the target's total.
template <class Tab>
__device__ __forceinline__ double coin_correction(const int32_t* coin_off, const int32_t* coin_src,
                                                  int64_t ti, double tx, double ty, const double2* sxy,
                                                  const double* q, Tab tab_lane) {
    const int k0 = coin_off[ti], k1 = coin_off[ti + 1];
    if (k0 == k1) return 0.0;
    LapAcc fix;
    for (int k = k0; k < k1; ++k) {
        const int j = coin_src[k];
        const double2 sp = sxy[j];
        lap_pair_fixup(tx, ty, sp.x, sp.y, q[j], tab_lane, fix);
    }
    return lap_total(fix);
}

static_assert(kLogTableSize * 16 <= kP2PWarps * kP2PBatch * 24, "table staging fits sbuf + qbuf");

__global__ void __launch_bounds__(kP2PWarps * 32, kP2PMinBlocks)
l2p_p2p_kernel(const P2PChunk* chunks, int64_t nchunks, const int2* ranges,
               const double2* sxy, const double* q, const double2* txy,
               const int32_t* tids, const int32_t* coin_off, const int32_t* coin_src,
               const double2* gtab, int* ticket, double* partial, int* pcount, double* out, int quota) {
    extern __shared__ double2 smp[];
    double2* tab = smp;                                                  // log table
    double2* sbuf = smp + kLogTableSize * kLogTableCopies;               // [warps][batch] xy
    double* qbuf = reinterpret_cast<double*>(sbuf + kP2PWarps * kP2PBatch);  // [warps][batch]
    int* rbuf = reinterpret_cast<int*>(qbuf + kP2PWarps * kP2PBatch);   // [warps][2][64]
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    // one bulk copy of the 257-entry table into the (still unused) source
    // slots, then replicate 8x (log_table_to_smem)
    bulk_stage(sbuf, gtab, uint32_t(kLogTableSize) * 16u, &bar, 0);
    log_table_to_smem(tab, sbuf);
    pdl_trigger();
    pdl_wait();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab_lane = log_table_lane_addr(tab, lane & (kLogTableCopies - 1));
    double2* mxy = sbuf + warp * kP2PBatch;
    double* mq = qbuf + warp * kP2PBatch;
    int* pre_s = rbuf + warp * 2 * kMaxNearRanges;
    int* st_s = pre_s + kMaxNearRanges;

    for (int done = 0; done < quota; ++done) {  // quota: tasks per warp before the CTA retires
        int k = 0;
        if (lane == 0) k = atomicAdd(&ticket[0], 1);
        const int64_t ch = __shfl_sync(0xffffffffu, k, 0);
        if (ch >= nchunks) break;
        const P2PChunk c = chunks[ch];
        const int nT = c.tcount;
        const NearList nl = near_list(ranges, c.rfirst, c.rcount, c.rself, lane, pre_s, st_s);
        if (c.nparts > 1) {
            // ---- one part of a split chunk: targets lane, lane + 32
            double tx[2], ty[2];
            LapAcc acc[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const double2 t = txy[c.tbegin + min(lane + 32 * u, nT - 1)];
                tx[u] = t.x;
                ty[u] = t.y;
            }
            const int f0 = int(int64_t(nl.total) * c.part / c.nparts);
            const int f1 = int(int64_t(nl.total) * (c.part + 1) / c.nparts);
            near_range(nl, f0, f1, 0, 1, true, lane, sxy, q, mxy, mq, tab_lane, tx, ty, acc);
            double* prow = partial + int64_t(c.pbase + c.part) * 64;
            prow[lane] = lap_total(acc[0]);
            prow[lane + 32] = lap_total(acc[1]);
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(&pcount[c.slot], 1) == c.nparts - 1;
            if (__shfl_sync(0xffffffffu, last, 0)) {
                // last finisher: add the parts in part order
                __threadfence();
                const double* pr = partial + int64_t(c.pbase) * 64;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int li = lane + 32 * u;
                    double sum = 0.0;
                    for (int i = 0; i < c.nparts; ++i) sum += __ldcg(pr + i * 64 + li);
                    if (li < nT) {
                        sum += coin_correction(coin_off, coin_src, c.tbegin + li, tx[u], ty[u], sxy, q,
                                               tab_lane);
                        out[tids[c.tbegin + li]] = -kInv4Pi * sum;
                    }
                }
            }
            continue;
        }
        // ---- a whole chunk: nTh target slots (two targets each), S source groups
        const int nTh = (nT + 1) >> 1;
        const int S = max(1, 32 / nTh);
        const int tl = lane % nTh;  // target slot: targets tl and tl + nTh
        const int grp = lane / nTh; // source group
        const bool active = grp < S;
        double tx[2], ty[2];
        LapAcc acc[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const double2 t = txy[c.tbegin + min(tl + nTh * u, nT - 1)];
            tx[u] = t.x;
            ty[u] = t.y;
        }
        near_range(nl, 0, nl.total, grp, S, active, lane, sxy, q, mxy, mq, tab_lane, tx, ty, acc);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            double v = active ? lap_total(acc[u]) : 0.0;
            // add the other groups' partials in group order
            for (int g2 = 1; g2 < S; ++g2) {
                const double w = __shfl_sync(0xffffffffu, v, min(31, tl + g2 * nTh));
                if (grp == 0) v += w;
            }
            const int li = tl + nTh * u;
            if (grp == 0 && li < nT) {
                v += coin_correction(coin_off, coin_src, c.tbegin + li, tx[u], ty[u], sxy, q, tab_lane);
                out[tids[c.tbegin + li]] = -kInv4Pi * v;
            }
        }
    }
}

// ------------------------------------------------- symmetric near field --
// (sym.cuh) with ln r^2 as the pair function
#ifndef VPG_SYM_LAP_WARPS
#define VPG_SYM_LAP_WARPS 12
#endif
#ifndef VPG_SYM_LAP_MINB
#define VPG_SYM_LAP_MINB 1
#endif
struct LapLogK {
    static constexpr int kSymWarps = VPG_SYM_LAP_WARPS, kSymMinB = VPG_SYM_LAP_MINB, kSymMaxR = kSymLapMaxR;
    __device__ __forceinline__ double operator()(double r2, uint32_t tab_lane) const { return lap_log(r2, tab_lane); }
};

// Per leaf (warp per leaf, persistent grid): matched targets add the leaf's
// slot partials in slot order plus the coincidence correction; unmatched
// targets sum their 3x3 near sources one-sided (lanes stride the flattened
// list, butterfly reduction); then the output scatter (out = near; L2P adds
// the far field).
constexpr int kFinWarps = 8;
constexpr size_t kFinScratch = size_t(kFinWarps) * 2 * kMaxNearRanges * sizeof(int) > size_t(kLogTableSize) * 16
                                   ? size_t(kFinWarps) * 2 * kMaxNearRanges * sizeof(int)
                                   : size_t(kLogTableSize) * 16;  // range slots, or the table's staging copy
constexpr size_t kFinSmem = size_t(kLogTableBytes) + kFinScratch;
// kTable = false (no unmatched targets, or the hybrid form): no smem table;
// the coincidence fix-ups read the global table (same bits), so the kernel
// runs at full occupancy -- the slot sums are latency-bound loads, and the
// kernel sits on the step's tail.
// kFar: the far field too -- the leaf's local expansion (plans whose leaves
// evaluate one row: the classical downward pass) is staged per warp and
// every target's Horner (l2p_kernel's arithmetic, same bits) runs under its
// slot loads, so the far field never makes the round trip through `out`
// (cfg4: l2p_kernel 0.10 ms + finalize 0.13 ms, one scattered write and one
// scattered read-modify-write of 4.2M doubles, become one kernel).
struct FarArgs {
    const int32_t* lrows;
    const double2* loc;
    const int32_t* row_level;
    const int32_t* row_morton;
    int P;
    double x0, y0, side;
};
template <bool kTable, bool kFar>
__global__ void __launch_bounds__(kFinWarps * 32)
sym_finalize_kernel(const SymLeaf* leaves, int64_t nleaves, const double* part, const int2* ranges,
                    const double2* sxy, const double* q, const double2* txy, const int32_t* tids,
                    const int32_t* coin_off, const int32_t* coin_src, const double2* gtab, double* out, int add,
                    FarArgs far) {
    extern __shared__ double2 smp[];
    __shared__ double2 rowbuf[kFar ? kFinWarps : 1][64];
    const bool coin = !(add & 4);  // 4: the slots hold exact sums (lattice.cu skips r^2 == 0 itself)
    add &= 3;
    double2* tab = smp;
    int* rbuf = reinterpret_cast<int*>(smp + kLogTableSize * kLogTableCopies);  // [warps][2][64]
    uint32_t tab_lane = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (kTable) {
        __shared__ __align__(8) uint64_t bar;
        if (threadIdx.x == 0) mbar_init(&bar, 1);
        __syncthreads();
        bulk_stage(rbuf, gtab, uint32_t(kLogTableSize) * 16u, &bar, 0);
        log_table_to_smem(tab, reinterpret_cast<const double2*>(rbuf));
        tab_lane = log_table_lane_addr(tab, lane & (kLogTableCopies - 1));
    }
    pdl_trigger();
    pdl_wait();
    if constexpr (kTable) __syncthreads();
    for (int64_t w = int64_t(blockIdx.x) * kFinWarps + warp; w < nleaves; w += int64_t(gridDim.x) * kFinWarps) {
        const SymLeaf lf = leaves[w];
        double fcx = 0.0, fcy = 0.0, finv = 0.0;
        if constexpr (kFar) {
            const int n = far.P + 1;
            const int r = far.lrows[lf.lfirst];
            __syncwarp();
            rowbuf[warp][lane] = lane < n ? far.loc[int64_t(r) * n + lane] : make_double2(0.0, 0.0);
            rowbuf[warp][lane + 32] = lane + 32 < n ? far.loc[int64_t(r) * n + lane + 32] : make_double2(0.0, 0.0);
            __syncwarp();
            const double s = far.side / double(1 << far.row_level[r]);
            box_center(far.x0, far.y0, s, uint32_t(far.row_morton[r]), fcx, fcy);
            finv = 1.0 / s;
        }
        // fused far field: the next target's coordinates, id and first slot are fetched under
        // the current target's Horner chain (the lane's targets are otherwise serial round trips)
        double2 tp_n = make_double2(0.0, 0.0);
        double a_n = 0.0;
        int id_n = 0;
        if constexpr (kFar) {
            if (lane < lf.n) {
                tp_n = txy[int64_t(lf.tgt) + lane];
                id_n = tids[int64_t(lf.tgt) + lane];
                a_n = __ldcg(part + lf.pbase + lane);
            }
        }
        for (int k = lane; k < lf.n; k += 32) {
            const int64_t t = int64_t(lf.tgt) + k;
            const double* pk = part + lf.pbase + k;
            double sum = 0.0;
            int sl = 0;
            double farv = 0.0;
            const double2 tp_c = tp_n;
            const double a_c = a_n;
            const int id_c = id_n;
            if constexpr (kFar) {  // issued ahead of the slot loads' use: the Horner chain hides them
                if (k + 32 < lf.n) {
                    tp_n = txy[t + 32];
                    id_n = tids[t + 32];
                    a_n = __ldcg(pk + 32);
                }
                const double2 tp = tp_c;
                const double2* buf = rowbuf[warp];
                const double ur = (tp.x - fcx) * finv, ui = (tp.y - fcy) * finv;
                double ar = buf[far.P].x, ai = buf[far.P].y;
                for (int kk = far.P - 1; kk >= 0; --kk) {
                    const double2 a = buf[kk];
                    const double nar = fma(ar, ur, fma(-ai, ui, a.x));
                    const double nai = fma(ar, ui, fma(ai, ur, a.y));
                    ar = nar;
                    ai = nai;
                }
                farv = -kInv2Pi * (0.0 + ar);
            }
            if constexpr (kFar) {  // slot 0 came with the prefetch
                if (lf.nslot > 0) {
                    sum += a_c;
                    sl = 1;
                }
                if (lf.nslot >= 8) {  // slots 1..7 in flight together
                    double a[7];
#pragma unroll
                    for (int u = 0; u < 7; ++u) a[u] = __ldcg(pk + int64_t(1 + u) * lf.n);
#pragma unroll
                    for (int u = 0; u < 7; ++u) sum += a[u];
                    sl = 8;
                }
            }
            for (; sl + 8 <= lf.nslot; sl += 8) {  // eight loads in flight, added in slot order
                double a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = __ldcg(pk + int64_t(sl + u) * lf.n);
#pragma unroll
                for (int u = 0; u < 8; ++u) sum += a[u];
            }
            if (sl + 4 <= lf.nslot) {
                double a[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = __ldcg(pk + int64_t(sl + u) * lf.n);
#pragma unroll
                for (int u = 0; u < 4; ++u) sum += a[u];
                sl += 4;
            }
            for (; sl < lf.nslot; ++sl) sum += __ldcg(pk + int64_t(sl) * lf.n);
            if (add == 1) {  // hybrid: the one-sided kernel wrote this target (coincidences included)
                out[tids[t]] += -kInv4Pi * sum;
                continue;
            }
            const double2 tp = kFar ? tp_c : txy[t];
            if (coin) {
                if constexpr (kTable) sum += coin_correction(coin_off, coin_src, t, tp.x, tp.y, sxy, q, tab_lane);
                else sum += coin_correction(coin_off, coin_src, t, tp.x, tp.y, sxy, q, gtab);
            }
            double& o = out[kFar ? id_c : tids[t]];
            if constexpr (kFar) {
                const double o0 = farv;
                o = o0 + -kInv4Pi * sum;
            } else {
                o = add == 2 ? o + -kInv4Pi * sum : -kInv4Pi * sum;  // 2: the far field is already there
            }
        }
        if constexpr (kTable) {
            if (add == 1 || lf.tgt + lf.n >= lf.t1) continue;
            int* pre_s = rbuf + warp * 2 * kMaxNearRanges;
            int* st_s = pre_s + kMaxNearRanges;
            const NearList nl = near_list(ranges, lf.rfirst, lf.rcount, 0, lane, pre_s, st_s);
            for (int t = lf.tgt + lf.n; t < lf.t1; ++t) {
                const double2 tp = txy[t];
                LapAcc acc;
                for (int ff = lane; ff < nl.total; ff += 32) {
                    int lo = 0, hi = nl.nr - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (nl.pre[mid] <= ff) lo = mid; else hi = mid - 1;
                    }
                    const int src = nl.st[lo] + (ff - nl.pre[lo]);
                    const double2 sp = sxy[src];
                    lap_pair_fast(tp.x, tp.y, sp.x, sp.y, q[src], tab_lane, acc);
                }
                double v = lap_total(acc);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) {
                    v += coin_correction(coin_off, coin_src, t, tp.x, tp.y, sxy, q, tab_lane);
                    double& o = out[tids[t]];
                    o = add == 2 ? o + -kInv4Pi * v : -kInv4Pi * v;
                }
            }
        }
    }
}

// ------------------------------------------------------ adaptive: M2P / P2L --
// M2P (W lists of adaptive trees): a box's multipole evaluated directly at a
// leaf's targets.  With a_0 = sum q and a_k = -(1/k) sum q w^k,
// w = (z - c)/s (P2M above), sum_j q_j log(t - z_j) = a_0 log(t - c)
// + sum_k a_k (s/(t - c))^k, so per target u = s/(t - c), Horner over k, plus
// a_0 log|t - c| (a_0 is real: real charges).  Warp per (leaf, 32 targets),
// W entries in list order, coefficients staged per warp in smem.
constexpr int kM2PWarps = 4;

__global__ void __launch_bounds__(kM2PWarps * 32)
m2p_kernel(const int4* work, int64_t nwork, const int32_t* wrows, const double2* txy,
           const double2* mult, const int32_t* row_level, const int32_t* row_morton, int P,
           double x0, double y0, double side, const int32_t* tids, double* out) {
    extern __shared__ double2 coef[];
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wi = int64_t(blockIdx.x) * kM2PWarps + warp;
    if (wi >= nwork) return;
    const int n = P + 1;
    double2* cw = coef + warp * n;
    const int4 w = work[wi];
    const int e = w.x + min(lane, w.y - 1);
    const double2 t = txy[e];
    double acc = 0.0;
    for (int k = 0; k < w.w; ++k) {
        const int r = wrows[w.z + k];
        __syncwarp();
        for (int i = lane; i < n; i += 32) cw[i] = mult[int64_t(r) * n + i];
        __syncwarp();
        const double s = side / double(1 << row_level[r]);
        double cx, cy;
        box_center(x0, y0, s, uint32_t(row_morton[r]), cx, cy);
        const double dx = t.x - cx, dy = t.y - cy;
        const double d2 = fma(dy, dy, dx * dx);
        const double inv = s / d2;
        const double ur = dx * inv, ui = -dy * inv;  // s / (t - c)
        double vr = cw[P].x, vi = cw[P].y;
        for (int j = P - 1; j >= 1; --j) {
            const double2 a = cw[j];
            const double nr = fma(vr, ur, fma(-vi, ui, a.x));
            const double ni = fma(vr, ui, fma(vi, ur, a.y));
            vr = nr;
            vi = ni;
        }
        const double re = vr * ur - vi * ui;  // times u once more: sum_{k>=1} a_k u^k
        acc += re + cw[0].x * 0.5 * log(d2);
    }
    if (lane < w.y) out[tids[e]] += -kInv2Pi * acc;
}

// P2L (X lists of adaptive trees): a coarser leaf's sources straight into a
// box's local expansion.  For |z - c| < |z_j - c|, log(z - z_j) =
// log(c - z_j) - sum_l (1/l) u^l v_j^l with u = (z - c)/s, v_j = s/(z_j - c):
// b_0 += q log|z_j - c| (only the real part is ever used), b_l += -q v^l / l.
// Warp per receiving box, the panel scheme of P2M (two lanes per source,
// half the powers each), X ranges in list order; loc += result (the box's
// only writer after M2L).
__global__ void __launch_bounds__(kP2MWarps * 32)
p2l_kernel(const int4* work, int64_t nwork, const int2* ranges, const double2* sxy,
           const double* q, const int32_t* row_level, const int32_t* row_morton, int P,
           double x0, double y0, double side, double2* loc) {
    extern __shared__ double2 panels[];
    pdl_trigger();
    pdl_wait();
    const int n = P + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wi = int64_t(blockIdx.x) * kP2MWarps + warp;
    if (wi >= nwork) return;
    const int ps = n | 1;  // odd row stride (see p2m_kernel)
    double2* panel = panels + warp * kP2MSrc * ps;
    const int4 w = work[wi];
    const int r = w.x;
    const double s = side / double(1 << row_level[r]);
    double cx, cy;
    box_center(x0, y0, s, uint32_t(row_morton[r]), cx, cy);
    const int j = lane & (kP2MSrc - 1), h = lane >> 4;
    const int kh = (P + 1) >> 1;
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    for (int ri = 0; ri < w.z; ++ri) {
        const int2 rg = ranges[w.y + ri];
        for (int base = rg.x; base < rg.x + rg.y; base += kP2MSrc) {
            const int cnt = min(kP2MSrc, rg.x + rg.y - base);
            if (j < cnt) {
                const double2 p = sxy[base + j];
                const double dx = p.x - cx, dy = p.y - cy;
                const double d2 = fma(dy, dy, dx * dx);
                const double inv = s / d2;
                const double vr = dx * inv, vi = -dy * inv;  // s / (z_j - c)
                const double qj = q[base + j];
                double2* row = panel + j * ps;
                double pr = qj, pi = 0.0;
                int k0 = 1, k1 = kh;
                if (h == 0) {
                    row[0] = make_double2(qj * 0.5 * log(d2), 0.0);
                } else {
                    double br = vr, bi = vi;
                    for (int e = kh; e; e >>= 1) {
                        if (e & 1) {
                            const double nr = pr * br - pi * bi;
                            pi = pr * bi + pi * br;
                            pr = nr;
                        }
                        const double sr = br * br - bi * bi;
                        bi = 2.0 * br * bi;
                        br = sr;
                    }
                    k0 = kh + 1;
                    k1 = P;
                }
                for (int k = k0; k <= k1; ++k) {
                    const double nr = pr * vr - pi * vi;
                    const double ni = pr * vi + pi * vr;
                    pr = nr;
                    pi = ni;
                    const double f = c_neg_inv_k[k];
                    row[k] = make_double2(f * pr, f * pi);
                }
            }
            __syncwarp();
            for (int t = 0; t < cnt; ++t) {
                if (lane <= P) {
                    const double2 v0 = panel[t * ps + lane];
                    acc0.x += v0.x;
                    acc0.y += v0.y;
                }
                if (lane + 32 <= P) {
                    const double2 v1 = panel[t * ps + lane + 32];
                    acc1.x += v1.x;
                    acc1.y += v1.y;
                }
            }
            __syncwarp();
        }
    }
    double2* dst = loc + int64_t(r) * n;
    if (lane <= P) {
        double2 v = dst[lane];
        v.x += acc0.x;
        v.y += acc0.y;
        dst[lane] = v;
    }
    if (lane + 32 <= P) {
        double2 v = dst[lane + 32];
        v.x += acc1.x;
        v.y += acc1.y;
        dst[lane + 32] = v;
    }
}

// Charges into leaf order; also zeroes the apply's counters: the two grid-
// barrier words of the shift passes, the near-field task ticket and the
// split-chunk completion counters.
__global__ void gather_q(const double* q, const int32_t* ids, int64_t n, double* qs, unsigned* gbar,
                         int* ticket, int* pcount, int64_t nslots) {
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e < 2) gbar[e] = 0u;
    if (e < 2) ticket[e] = 0;
    for (int64_t i = e; i < nslots; i += int64_t(gridDim.x) * blockDim.x) pcount[i] = 0;
    if (e < n) qs[e] = q[ids[e]];
}


}  // namespace

// ------------------------------------------------------------- operators --
// Plan time: the (target, near source) pairs whose r^2 -- computed exactly
// as in lap_pair_fast -- is zero or subnormal.  All of the chunk's near
// ranges are scanned (exact duplicates share a leaf, but a pair closer than
// 2^-511 can straddle a leaf edge).  Warp per chunk (first part of split
// chunks), lane per target; pass 1 counts (src == nullptr), pass 2 writes
// the sorted source indices at off.
__global__ void coin_scan_kernel(const P2PChunk* chunks, int64_t nchunks, const int2* ranges,
                                 const double2* sxy, const double2* txy, int32_t* cnt,
                                 const int32_t* off, int32_t* src) {
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nchunks) return;
    const P2PChunk c = chunks[w];
    if (c.nparts > 1 && c.part != 0) return;
    for (int u = lane; u < c.tcount; u += 32) {
        const int64_t ti = int64_t(c.tbegin) + u;
        const double2 t = txy[ti];
        int k = 0;
        const int base = src ? off[ti] : 0;
        for (int r = 0; r < c.rcount; ++r) {
            const int2 rg = ranges[c.rfirst + r];
            for (int j = 0; j < rg.y; ++j) {
                const double2 sp = sxy[rg.x + j];
                const double dx = t.x - sp.x, dy = t.y - sp.y;
                const double r2 = fma(dy, dy, dx * dx);
                if (__double2hiint(r2) < 0x00100000) {
                    if (src) src[base + k] = rg.x + j;
                    ++k;
                }
            }
        }
        if (!src) cnt[ti] = k;
    }
}

static void build_coincidences(Plan& pl) {
    const int64_t nt = pl.nt;
    pl.coin_off.alloc(size_t(nt) + 1);
    std::vector<int32_t> off(size_t(nt) + 1, 0);
    if (pl.n_p2p_chunks > 0 && nt > 0) {
        DBuf<int32_t> cnt;
        cnt.alloc(size_t(nt));
        VPG_CUDA(cudaMemset(cnt.p, 0, cnt.bytes()));
        const unsigned grid = unsigned(nblk(pl.n_p2p_chunks * 32, 256));
        coin_scan_kernel<<<grid, 256>>>(pl.p2p_chunks.p, pl.n_p2p_chunks, pl.near_ranges.p, pl.src_sorted.p,
                                        pl.tgt_sorted.p, cnt.p, nullptr, nullptr);
        VPG_CUDA(cudaGetLastError());
        VPG_CUDA(cudaMemcpy(off.data() + 1, cnt.p, cnt.bytes(), cudaMemcpyDeviceToHost));
        for (size_t i = 1; i < off.size(); ++i) off[i] += off[i - 1];
    }
    VPG_CUDA(cudaMemcpy(pl.coin_off.p, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice));
    pl.coin_src.alloc(size_t(std::max<int32_t>(off.back(), 1)));
    if (off.back() > 0) {
        const unsigned grid = unsigned(nblk(pl.n_p2p_chunks * 32, 256));
        coin_scan_kernel<<<grid, 256>>>(pl.p2p_chunks.p, pl.n_p2p_chunks, pl.near_ranges.p, pl.src_sorted.p,
                                        pl.tgt_sorted.p, nullptr, pl.coin_off.p, pl.coin_src.p);
        VPG_CUDA(cudaGetLastError());
    }
}

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

    // M2M / L2L, factorised (shift_kernel): binomial triangles, transposed
    // [k][row] with row stride kM2LHS, and per child c at (+-1/4, +-1/4) of
    // the parent side (bit 0 = x, summation.cpp:170-197) the diagonals
    // t_c^j and (2 t_c)^-j.
    pl.KP = ((P + 3) / 4) * 4;      // M2M (and M2L): k = 1..P
    pl.KPd = ((P + 1 + 3) / 4) * 4;  // L2L: l = 0..P
    std::vector<double> up_b(size_t(pl.KP) * kM2LHS, 0.0), dn_b(size_t(pl.KPd) * kM2LHS, 0.0);
    for (int l = 1; l <= P; ++l)
        for (int k = 1; k <= l; ++k) up_b[size_t(k - 1) * kM2LHS + l] = B(l - 1, k - 1);
    for (int l = 0; l <= P; ++l)
        for (int m = 0; m <= l; ++m) dn_b[size_t(l) * kM2LHS + m] = B(l, m);
    std::vector<cplx> stab(size_t(8) * n);
    for (int c = 0; c < 4; ++c) {
        const cplx t{(c & 1) ? 0.25 : -0.25, (c & 2) ? 0.25 : -0.25};
        const double m2 = 4.0 * (t.re * t.re + t.im * t.im);
        const cplx inv2t{2.0 * t.re / m2, -2.0 * t.im / m2};  // 1 / (2t)
        cplx tp{1.0, 0.0}, ti{1.0, 0.0};
        for (int j = 0; j <= P; ++j) {
            stab[size_t(c) * n + j] = tp;
            stab[size_t(4 + c) * n + j] = ti;
            tp = cmul(tp, t);
            ti = cmul(ti, inv2t);
        }
    }
    // M2L factors: H^T[k-1][l] = C(l+k-1, k-1); d^-j and log(-d) per offset
    // (summation.cpp:199-220).
    std::vector<double> ht(size_t(pl.KP) * kM2LHS, 0.0);
    for (int k = 1; k <= P; ++k)
        for (int l = 0; l <= P; ++l) ht[size_t(k - 1) * kM2LHS + l] = B(l + k - 1, k - 1);
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

    // canonical offsets and the map offset -> (canonical, conj, quarter turns)
    const int canon_xy[kM2LCanon][2] = {{2, 0}, {2, 1}, {2, 2}, {3, 0}, {3, 1}, {3, 2}, {3, 3}};
    std::vector<cplx> canon(size_t(kM2LCanon) * n, cplx{0, 0});
    for (int ci = 0; ci < kM2LCanon; ++ci) {
        const double cx = canon_xy[ci][0], cy = canon_xy[ci][1];
        const double m2 = cx * cx + cy * cy;
        const cplx cinv{cx / m2, -cy / m2};
        cplx* row = canon.data() + size_t(ci) * n;
        row[0] = {1.0, 0.0};
        for (int j = 1; j <= P; ++j) row[j] = cmul(row[j - 1], cinv);
    }
    std::vector<int32_t> omap(49, 0);
    for (int dy = -3; dy <= 3; ++dy)
        for (int dx = -3; dx <= 3; ++dx) {
            if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
            const int o = (dx + 3) + 7 * (dy + 3);
            bool found = false;
            for (int sc = 0; sc < 2 && !found; ++sc)
                for (int mq = 0; mq < 4 && !found; ++mq) {
                    // cand = conj^sc(d * i^-mq)
                    int ax = dx, ay = dy;
                    for (int r = 0; r < mq; ++r) {  // multiply by -i: (x, y) -> (y, -x)
                        const int t = ax;
                        ax = ay;
                        ay = -t;
                    }
                    if (sc) ay = -ay;
                    for (int ci = 0; ci < kM2LCanon; ++ci)
                        if (ax == canon_xy[ci][0] && ay == canon_xy[ci][1]) {
                            // d = i^mq conj^sc(c)  =>  d^-j = i^(-mq j) conj^sc(c^-j)
                            omap[size_t(o)] = ci | (sc << 3) | (((4 - mq) & 3) << 4);
                            found = true;
                            break;
                        }
                }
            if (!found) throw Error{VPG_ERR_CUDA, "offset symmetry map incomplete"};
        }

    cudaStream_t st = 0;
    pl.m2l_canon.alloc(canon.size());
    pl.m2l_omap.alloc(omap.size());
    VPG_CUDA(cudaMemcpyAsync(pl.m2l_canon.p, canon.data(), pl.m2l_canon.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.m2l_omap.p, omap.data(), pl.m2l_omap.bytes(), cudaMemcpyHostToDevice, st));
    pl.m2m_ops.alloc(up_b.size());
    pl.l2l_ops.alloc(dn_b.size());
    pl.shift_tab.alloc(stab.size());
    pl.h_t.alloc(ht.size());
    pl.dpow.alloc(dpw.size());
    pl.logmd.alloc(lg.size());
    VPG_CUDA(cudaMemcpyAsync(pl.m2m_ops.p, up_b.data(), pl.m2m_ops.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.l2l_ops.p, dn_b.data(), pl.l2l_ops.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaMemcpyAsync(pl.shift_tab.p, stab.data(), pl.shift_tab.bytes(), cudaMemcpyHostToDevice, st));
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
    pl.exp_total = pl.adaptive ? pl.n_rows * n : off;
    pl.exp_off_dev.alloc(pl.exp_off.size());
    VPG_CUDA(cudaMemcpy(pl.exp_off_dev.p, pl.exp_off.data(), pl.exp_off_dev.bytes(),
                        cudaMemcpyHostToDevice));

    for (int mt = 2; mt <= kM2LMaxMT; ++mt) smem_optin((const void*)m2l_kernel_for(mt, 0), 225 * 1024);
    smem_optin((const void*)m2l_kernel_for(pl.RP / 8, pl.KP), 225 * 1024);
    smem_optin((const void*)p2l_kernel, 100 * 1024);
    {
        // co-resident CTAs for the cooperative shift passes
        const size_t sm_up = sizeof(double) * size_t(pl.KP) * kM2LHS + sizeof(double2) * 8 * n;
        const size_t sm_dn = sizeof(double) * size_t(pl.KPd) * kM2LHS + sizeof(double2) * 8 * n;
        int pu = 0, pd = 0;
        VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pu, shift_kernel_for<true>(pl.RP / 8),
                                                               kShiftWarps * 32, sm_up));
        VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pd, shift_kernel_for<false>(pl.RP / 8),
                                                               kShiftWarps * 32, sm_dn));
        pl.shift_grid = std::max(1, std::min(pu, pd)) * pl.sm_count;
    }
    smem_optin((const void*)l2p_p2p_kernel, kLogTableBytes + 48 * 1024);
    smem_optin((const void*)p2p_sym_kernel<LapLogK>, int(sym_smem<LapLogK>()));
    smem_optin((const void*)sym_finalize_kernel<true, false>, int(kFinSmem));
    build_coincidences(pl);
    pl.coin_ready = true;
    if (!pl.adaptive) build_sym_near(pl, pl.shard_lb, pl.shard_le);
}

// ----------------------------------------------------------------- apply --
// Per-apply scratch of the Laplace FMM, carved from one block: sorted
// charges, mult / loc rows, far-field potentials, task counters (+ grid
// barrier words), split-chunk partials and counters, P2M split partials.
namespace {
size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

size_t laplace_work_bytes(const Plan& pl) {
    const size_t n = size_t(pl.P + 1);
    return al256(sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1))) +
           2 * al256(sizeof(double2) * size_t(std::max<int64_t>(pl.exp_total, 1))) +
           al256(sizeof(double) * size_t(std::max<int64_t>(pl.nt, 1))) + al256(sizeof(int) * 32) +
           al256(sizeof(double) * 64 * size_t(std::max<int64_t>(pl.n_p2p_parts, 1))) +
           al256(sizeof(int) * size_t(std::max<int64_t>(pl.n_p2p_heavy, 1))) +
           al256(sizeof(double2) * n * size_t(pl.n_p2m_splits > 0 ? pl.n_p2m_items : 1)) +
           (pl.sym ? al256(sizeof(double) * size_t(std::max<int64_t>(pl.sym_nparts, 1))) : 0);
}

LaplaceWork laplace_work_at(const Plan& pl, void* base) {
    const size_t n = size_t(pl.P + 1);
    char* p = static_cast<char*>(base);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += al256(bytes);
        return r;
    };
    LaplaceWork w;
    w.qs = reinterpret_cast<double*>(take(sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1))));
    w.mult = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(std::max<int64_t>(pl.exp_total, 1))));
    w.loc = reinterpret_cast<double2*>(take(sizeof(double2) * size_t(std::max<int64_t>(pl.exp_total, 1))));
    w.pot_far = reinterpret_cast<double*>(take(sizeof(double) * size_t(std::max<int64_t>(pl.nt, 1))));
    w.ticket = reinterpret_cast<int*>(take(sizeof(int) * 32));
    w.partial_p2p = reinterpret_cast<double*>(take(sizeof(double) * 64 * size_t(std::max<int64_t>(pl.n_p2p_parts, 1))));
    w.pcount = reinterpret_cast<int*>(take(sizeof(int) * size_t(std::max<int64_t>(pl.n_p2p_heavy, 1))));
    w.p2m_partial = reinterpret_cast<double2*>(take(sizeof(double2) * n * size_t(pl.n_p2m_splits > 0 ? pl.n_p2m_items : 1)));
    w.sym_part = pl.sym ? reinterpret_cast<double*>(take(sizeof(double) * size_t(std::max<int64_t>(pl.sym_nparts, 1))))
                        : nullptr;
    return w;
}

void laplace_apply(const Plan& pl, const double* q_dev, double* out_dev,
                   cudaStream_t st, cudaEvent_t* ev, int64_t& launches) {
    void* base = nullptr;
    VPG_CUDA(cudaMallocAsync(&base, laplace_work_bytes(pl), st));
    struct Free {
        void* p;
        cudaStream_t s;
        ~Free() {
            if (p) cudaFreeAsync(p, s);
        }
    } fr{base, st};
    laplace_issue(pl, q_dev, out_dev, laplace_work_at(pl, base), st, ev, launches, nullptr, nullptr, nullptr,
                  nullptr);
}

// The kernels of one Laplace apply, in stream order, on a given workspace
// (no allocation: the sequence can be captured into a CUDA graph).
//   With a side stream (graph capture) the near field runs concurrently
// with the whole far-field chain: gather -> [near field (side)] -> P2M ->
// M2M -> M2L -> P2L -> L2L -> join -> L2P (out += far) -> M2P (out += W).
// Without one, the same kernels run in one stream with the near field right
// before L2P.  out = near + far either way (one fixed order).
void laplace_issue(const Plan& pl, const double* q_dev, double* out_dev, const LaplaceWork& w,
                   cudaStream_t st, cudaEvent_t* ev, int64_t& launches, cudaStream_t side,
                   cudaEvent_t fork, cudaEvent_t join, cudaEvent_t far_done) {
    const int P = pl.P, n = P + 1, L = pl.L;
    auto mark = [&](int i) {
        if (ev) VPG_CUDA(cudaEventRecord(ev[i], st));
    };
    double* qs = w.qs;
    double2* mult = w.mult;
    double2* loc = w.loc;
    int* ticket = w.ticket;
    double* partial_p2p = w.partial_p2p;
    int* pcount = w.pcount;
    unsigned* gbar = reinterpret_cast<unsigned*>(ticket) + 8;  // grid barriers of the shift passes

    auto one_sided = [&](cudaStream_t s, const P2PChunk* nchunks, int64_t nnear, const int2* nranges) {
        if (nnear == 0) return;
        const size_t smem = size_t(kLogTableBytes) +
                            (sizeof(double2) + sizeof(double)) * kP2PBatch * kP2PWarps +
                            sizeof(int) * 2 * kMaxNearRanges * kP2PWarps;
        int per_sm = 1;
        VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l2p_p2p_kernel, kP2PWarps * 32, smem));
        const int64_t want = (nnear + kP2PWarps - 1) / kP2PWarps;
        int64_t cap = int64_t(pl.sm_count) * std::max(per_sm, 1);
        static const int pct = [] {
            const char* v = std::getenv("VPG_P2P_SIDE_PCT");
            return v ? std::atoi(v) : 100;
        }();
        if (s != st && pct > 0 && pct < 100) cap = std::max<int64_t>(1, cap * pct / 100);
        static const int quota = [] {
            const char* v = std::getenv("VPG_P2P_QUOTA");
            return v ? std::max(1, std::atoi(v)) : 0;
        }();
        unsigned grid = unsigned(std::min<int64_t>(want, cap));
        if (quota > 0 && s != st) grid = unsigned(std::max<int64_t>(1, (want + quota - 1) / quota));
        launch_pdl(l2p_p2p_kernel, dim3(grid), dim3(kP2PWarps * 32), smem, s, nchunks, nnear,
                   nranges, (const double2*)pl.src_sorted.p, (const double*)qs,
                   (const double2*)pl.tgt_sorted.p, (const int32_t*)pl.tgt_ids.p, pl.coin_off.p,
                   pl.coin_src.p, lap_log_table_dev(), ticket, partial_p2p, pcount, out_dev,
                   (quota > 0 && s != st) ? quota : INT32_MAX);
        ++launches;
    };

    // Symmetric near field on the side stream: the far field's L2P writes out
    // = far concurrently (main stream) and the finalize adds the near field
    // after it, so L2P leaves the step's tail (addition order far + near gives
    // the same bits as near + far)
    const bool far_first = side && far_done && pl.sym && !pl.sym_hybrid && pl.n_sym_leaves > 0;
    auto sym_finalize = [&](cudaStream_t s, int mode) {
        // the table variant only for unmatched targets summed one-sided here
        const bool table = pl.sym_unmatched && mode != 1;
        const int kmode = mode | (pl.lat ? 4 : 0);
        const auto fk = mode == 3 ? sym_finalize_kernel<false, true>
                                  : table ? sym_finalize_kernel<true, false> : sym_finalize_kernel<false, false>;
        const size_t fsmem = table ? kFinSmem : 0;
        int per_sm = 1;
        VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk, kFinWarps * 32, fsmem));
        const unsigned fgrid = unsigned(std::min<int64_t>(nblk(pl.n_sym_leaves, kFinWarps),
                                                          int64_t(pl.sm_count) * std::max(per_sm, 1)));
        launch_pdl(fk, dim3(fgrid), dim3(kFinWarps * 32), fsmem, s,
                   (const SymLeaf*)pl.sym_leaves.p, pl.n_sym_leaves, (const double*)w.sym_part,
                   (const int2*)pl.near_ranges.p, (const double2*)pl.src_sorted.p,
                   (const double*)qs, (const double2*)pl.tgt_sorted.p, (const int32_t*)pl.tgt_ids.p,
                   (const int32_t*)pl.coin_off.p, (const int32_t*)pl.coin_src.p, lap_log_table_dev(),
                   out_dev, kmode,
                   FarArgs{(const int32_t*)pl.l2p_rows.p, (const double2*)loc, (const int32_t*)pl.row_level.p,
                           (const int32_t*)pl.row_morton.p, P, pl.x0, pl.y0, pl.side});
        ++launches;
    };
    auto near_field = [&](cudaStream_t s) {
        if (pl.sym) {
            if (pl.lat) {  // translation-invariant leaves: dense GEMMs on the tensor cores (lattice.cu)
                lattice_near_issue(pl, qs, w.sym_part, s);
                ++launches;
            }
            if (pl.n_sym_tasks > 0) {
                int per_sm = 1;
                constexpr int kSymWarps = SymShape<LapLogK>::kWarps;
                constexpr size_t kSymSmem = sym_smem<LapLogK>();
                VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p2p_sym_kernel<LapLogK>, kSymWarps * 32,
                                                                       kSymSmem));
                const int64_t want = (pl.n_sym_tasks + kSymWarps - 1) / kSymWarps;
                const unsigned grid = unsigned(std::min<int64_t>(want, int64_t(pl.sm_count) * std::max(per_sm, 1)));
                launch_pdl(p2p_sym_kernel<LapLogK>, dim3(grid), dim3(kSymWarps * 32), kSymSmem, s, LapLogK{},
                           (const SymTask*)pl.sym_tasks.p, pl.n_sym_tasks, (const SymRange*)pl.sym_ranges.p,
                           (const double2*)pl.src_sorted.p, (const double*)qs, lap_log_table_dev(), ticket,
                           w.sym_part);
                ++launches;
            }
            if (pl.sym_hybrid) one_sided(s, pl.hyb_chunks.p, pl.n_hyb_chunks, pl.hyb_ranges.p);
            if (pl.n_sym_leaves > 0 && !far_first) sym_finalize(s, pl.sym_hybrid ? 1 : 0);
            return;  // unmatched targets: sym_finalize_kernel (full) or the one-sided pass (hybrid)
        }
        one_sided(s, pl.p2p_chunks.p, pl.n_p2p_chunks, pl.near_ranges.p);
    };
    mark(0);
    gather_q<<<nblk(std::max<int64_t>(pl.ns, pl.n_p2p_heavy), 256), 256, 0, st>>>(
        q_dev, pl.src_ids.p, pl.ns, qs, gbar, ticket, pcount, pl.n_p2p_heavy);
    VPG_LAUNCH_CHECK();
    ++launches;
    if (side) {
        VPG_CUDA(cudaEventRecord(fork, st));
        VPG_CUDA(cudaStreamWaitEvent(side, fork, 0));
        near_field(side);
        if (!far_first) VPG_CUDA(cudaEventRecord(join, side));
    }
    mark(1);

    double2* partial = w.p2m_partial;
    if (pl.lat && pl.lat_p2m && pl.n_p2m_items > 0) {  // lattice plans: power sums by one GEMM + per-leaf shift
        lattice_p2m_issue(pl, qs, w.sym_part + pl.lat_near_parts, mult, st);
        launches += 2;
    } else if (pl.n_p2m_items > 0) {
        auto p2m = [&](auto kern) {
            launch_pdl(kern, dim3(nblk(pl.n_p2m_items, kP2MWarps)), dim3(kP2MWarps * 32), 0, st,
                       (const P2MItem*)pl.p2m_items.p, pl.n_p2m_items, (const double2*)pl.src_sorted.p,
                       (const double*)qs, P, pl.x0, pl.y0, pl.side, mult, partial);
        };
        const int kq = (P + 3) / 4;  // powers per lane quarter
        if (kq <= 7) p2m(p2m_kernel<7>);
        else if (kq <= 10) p2m(p2m_kernel<10>);
        else if (kq <= 13) p2m(p2m_kernel<13>);
        else p2m(p2m_kernel<16>);
        ++launches;
    }
    if (pl.n_p2m_splits > 0) {
        launch_pdl(p2m_reduce_kernel, dim3(unsigned(pl.n_p2m_splits)), dim3(kRedGroups * 64), 0, st,
                   (const P2MSplit*)pl.p2m_splits.p, (const double2*)partial, P, mult);
        ++launches;
    }
    mark(2);
    {
        // M2M, bottom-up (summation.cpp:257-267)
        ShiftLevels lv{};
        for (int l = L - 1; l >= 2; --l) {
            const int64_t np = pl.m2m_count[size_t(l)];
            if (!np) continue;
            lv.parents[lv.nlev] = pl.updown_boxes.p + pl.m2m_first[size_t(l)];
            lv.kids[lv.nlev] = pl.updown_kids.p + pl.m2m_first[size_t(l)];
            lv.nparents[lv.nlev] = np;
            ++lv.nlev;
        }
        if (lv.nlev) {
            const size_t smem = sizeof(double) * size_t(pl.KP) * kM2LHS + sizeof(double2) * 8 * n;
            launch_coop(shift_kernel_for<true>(pl.RP / 8), pl.shift_grid, dim3(kShiftWarps * 32), smem, st, lv,
                        (const double*)pl.m2m_ops.p, (const double2*)pl.shift_tab.p, P, pl.KP, mult, gbar + 0);
            ++launches;
        }
    }
    mark(3);
    if (pl.n_gt_tiles > 0 && pl.n_m2l_batches > 0) {  // uniform tree: by offset (m2lgrid.cu), same bits
        m2l_grid_issue(pl, (const double2*)mult, loc, st);
        ++launches;
    } else if (pl.n_m2l_batches > 0) {
        const size_t smem = sizeof(double) * size_t(pl.KP) * kM2LHS +
                            sizeof(double2) * (size_t(kM2LCanon) * n + 49) + sizeof(int32_t) * 52 +
                            kM2LRaw * sizeof(double2) * size_t(kM2LPairs) * n +
                            kM2LYs * (sizeof(double2) * kM2LPairs + sizeof(double) * size_t(n) * kM2LXS) +
                            kWSStages * sizeof(M2LStage);
        const unsigned grid = unsigned(std::min<int64_t>(pl.n_m2l_batches, int64_t(pl.sm_count)));
        void (*kern)(const M2LBatch*, int64_t, const int32_t*, const int32_t*, const int32_t*,
                     const int32_t*, const double*, const double2*, const int32_t*, const double2*,
                     const double2*, double2*, int, int, int, double) = m2l_kernel_for(pl.RP / 8, pl.KP);
        launch_pdl(kern, dim3(grid), dim3(kWSThreads), smem, st,
                   (const M2LBatch*)pl.m2l_batches.p, pl.n_m2l_batches, (const int32_t*)pl.m2l_tbox.p,
                   (const int32_t*)pl.m2l_toff.p, (const int32_t*)pl.m2l_src.p,
                   (const int32_t*)pl.m2l_oidx.p, (const double*)pl.h_t.p,
                   (const double2*)pl.m2l_canon.p, (const int32_t*)pl.m2l_omap.p,
                   (const double2*)pl.logmd.p, (const double2*)mult, loc, P, pl.RP, pl.KP, pl.side);
        ++launches;
    }
    if (pl.n_p2l_work > 0) {
        launch_pdl(p2l_kernel, dim3(nblk(pl.n_p2l_work, kP2MWarps)), dim3(kP2MWarps * 32),
                   size_t(kP2MWarps) * kP2MSrc * (n | 1) * sizeof(double2), st, (const int4*)pl.p2l_work.p,
                   pl.n_p2l_work, (const int2*)pl.p2l_ranges.p, (const double2*)pl.src_sorted.p,
                   (const double*)qs, (const int32_t*)pl.row_level.p, (const int32_t*)pl.row_morton.p, P,
                   pl.x0, pl.y0, pl.side, loc);
        ++launches;
    }
    mark(4);
    {
        // L2L, top-down (summation.cpp:305-312)
        ShiftLevels lv{};
        for (int l = 2; l < L; ++l) {
            const int64_t np = pl.l2l_count[size_t(l)];
            if (!np) continue;
            lv.parents[lv.nlev] = pl.updown_boxes.p + pl.l2l_first[size_t(l)];
            lv.kids[lv.nlev] = pl.updown_kids.p + pl.l2l_first[size_t(l)];
            lv.nparents[lv.nlev] = np;
            ++lv.nlev;
        }
        if (lv.nlev) {
            const size_t smem = sizeof(double) * size_t(pl.KPd) * kM2LHS + sizeof(double2) * 8 * n;
            launch_coop(shift_kernel_for<false>(pl.RP / 8), pl.shift_grid, dim3(kShiftWarps * 32), smem, st, lv,
                        (const double*)pl.l2l_ops.p, (const double2*)pl.shift_tab.p, P, pl.KPd, loc, gbar + 1);
            ++launches;
        }
    }
    mark(5);
    if (!far_first) {
        if (side) VPG_CUDA(cudaStreamWaitEvent(st, join, 0));
        else near_field(st);
    }
    // symmetric plans whose leaves evaluate one local expansion: the finalize does the L2P too
    static const bool fuse_env = !(std::getenv("VPG_FUSE_L2P") && std::atoi(std::getenv("VPG_FUSE_L2P")) == 0);
    const bool fused_far = far_first && fuse_env && pl.sym_l2p_single && !pl.sym_unmatched;
    if (pl.n_p2p_chunks > 0 && !fused_far) {
        const int64_t want = (pl.n_p2p_chunks + kL2PWarps - 1) / kL2PWarps;
        const unsigned grid = unsigned(std::min<int64_t>(want, int64_t(pl.sm_count) * 8));
        launch_pdl(l2p_kernel, dim3(grid), dim3(kL2PWarps * 32), 0, st, (const P2PChunk*)pl.p2p_chunks.p,
                   pl.n_p2p_chunks, (const int32_t*)pl.l2p_rows.p, (const double2*)pl.tgt_sorted.p,
                   (const double2*)loc, (const int32_t*)pl.row_level.p, (const int32_t*)pl.row_morton.p, P,
                   pl.x0, pl.y0, pl.side, (const int32_t*)pl.tgt_ids.p, out_dev, far_first ? 1 : 0);
        ++launches;
    }
    if (far_first) {
        VPG_CUDA(cudaEventRecord(far_done, st));
        VPG_CUDA(cudaStreamWaitEvent(side, far_done, 0));
        sym_finalize(side, fused_far ? 3 : 2);
        VPG_CUDA(cudaEventRecord(join, side));
        VPG_CUDA(cudaStreamWaitEvent(st, join, 0));
    }
    if (pl.n_m2p_work > 0) {
        launch_pdl(m2p_kernel, dim3(nblk(pl.n_m2p_work, kM2PWarps)), dim3(kM2PWarps * 32),
                   size_t(kM2PWarps) * n * sizeof(double2), st, (const int4*)pl.m2p_work.p, pl.n_m2p_work,
                   (const int32_t*)pl.m2p_rows.p, (const double2*)pl.tgt_sorted.p, (const double2*)mult,
                   (const int32_t*)pl.row_level.p, (const int32_t*)pl.row_morton.p, P, pl.x0, pl.y0,
                   pl.side, (const int32_t*)pl.tgt_ids.p, out_dev);
        ++launches;
    }
    mark(6);
}

}  // namespace vpg
