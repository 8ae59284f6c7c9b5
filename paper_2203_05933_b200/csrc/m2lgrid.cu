// m2lgrid.cu -- M2L of uniform trees, batched by OFFSET instead of by target box.
//
// On a uniform tree every target box of one level and one position in its
// parent (four classes) has the same 27 interaction offsets in the same list
// order (summation.cpp:269-296: parent neighbours qy, qx, children c; only
// domain edges and empty boxes drop entries).  m2l_kernel (fmm.cu) batches
// the list entries of two target boxes; here a CTA takes 32 target boxes of
// one class and walks the class's 27 offsets: per offset one real GEMM
//   T[56 x 64] = H[56 x 52] . X_o[52 x 64],   X_o = (-1)^k d_o^-k a_k(box + o)
// (re and im columns of the 32 source boxes, zeros where the neighbour is
// missing) on the FP64 tensor cores, then the diagonal epilogue
// b = d_o^-l (T - a_0 / l) ON THE ACCUMULATORS, added to running sums that
// stay in registers over all 27 offsets -- the factorisation, the arithmetic
// per entry and the order of the entry sums are m2l_kernel's (the results
// agree to rounding: the compiler contracts the running sums differently).
// What changes is the schedule:
//   * 8 MMA warps, one 8-column tile each: two per scheduler (m2l_kernel's 14
//     column tiles sit 4/4/3/3 on the four schedulers, each of which owns a
//     quarter of the DMMA rate);
//   * H, the canonical offset powers and the tables stay in smem for the
//     CTA's lifetime; X_o is double-buffered and built by all 256 threads
//     from rows prefetched into registers during the previous offset's
//     DMMAs; one __syncthreads per offset, no mbarrier pipeline;
//   * no Y buffer and no reduction warps: 90 KB of smem, so two CTAs share
//     an SM and one CTA's build / epilogue overlaps the other's DMMAs.
// RESULT: no faster (cfg2 M2L 0.225 vs 0.202 ms, cfg4 0.358 vs 0.355 ms), so it
// is opt-in (VPG_M2L_GRID=1).  Two unrelated schedules landing on the same
// time says the bound is not the schedule: per list entry the kernel issues
// ~23 DMMAs and ~21 FP64 CUDA-core warp instructions (X build 4 per complex
// element, epilogue 8 per coefficient), and an FP64 CUDA-core instruction
// issued among DMMAs costs ~9 cycles of the shared FP64 pipe against 16 for a
// DMMA (tools/dmma_with_dfma.cu): the pipe is busy ~1.5x the DMMA time, which
// is the ~50% DMMA-path utilisation both kernels show.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "plan.cuh"

namespace vpg {

static __constant__ double c_neg_inv_k_grid[64];  // -1/k, k = 1..63

namespace {

constexpr int kGHS = 60;      // row stride of H^T in smem (fmm.cu kM2LHS)
constexpr int kGCanon = 7;
constexpr int kGBoxes = 32;   // target boxes per tile: 64 columns = 8 column tiles = 8 warps
constexpr int kGXS = 68;      // X row stride (== 4 mod 16: conflict-free B fragments)
constexpr int kGOff = 27;     // offsets per class
constexpr int kGThreads = 256;
constexpr int kGRegs = 7;     // k values per build thread: 8 threads per box, k = 1 + kp + 8 r

__device__ __forceinline__ double2 gturn(double2 v, int r, int sconj) {  // fmm.cu turn()
    int xh = __double2hiint(v.x), xl = __double2loint(v.x);
    int yh = __double2hiint(v.y) ^ (sconj << 31), yl = __double2loint(v.y);
    const bool sw = r & 1;
    int ah = sw ? yh : xh, al = sw ? yl : xl;
    int bh = sw ? xh : yh, bl = sw ? xl : yl;
    ah ^= ((r + 1) & 2) << 30;
    bh ^= (r & 2) << 30;
    return make_double2(__hiloint2double(ah, al), __hiloint2double(bh, bl));
}

__device__ __forceinline__ void gdmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int MT, int NK>  // row tiles RP / 8; k-steps KP / 4 when known at compile time (0: runtime)
__global__ void __launch_bounds__(kGThreads, 2)
m2l_grid_kernel(const GridTile* tiles, int ntiles, const int32_t* trows, const int32_t* nbr,
                const int32_t* cls_oidx, const double* h_t, const double2* canon_g, const int32_t* omap_g,
                const double2* logmd_g, const double2* mult, double2* loc, int P, int KP, double side) {
    extern __shared__ __align__(16) double gsm[];
    const int n = P + 1;
    double* hs = gsm;                                                   // [KP][kGHS]
    double2* canon = reinterpret_cast<double2*>(hs + KP * kGHS);        // [7][n]
    double2* logmd = canon + kGCanon * n;                               // [49]
    double2* a0s = logmd + 49;                                          // [2][kGBoxes]
    double* Xs = reinterpret_cast<double*>(a0s + 2 * kGBoxes);          // [2][KP][kGXS]
    int32_t* omap_s = reinterpret_cast<int32_t*>(Xs + 2 * KP * kGXS);   // [52]
    int32_t* oidx_s = omap_s + 52;                                      // [4][kGOff]
    __shared__ double ninv[64];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    for (int i = tid; i < KP * kGHS; i += kGThreads) hs[i] = h_t[i];
    for (int i = tid; i < kGCanon * n; i += kGThreads) canon[i] = canon_g[i];
    for (int i = tid; i < 49; i += kGThreads) {
        logmd[i] = logmd_g[i];
        omap_s[i] = omap_g[i];
    }
    for (int i = tid; i < 4 * kGOff; i += kGThreads) oidx_s[i] = cls_oidx[i];
    for (int i = tid; i < 64; i += kGThreads) ninv[i] = c_neg_inv_k_grid[i];
    for (int i = tid; i < 2 * KP * kGXS; i += kGThreads) Xs[i] = 0.0;  // rows P .. KP - 1 stay zero
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const int bj = tid >> 3, kp = tid & 7;  // build: box bj, powers k = 1 + kp + 8 r
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const GridTile T = tiles[tile];
        const int32_t* tn = nbr + int64_t(T.first) * kGOff;
        const int32_t* ox = oidx_s + T.cls * kGOff;
        double racc[MT][2];
#pragma unroll
        for (int i = 0; i < MT; ++i) racc[i][0] = racc[i][1] = 0.0;
        double qsum = 0.0;
        double2 areg[kGRegs], a0reg;
        auto fetch = [&](int oi) {
            const int src = bj < T.count ? tn[bj * kGOff + oi] : -1;
#pragma unroll
            for (int r = 0; r < kGRegs; ++r) {
                const int k = 1 + kp + 8 * r;
                areg[r] = (src >= 0 && k <= P) ? mult[int64_t(src) * n + k] : make_double2(0.0, 0.0);
            }
            a0reg = (src >= 0 && kp == 0) ? mult[int64_t(src) * n] : make_double2(0.0, 0.0);
        };
        auto build = [&](int oi, int buf) {
            const int om = omap_s[ox[oi]];
            const int ci = om & 7, sc = (om >> 3) & 1, m2 = ((om >> 4) & 3) + 2;
            double* X = Xs + buf * KP * kGXS;
#pragma unroll
            for (int r = 0; r < kGRegs; ++r) {
                const int k = 1 + kp + 8 * r;
                if (k <= P) {
                    const double2 a = areg[r];
                    const double2 d = gturn(canon[ci * n + k], (m2 * k) & 3, sc);
                    const double vr = fma(a.x, d.x, -(a.y * d.y));
                    const double vi = fma(a.x, d.y, a.y * d.x);
                    *reinterpret_cast<double2*>(X + (k - 1) * kGXS + 2 * bj) = make_double2(vr, vi);
                }
            }
            if (kp == 0) a0s[buf * kGBoxes + bj] = a0reg;
        };
        fetch(0);
        build(0, 0);
        __syncthreads();
        for (int oi = 0; oi < kGOff; ++oi) {
            const int buf = oi & 1;
            if (oi + 1 < kGOff) fetch(oi + 1);
            double acc[MT][2];
#pragma unroll
            for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = 0.0;
            const double* X = Xs + buf * KP * kGXS + kq * kGXS + 8 * w + rq;
            const double* hcol = hs + kq * kGHS + rq;
            auto kstep = [&](int k4) {
                const double bfr = X[k4 * kGXS];
#pragma unroll
                for (int i = 0; i < MT; ++i) gdmma(acc[i][0], acc[i][1], hcol[k4 * kGHS + 8 * i], bfr);
            };
            if constexpr (NK > 0) {
#pragma unroll
                for (int s4 = 0; s4 < NK; ++s4) kstep(4 * s4);
            } else {
#pragma unroll 2
                for (int k4 = 0; k4 < KP; k4 += 4) kstep(k4);
            }
            // diagonal epilogue on the accumulators (m2l_kernel's, same expressions), added in list order
            {
                const int o = ox[oi];
                const int om = omap_s[o];
                const int ci = om & 7, sc = (om >> 3) & 1, m = (om >> 4) & 3;
                const double2 a0 = a0s[buf * kGBoxes + 4 * w + kq];
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int l = 8 * i + rq;
                    if (l <= P) {
                        const double yr = acc[i][0], yi = acc[i][1];
                        double br, bim;
                        if (l == 0) {
                            const double2 lg = logmd[o];
                            br = yr + (lg.x * a0.x - lg.y * a0.y);
                            bim = yi + (lg.x * a0.y + lg.y * a0.x);
                            qsum += a0.x;
                        } else {
                            const double inv_l = ninv[l];  // -1/l
                            const double zr = fma(inv_l, a0.x, yr), zi = fma(inv_l, a0.y, yi);
                            const double2 dl = gturn(canon[ci * n + l], (m * l) & 3, sc);
                            br = dl.x * zr - dl.y * zi;
                            bim = dl.x * zi + dl.y * zr;
                        }
                        racc[i][0] += br;
                        racc[i][1] += bim;
                    }
                }
            }
            if (oi + 1 < kGOff) build(oi + 1, buf ^ 1);
            __syncthreads();
        }
        // the target boxes' local expansions, with the monopole shift (summation.cpp:297-301)
        const int j = 4 * w + kq;
        if (j < T.count) {
            const double logs = log(side / double(1 << T.level));
            const int64_t row = trows[T.first + j];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int l = 8 * i + rq;
                if (l <= P) {
                    double sr = racc[i][0];
                    if (l == 0) sr += qsum * logs;
                    loc[row * n + l] = make_double2(sr, racc[i][1]);
                }
            }
        }
    }
}

using GridKernel = void (*)(const GridTile*, int, const int32_t*, const int32_t*, const int32_t*, const double*,
                            const double2*, const int32_t*, const double2*, const double2*, double2*, int, int,
                            double);

GridKernel grid_kernel_for(int mt, int kp) {
    if (mt == 7 && kp == 52) return m2l_grid_kernel<7, 13>;
    if (mt == 5 && kp == 40) return m2l_grid_kernel<5, 10>;
    if (mt == 4 && kp == 28) return m2l_grid_kernel<4, 7>;
    switch (mt) {
        case 2: return m2l_grid_kernel<2, 0>;
        case 3: return m2l_grid_kernel<3, 0>;
        case 4: return m2l_grid_kernel<4, 0>;
        case 5: return m2l_grid_kernel<5, 0>;
        case 6: return m2l_grid_kernel<6, 0>;
        default: return m2l_grid_kernel<7, 0>;
    }
}

size_t grid_smem(int P, int KP) {
    const int n = P + 1;
    return sizeof(double) * size_t(KP) * kGHS + sizeof(double2) * (size_t(kGCanon) * n + 49 + 2 * kGBoxes) +
           sizeof(double) * 2 * size_t(KP) * kGXS + sizeof(int32_t) * (52 + 4 * kGOff);
}

}  // namespace

// The by-offset schedule for the target boxes over the leaf range [lb, le):
// per (level, class) the target rows, their 27 neighbour rows in the class's
// list order (-1: outside the domain or without sources) and tiles of 32.
void build_m2l_grid(Plan& pl, int64_t lb, int64_t le) {
    pl.n_gt_tiles = 0;
    // opt-in (VPG_M2L_GRID=1): measured no faster than m2l_kernel (cfg2 0.225 vs 0.202 ms, cfg4
    // 0.358 vs 0.355 ms) -- see the note at the top
    const char* ev = std::getenv("VPG_M2L_GRID");
    if (!(ev && std::atoi(ev) == 1) || pl.adaptive || pl.direct || pl.family != VPG_LAPLACE) return;
    const int L = pl.L;
    std::vector<int32_t> oidx(4 * kGOff, 0);
    int dxs[4][kGOff], dys[4][kGOff];
    for (int cls = 0; cls < 4; ++cls) {
        const int cx = cls & 1, cy = cls >> 1;
        int pos = 0;
        for (int qy = -1; qy <= 1; ++qy)
            for (int qx = -1; qx <= 1; ++qx)
                for (int c = 0; c < 4; ++c) {
                    const int dx = 2 * qx + (c & 1) - cx, dy = 2 * qy + ((c & 2) >> 1) - cy;
                    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
                    dxs[cls][pos] = dx;
                    dys[cls][pos] = dy;
                    oidx[size_t(cls * kGOff + pos)] = (dx + 3) + 7 * (dy + 3);
                    ++pos;
                }
        if (pos != kGOff) throw Error{VPG_ERR_CUDA, "M2L class list size"};
    }
    std::vector<GridTile> tiles;
    std::vector<int32_t> rows, nbr;
    for (int l = 2; l <= L; ++l) {
        const int nb = 1 << l, sh = 2 * (L - l);
        const int64_t base = lvl_base(l) - lvl_base(2);
        for (int cls = 0; cls < 4; ++cls) {
            const int32_t first = int32_t(rows.size());
            for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
                const int ix = int(squash2(uint32_t(b))), iy = int(squash2(uint32_t(b) >> 1));
                if (((ix & 1) | ((iy & 1) << 1)) != cls) continue;
                if (!pl.h_tflag[size_t(base + b)]) continue;
                if (!((b << sh) < le && ((b + 1) << sh) > lb)) continue;
                rows.push_back(int32_t(base + b));
                for (int p = 0; p < kGOff; ++p) {
                    const int jx = ix + dxs[cls][p], jy = iy + dys[cls][p];
                    int32_t src = -1;
                    if (jx >= 0 && jy >= 0 && jx < nb && jy < nb) {
                        const int64_t sid = int64_t(mort(uint32_t(jx), uint32_t(jy)));
                        if (pl.h_scnt[size_t(lvl_base(l) + sid)] > 0) src = int32_t(base + sid);
                    }
                    nbr.push_back(src);
                }
            }
            const int32_t count = int32_t(rows.size()) - first;
            for (int32_t t = 0; t < count; t += kGBoxes)
                tiles.push_back(GridTile{l, cls, first + t, std::min(kGBoxes, count - t)});
        }
    }
    if (tiles.empty()) return;
    // big tiles first (the top levels' small ones fill the tail)
    std::stable_sort(tiles.begin(), tiles.end(), [](const GridTile& a, const GridTile& b) { return a.count > b.count; });
    auto up = [](auto& d, const auto& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    };
    up(pl.gt_tiles, tiles);
    up(pl.gt_rows, rows);
    up(pl.gt_nbr, nbr);
    up(pl.gt_oidx, oidx);
    double nik[64] = {0.0};
    for (int k = 1; k < 64; ++k) nik[k] = -1.0 / k;
    VPG_CUDA(cudaMemcpyToSymbol(c_neg_inv_k_grid, nik, sizeof(nik)));
    pl.n_gt_tiles = int64_t(tiles.size());
}

void m2l_grid_issue(const Plan& pl, const double2* mult, double2* loc, cudaStream_t st) {
    const int P = pl.P;
    const size_t smem = grid_smem(P, pl.KP);
    GridKernel kern = grid_kernel_for(pl.RP / 8, pl.KP);
    smem_optin((const void*)kern, int(smem));
    int per_sm = 1;
    VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGThreads, smem));
    const unsigned grid = unsigned(std::min<int64_t>(pl.n_gt_tiles, int64_t(pl.sm_count) * std::max(per_sm, 1)));
    launch_pdl(kern, dim3(grid), dim3(kGThreads), smem, st, (const GridTile*)pl.gt_tiles.p, int(pl.n_gt_tiles),
               (const int32_t*)pl.gt_rows.p, (const int32_t*)pl.gt_nbr.p, (const int32_t*)pl.gt_oidx.p,
               (const double*)pl.h_t.p, (const double2*)pl.m2l_canon.p, (const int32_t*)pl.m2l_omap.p,
               (const double2*)pl.logmd.p, mult, loc, P, pl.KP, pl.side);
}

}  // namespace vpg
