// helm.cu -- modified-Helmholtz summation on the device: the reference's
// Chebyshev-proxy treecode (summation.cpp:350-497) on the same tree.
//
//   build_helm_ops (summation.cpp:367-396): first proxy level, skip
//     distance, per-level Chebyshev node counts m and barycentric weights.
//   anterpolation (summation.cpp:423-447): per box and level, the m x m
//     proxy charges W[a][b] = sum_j q_j l_a(x_j) l_b(y_j); one CTA per box,
//     one thread per (a, b), sources staged 32 at a time with their
//     barycentric weight rows in smem.  Sums run in source order like the
//     reference loop.
//   traversal (summation.cpp:449-496): per target, the reference DFS (push
//     order, acceptance d^2 >= 4.5 s^2 at levels >= min_level, far boxes
//     beyond the decay cutoff skipped, direct K0 sums at leaves), executed
//     warp-cooperatively: 32 neighbouring targets share one stack with lane
//     masks (traverse_kernel).  Results scatter back to the original target
//     order.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <type_traits>
#include <vector>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "k0.cuh"
#include "plan.cuh"
#include "sym.cuh"

namespace vpg {
namespace {

constexpr int kMaxLevels = 16;
constexpr int kMaxM = 26;

struct HelmParams {
    int L, min_level;
    double x0, y0, side, lambda, skip_x;
    int m[kMaxLevels];
    int64_t w_off[kMaxLevels];  // doubles
};

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

__device__ inline void bary_row(const double* nodes, const double* bw, int m,
                                double x, double* w) {
    // summation.cpp:398-414
    for (int a = 0; a < m; ++a)
        if (x == nodes[a]) {
            for (int b = 0; b < m; ++b) w[b] = b == a ? 1.0 : 0.0;
            return;
        }
    double sum = 0.0;
    for (int a = 0; a < m; ++a) {
        w[a] = bw[a] / (x - nodes[a]);
        sum += w[a];
    }
    const double inv = 1.0 / sum;
    for (int a = 0; a < m; ++a) w[a] *= inv;
}

constexpr int kAntChunk = 32;

__global__ void anterp_kernel(HelmParams hp, int level, const int32_t* src_cnt_l,
                              const int32_t* soff, const double2* sxy,
                              const double* q, const double* nodes_all,
                              const double* bw_all, double* W) {
    extern __shared__ double sma[];
    const int m = hp.m[level];
    const int mm = m * m;
    double* lx = sma;                    // [chunk][m]
    double* ly = sma + kAntChunk * kMaxM;  // [chunk][m]
    __shared__ double nodes[kMaxM], bw[kMaxM];
    const int64_t b = blockIdx.x;
    if (src_cnt_l[b] == 0) return;
    if (threadIdx.x < m) {
        nodes[threadIdx.x] = nodes_all[level * 32 + threadIdx.x];
        bw[threadIdx.x] = bw_all[level * 32 + threadIdx.x];
    }
    const double s = hp.side / double(1 << level);
    const double cx = hp.x0 + (squash2(uint32_t(b)) + 0.5) * s;
    const double cy = hp.y0 + (squash2(uint32_t(b) >> 1) + 0.5) * s;
    const double inv_h = 2.0 / s;
    const int shift = 2 * (hp.L - level);
    const int e0 = soff[b << shift], e1 = soff[(b + 1) << shift];
    const int a = threadIdx.x / m, bb = threadIdx.x % m;
    double acc = 0.0;
    __syncthreads();
    for (int base = e0; base < e1; base += kAntChunk) {
        const int cnt = min(kAntChunk, e1 - base);
        if (threadIdx.x < 2 * cnt) {
            const bool isy = int(threadIdx.x) >= cnt;
            const int j = isy ? int(threadIdx.x) - cnt : int(threadIdx.x);
            const double2 p = sxy[base + j];
            const double x = isy ? (p.y - cy) * inv_h : (p.x - cx) * inv_h;
            bary_row(nodes, bw, m, x, (isy ? ly : lx) + j * kMaxM);
        }
        __syncthreads();
        if (threadIdx.x < mm)
            for (int j = 0; j < cnt; ++j) {
                const double f = q[base + j] * lx[j * kMaxM + a];
                acc = fma(f, ly[j * kMaxM + bb], acc);
            }
        __syncthreads();
    }
    if (threadIdx.x < mm) W[hp.w_off[level] + b * mm + threadIdx.x] = acc;
}

// Warp-cooperative traversal.  A warp takes 32 consecutive (Morton-sorted,
// hence spatially close) targets and walks ONE shared DFS stack in smem
// whose entries carry the mask of lanes still descending.  For the popped
// box every active lane makes the reference decision for its own target
// (skip / proxies / direct leaf / descend); the lanes that take the proxies
// (or the leaf) evaluate them together -- same box, same W row, broadcast
// loads, no divergence in the loop structure -- and the descending lanes'
// mask goes with the four children, pushed in the reference order.  Each
// lane therefore visits exactly the boxes of its own DFS, in the same
// order, with the same arithmetic as a per-target traversal: results are
// those of summation.cpp:449-496 bit for bit.
constexpr int kTravWarps = 4;
constexpr int kTravStack = 96;

__global__ void __launch_bounds__(kTravWarps * 32)
traverse_kernel(HelmParams hp, const int32_t* src_cnt, const int32_t* soff,
                const double2* sxy, const double* q, const double2* txy,
                const int32_t* tids, int64_t nt, const double* nodes_all,
                const double* W, const double* k0f, double* out) {
    __shared__ uint64_t st_ent[kTravWarps][kTravStack];
    __shared__ uint32_t st_mask[kTravWarps][kTravStack];
    __shared__ double k0tab[kK0FastIntervals * kK0FastStride];
    for (int i = threadIdx.x; i < kK0FastIntervals * kK0FastStride; i += blockDim.x) k0tab[i] = k0f[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i0 = (int64_t(blockIdx.x) * kTravWarps + warp) * 32;
    if (i0 >= nt) return;
    const int64_t i = i0 + lane;
    const bool valid = i < nt;
    const double2 t = txy[valid ? i : nt - 1];
    const double lambda = hp.lambda;
    double pot = 0.0;
    uint64_t* sent = st_ent[warp];
    uint32_t* smask = st_mask[warp];
    int top = 0;
    if (lane == 0) {
        sent[0] = 0;
        smask[0] = __ballot_sync(0xffffffffu, valid);
    } else {
        (void)__ballot_sync(0xffffffffu, valid);
    }
    top = 1;
    __syncwarp();
    while (top > 0) {
        --top;
        const uint64_t ent = sent[top];
        const uint32_t mask = smask[top];
        __syncwarp();
        const int l = int(ent >> 32);
        const uint32_t id = uint32_t(ent);
        if (src_cnt[lvl_base(l) + id] == 0) continue;
        const bool me = (mask >> lane) & 1u;
        const double s = hp.side / double(1 << l);
        const double cx = hp.x0 + (squash2(id) + 0.5) * s;
        const double cy = hp.y0 + (squash2(id >> 1) + 0.5) * s;
        const double dx = t.x - cx, dy = t.y - cy;
        const double d2 = dx * dx + dy * dy;
        const double rbox = s * 0.7071067811865476;
        const bool skip = lambda * (sqrt(d2) - rbox) > hp.skip_x;
        const bool proxy = !skip && l >= hp.min_level && d2 >= 4.5 * s * s;
        const bool direct = !skip && !proxy && l == hp.L;
        const uint32_t pm = __ballot_sync(0xffffffffu, me && proxy);
        const uint32_t dm = __ballot_sync(0xffffffffu, me && direct);
        const uint32_t cm = __ballot_sync(0xffffffffu, me && !skip && !proxy && !direct);
        if (pm) {
            const bool on = (pm >> lane) & 1u;
            const int m = hp.m[l];
            const double* wb = W + hp.w_off[l] + int64_t(id) * m * m;
            const double* nd = nodes_all + l * 32;
            const double h = 0.5 * s;
            double acc = pot;
            for (int a = 0; a < m; ++a) {
                const double ex = t.x - (cx + h * nd[a]);
                const double ex2 = ex * ex;
                for (int bb = 0; bb < m; ++bb) {
                    const double ey = t.y - (cy + h * nd[bb]);
                    const double r = sqrt(fma(ey, ey, ex2));
                    acc = fma(wb[a * m + bb], kInv2Pi * k0_fast(lambda * r, k0tab), acc);
                }
            }
            if (on) pot = acc;
        }
        if (dm) {
            const bool on = (dm >> lane) & 1u;
            double acc = pot;
            for (int f = soff[id]; f < soff[id + 1]; ++f) {
                const double2 sp = sxy[f];
                const double dx = t.x - sp.x, dy = t.y - sp.y;
                const double r2 = fma(dy, dy, dx * dx);  // r^2 == 0 skipped (summation.cpp:486)
                acc = fma(kInv2Pi, r2 == 0.0 ? 0.0 : q[f] * k0_fast(lambda * sqrt(r2), k0tab), acc);
            }
            if (on) pot = acc;
        }
        if (cm) {
            if (lane < 4) {
                sent[top + lane] = (uint64_t(l + 1) << 32) | ((uint64_t(id) << 2) | uint64_t(lane));
                smask[top + lane] = cm;
            }
            top += 4;
            __syncwarp();
        }
    }
    if (valid) out[tids[i]] = pot;
}

__global__ void gather_q_h(const double* q, const int32_t* ids, int64_t n, double* qs) {
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e < n) qs[e] = q[ids[e]];
}

HelmParams make_params(const Plan& pl) {
    HelmParams hp{};
    hp.L = pl.L;
    hp.min_level = pl.helm_min_level;
    hp.x0 = pl.x0;
    hp.y0 = pl.y0;
    hp.side = pl.side;
    hp.lambda = pl.lambda;
    hp.skip_x = pl.helm_skip_x;
    for (int l = 0; l <= pl.L && l < kMaxLevels; ++l) {
        hp.m[l] = pl.helm_m[size_t(l)];
        hp.w_off[l] = pl.helm_w_off[size_t(l)];
    }
    return hp;
}


// ===================================================== native-mode FMM ==
// Compressed Chebyshev-interpolation FMM for G = (1/2pi) K0(lambda r)
// (kernel-independent, Fong & Darve): each box at levels lmin..L carries
// values at n x n Chebyshev nodes.
//   P2M   leaves: W[a][b] = sum_j q_j l_a(x_j) l_b(y_j) (anterp_kernel);
//   M2M   W_P = sum_c S_c W_c S_c^T, S_c[a][a'] = l^P_a(x^C_a') (exact:
//         same n on both sides), children in quadrant order;
//   M2L   through a per-level rank-k SVD basis V of the stacked kernel
//         matrices K_o (offsets o, symmetric set => one basis serves both
//         sides): Wt = V^T W, Lt_T = sum_o C_o Wt_S with C_o = V^T K_o V,
//         entries in list order; lists: children of the parent's 3x3
//         neighbours not adjacent to T, and at lmin (the first level with
//         lambda s <= 5, like the treecode's proxies, summation.cpp:367-372)
//         every non-adjacent box; pairs beyond the decay cutoff
//         lambda (d - sqrt(2) s) > skip_x dropped;
//   L2L   Lv_child = V Lt_child + S_c^T Lv_P S_c;
//   L2P + near field: barycentric evaluation of the leaf's Lv at the target
//         plus direct (1/2pi) K0 over the 3x3 neighbour leaves (r = 0 skipped,
//         summation.cpp:486).
// n and k follow epsilon; the basis, the C_o and the lists are built once
// per plan (cuSOLVER SVD and cuBLAS GEMMs at plan time only).
constexpr int kHfMaxN = 20;
constexpr int kHfMaxK = 64;
constexpr int kHfWarps = 8;

__global__ void hf_kmat_kernel(const int2* offs, int noff, int n, const double* nodes, double s,
                               double lambda, const double* k0tab, double* A) {
    const int n2 = n * n;
    const int64_t m = int64_t(noff) * n2;
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= m * n2) return;
    const int64_t row = idx % m;
    const int col = int(idx / m);
    const int o = int(row / n2), t = int(row % n2);
    const int ta = t / n, tb = t % n, sa = col / n, sb = col % n;
    const double dx = offs[o].x * s + (nodes[ta] - nodes[sa]) * 0.5 * s;
    const double dy = offs[o].y * s + (nodes[tb] - nodes[sb]) * 0.5 * s;
    A[idx] = kInv2Pi * k0_dev(lambda * sqrt(dx * dx + dy * dy), k0tab);
}

// Child-to-parent interpolation on the FP64 pipe with the matrix in the
// constant bank.  S_h[a][a'] = l_a(x_h(a')) (parent basis a at child node a',
// h = the child half) depends on n only, and the Chebyshev nodes are
// symmetric, so S_1 = J S_0 J (J = index reversal): every product below uses
// S_0 with compile-time indices (DFMA with a c[][] operand, no loads) and the
// child half only reverses which smem element a thread reads or writes.
constexpr int kHfNMin = 8;
__host__ __device__ constexpr int hf_s0_off(int n) { return n <= kHfNMin ? 0 : hf_s0_off(n - 1) + (n - 1) * (n - 1); }
constexpr int kHfS0Total = hf_s0_off(kHfMaxN + 1);
__constant__ double c_hfS0[kHfS0Total];  // S_0 for n = 8..20, row-major [a][a']

template <int N>
__device__ __forceinline__ double hf_s0(int a, int ap) {
    constexpr int kOff = hf_s0_off(N);
    return c_hfS0[kOff + a * N + ap];
}

// parents per CTA (4 N threads each) and target boxes per CTA (N threads
// each), within 48 KB of static smem
__host__ __device__ constexpr int hf_m2m_parents(int n) { return n <= 18 ? 2 : 1; }
__host__ __device__ constexpr int hf_l2l_boxes(int n) { return n <= 18 ? 8 : 6; }

// M2M: W_P = sum_c S_{c&1} W_c S_{c>>1}^T over the children with sources.
// Pass 1: thread (parent, c, column j) forms column j of T_c = S_{c&1} W_c;
// pass 2: thread (parent, c, row a) forms row a of T_c S_{c>>1}^T; the four
// partials are then summed in quadrant order.  Empty children contribute
// zeros; parents without sources are not written (never read downstream).
template <int N>
__global__ void __launch_bounds__(4 * N * hf_m2m_parents(N))
hf_m2m_kernel(int64_t nparents, const int32_t* scnt_l, const int32_t* scnt_c, int64_t base_p, int64_t base_c,
              double* W) {
    constexpr int N2 = N * N, RS = N | 1, MS = N * RS;  // odd row stride: conflict-free rows and columns
    constexpr int P = hf_m2m_parents(N);
    __shared__ double wc[P][4][MS], tt[P][4][MS];
    const int64_t b0 = int64_t(blockIdx.x) * P;
    for (int i = threadIdx.x; i < P * 4 * N2; i += blockDim.x) {
        const int p = i / (4 * N2), r = i % (4 * N2), c = r / N2, e = r % N2;
        const int64_t child = ((b0 + p) << 2) | c;
        wc[p][c][(e / N) * RS + e % N] =
            (b0 + p < nparents && scnt_c[child] > 0) ? W[(base_c + child) * N2 + e] : 0.0;
    }
    __syncthreads();
    const int p = threadIdx.x / (4 * N), c = (threadIdx.x / N) & 3, j = threadIdx.x % N;
    {
        const bool rx = c & 1;
        double w[N];
#pragma unroll
        for (int q = 0; q < N; ++q) w[q] = wc[p][c][(rx ? N - 1 - q : q) * RS + j];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            double u = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) u = fma(hf_s0<N>(a, q), w[q], u);
            tt[p][c][(rx ? N - 1 - a : a) * RS + j] = u;
        }
    }
    __syncthreads();
    {
        const bool ry = c >> 1;
        double t[N];
#pragma unroll
        for (int q = 0; q < N; ++q) t[q] = tt[p][c][j * RS + (ry ? N - 1 - q : q)];
#pragma unroll
        for (int bb = 0; bb < N; ++bb) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) v = fma(hf_s0<N>(bb, q), t[q], v);
            wc[p][c][j * RS + (ry ? N - 1 - bb : bb)] = v;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P * N2; i += blockDim.x) {
        const int pp = i / N2, e = i % N2;
        const int64_t b = b0 + pp;
        if (b >= nparents || scnt_l[b] == 0) continue;
        const int s = (e / N) * RS + e % N;
        W[(base_p + b) * N2 + e] = ((wc[pp][0][s] + wc[pp][1][s]) + wc[pp][2][s]) + wc[pp][3][s];
    }
}

// L2L: Lv[r] += S_{c&1}^T Lp S_{c>>1} (Lp = the parent's Lv, c = r's
// quadrant).  Pass 1: thread (box, row a') forms row a' of Lp S_{c>>1};
// pass 2: thread (box, column j) forms column j of S_{c&1}^T (that) and adds
// it into Lv[r].
template <int N>
__global__ void __launch_bounds__(N * hf_l2l_boxes(N))
hf_l2l_kernel(int64_t nbox, int64_t base_l, int64_t base_p, const int32_t* tbox, double* Lv) {
    constexpr int N2 = N * N, RS = N | 1, MS = N * RS;
    constexpr int P = hf_l2l_boxes(N);
    __shared__ double lp[P][MS], tt[P][MS];
    const int64_t i0 = int64_t(blockIdx.x) * P;
    for (int i = threadIdx.x; i < P * N2; i += blockDim.x) {
        const int p = i / N2, e = i % N2;
        if (i0 + p < nbox) {
            const int64_t b = tbox[i0 + p] - base_l;
            lp[p][(e / N) * RS + e % N] = Lv[(base_p + (b >> 2)) * N2 + e];
        }
    }
    __syncthreads();
    const int p = threadIdx.x / N, j = threadIdx.x % N;
    const bool live = i0 + p < nbox;
    const int64_t r = live ? tbox[i0 + p] : 0;
    const int c = int((r - base_l) & 3);
    if (live) {
        const bool ry = c >> 1;
        double l[N];
#pragma unroll
        for (int q = 0; q < N; ++q) l[q] = lp[p][j * RS + (ry ? N - 1 - q : q)];
#pragma unroll
        for (int bb = 0; bb < N; ++bb) {
            double u = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) u = fma(hf_s0<N>(q, bb), l[q], u);
            tt[p][j * RS + (ry ? N - 1 - bb : bb)] = u;
        }
    }
    __syncthreads();
    if (live) {
        const bool rx = c & 1;
        double t[N];
#pragma unroll
        for (int q = 0; q < N; ++q) t[q] = tt[p][(rx ? N - 1 - q : q) * RS + j];
        double* out = Lv + r * N2 + j;
#pragma unroll
        for (int a = 0; a < N; ++a) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) v = fma(hf_s0<N>(q, a), t[q], v);
            const int row = rx ? N - 1 - a : a;
            out[row * N] += v;
        }
    }
}

// Lagrange weights l_a(x) of x in [-1, 1] on the n Chebyshev nodes, in the product form
// l_a = bw_a prod_{c != a} (x - x_c) / sum, the products by a forward and a backward running
// product and ONE division for the normalisation (the barycentric quotients bw_a / (x - x_a)
// cost n FP64 divisions, ~30 instructions each: 36 per point dominated the leaf P2M and the
// L2P).  At a node every other weight is an exact 0 and the node's own weight 1 to an ulp.
__device__ __forceinline__ void hf_bary(const double* nodes, const double* bw, int n, double x, double* w) {
    double run = 1.0;
#pragma unroll
    for (int a = 0; a < kHfMaxN; ++a) {
        if (a < n) {
            w[a] = run;
            run *= x - nodes[a];
        }
    }
    run = 1.0;
    double sum = 0.0;
#pragma unroll
    for (int a = kHfMaxN - 1; a >= 0; --a) {
        if (a < n) {
            w[a] *= run * bw[a];
            sum += w[a];
            run *= x - nodes[a];
        }
    }
    const double inv = 1.0 / sum;
#pragma unroll
    for (int a = 0; a < kHfMaxN; ++a)
        if (a < n) w[a] *= inv;
}

// P2M at the leaves of the Chebyshev FMM: a warp per leaf (leaves hold
// ~16 points), sources 32 at a time: lane j builds the rows q_j l_a(x_j),
// l_b(y_j) in smem, then the lanes, as a 4 x 8 grid, accumulate register
// tiles of 5 x 3 entries of W[a][b] = sum_j q_j l_a(x_j) l_b(y_j) in source
// order (8 smem loads per 15 DFMAs; one entry per (lane, round) took 3 per 2).
constexpr int kAntWarps = 4;  // 41 KB of static smem
constexpr int kAntTA = (kHfMaxN + 3) / 4, kAntTB = (kHfMaxN + 7) / 8;

__global__ void __launch_bounds__(kAntWarps * 32)
hf_anterp_leaf_kernel(int L, int n, double x0, double y0, double side, const int32_t* scnt_leaf,
                      const int32_t* soff, const double2* sxy, const double* q, const double* tab,
                      int64_t base_leaf, double* W) {
    __shared__ double rows[kAntWarps][2][32][kHfMaxN];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b = int64_t(blockIdx.x) * kAntWarps + warp;
    if (b >= (int64_t(1) << (2 * L)) || scnt_leaf[b] == 0) return;
    const int n2 = n * n;
    const double* nodes = tab;
    const double* bw = tab + 32;
    const double s = side / double(1 << L);
    const double cx = x0 + (squash2(uint32_t(b)) + 0.5) * s;
    const double cy = y0 + (squash2(uint32_t(b) >> 1) + 0.5) * s;
    const int e0 = soff[b], e1 = soff[b + 1];
    const int a0 = (lane >> 3) * kAntTA, b0 = (lane & 7) * kAntTB;  // the lane's tile of W
    double acc[kAntTA][kAntTB];
#pragma unroll
    for (int i = 0; i < kAntTA; ++i)
#pragma unroll
        for (int k = 0; k < kAntTB; ++k) acc[i][k] = 0.0;
    for (int base = e0; base < e1; base += 32) {
        const int cnt = min(32, e1 - base);
        __syncwarp();
        if (lane < cnt) {
            const double2 p = sxy[base + lane];
            const double qj = q[base + lane];
            double w[kHfMaxN];
            hf_bary(nodes, bw, n, (p.x - cx) * 2.0 / s, w);
#pragma unroll
            for (int a = 0; a < kHfMaxN; ++a) rows[warp][0][lane][a] = a < n ? qj * w[a] : 0.0;
            hf_bary(nodes, bw, n, (p.y - cy) * 2.0 / s, w);
#pragma unroll
            for (int a = 0; a < kHfMaxN; ++a) rows[warp][1][lane][a] = a < n ? w[a] : 0.0;
        }
        __syncwarp();
        for (int j = 0; j < cnt; ++j) {
            double ra[kAntTA], rb[kAntTB];
#pragma unroll
            for (int i = 0; i < kAntTA; ++i) ra[i] = rows[warp][0][j][a0 + i];
#pragma unroll
            for (int k = 0; k < kAntTB; ++k) rb[k] = b0 + k < kHfMaxN ? rows[warp][1][j][b0 + k] : 0.0;
#pragma unroll
            for (int i = 0; i < kAntTA; ++i)
#pragma unroll
                for (int k = 0; k < kAntTB; ++k) acc[i][k] = fma(ra[i], rb[k], acc[i][k]);
        }
    }
#pragma unroll
    for (int i = 0; i < kAntTA; ++i)
#pragma unroll
        for (int k = 0; k < kAntTB; ++k)
            if (a0 + i < n && b0 + k < n) W[(base_leaf + b) * n2 + (a0 + i) * n + b0 + k] = acc[i][k];
}

struct HfLevels {
    int lmin, L, n, k;
    int64_t base[17];    // first row of each level
    int64_t voff[17];    // V offsets (doubles) per level
};

// M2L on the FP64 tensor cores: a CTA takes a tile of up to 64 target boxes
// of one level and walks the level's offsets in a fixed order; per offset
// it stages C_o (64 x 64) once for the whole tile and the sources' Wt as
// the B operand (zeros where a target has no source at that offset), and
// warp w accumulates output rows 8w..8w+7 for the 16 targets with
// mma.sync m8n8k4 f64.  C_o is read once per tile instead of once per list
// entry (the per-entry form was L2-bandwidth bound).
constexpr int kHfTile = 64;

#ifndef VPG_HF_KUNROLL
#define VPG_HF_KUNROLL 16
#endif
constexpr int kHfKUnroll = VPG_HF_KUNROLL;  // k-loop unroll of the tensor-core M2L
#ifndef VPG_HF_NEAR_UNROLL
#define VPG_HF_NEAR_UNROLL 2
#endif
constexpr int kHfNearUnroll = VPG_HF_NEAR_UNROLL;  // source-loop unroll of the K0 near field

__global__ void __launch_bounds__(256)
hf_m2l_tc_kernel(const int4* tiles, const int32_t* tbox, const int32_t* srcof, const double* C,
                 const double* Wt, double* Lt, double* Lpart) {
    constexpr int k = kHfMaxK;
    // row strides == 4 (mod 16) doubles: the DMMA fragment loads are
    // bank-conflict free (lanes (kq, rq) -> 4 kq + rq distinct)
    constexpr int kCS = k + 4, kWS = kHfTile + 4;
    extern __shared__ __align__(16) double hm2l[];
    double* cs = hm2l;                 // [j][i]  (k x kCS)
    double* ws = hm2l + k * kCS;       // [j][t]  (k x kWS)
    const int4 tl = tiles[2 * blockIdx.x], tr = tiles[2 * blockIdx.x + 1];
    const int t0 = tl.x, nt = tl.y, sbase = tl.z, noff = tl.w;
    const int o0 = tr.x, o1 = tr.y, slot = tr.z;
    const int64_t cb = tr.w;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    constexpr int kNT = kHfTile / 8;  // n-tiles per warp (all of them)
    double acc[kNT][2];
#pragma unroll
    for (int q = 0; q < kNT; ++q) acc[q][0] = acc[q][1] = 0.0;
    // per thread: C elements i2 = tid + 256 r (double2), W column j = tid % 64
    // for targets tid / 64 + 4 r -- all loads of offset o+1 are in flight
    // while the DMMAs of offset o run (register double buffer)
    constexpr int kCR = k * k / 2 / 256, kWR = k * kHfTile / 256;
    const int wj = threadIdx.x & 63, wt0 = threadIdx.x >> 6;
    double2 creg[kCR];
    double wreg[kWR];
    auto fetch = [&](int o) {
        const double2* cg = reinterpret_cast<const double2*>(C + (cb + o) * int64_t(k) * k);
#pragma unroll
        for (int r = 0; r < kCR; ++r) creg[r] = cg[threadIdx.x + 256 * r];
#pragma unroll
        for (int r = 0; r < kWR; ++r) {
            const int t = wt0 + 4 * r;
            const int sr = t < nt ? srcof[sbase + int64_t(t0 + t) * noff + o] : -1;
            wreg[r] = sr >= 0 ? Wt[int64_t(sr) * k + wj] : 0.0;
        }
    };
    if (o0 < o1) fetch(o0);
    for (int o = o0; o < o1; ++o) {
        __syncthreads();  // the previous offset's DMMAs are done with cs / ws
#pragma unroll
        for (int r = 0; r < kCR; ++r) {
            const int e = 2 * (threadIdx.x + 256 * r), jj = e / k, ii = e % k;
            *reinterpret_cast<double2*>(cs + jj * kCS + ii) = creg[r];
        }
#pragma unroll
        for (int r = 0; r < kWR; ++r) ws[wj * kWS + wt0 + 4 * r] = wreg[r];
        __syncthreads();
        if (o + 1 < o1) fetch(o + 1);
#pragma unroll kHfKUnroll
        for (int k4 = 0; k4 < k; k4 += 4) {
            const double a = cs[(k4 + kq) * kCS + 8 * warp + rq];
#pragma unroll
            for (int n8 = 0; n8 < kNT; ++n8) {
                const double b = ws[(k4 + kq) * kWS + 8 * n8 + rq];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(acc[n8][0]), "+d"(acc[n8][1])
                             : "d"(a), "d"(b));
            }
        }
    }
    // lane holds rows 8w + rq, targets 8 n8 + 2 kq + {0, 1}
    const int i = 8 * warp + rq;
#pragma unroll
    for (int n8 = 0; n8 < kNT; ++n8)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = 8 * n8 + 2 * kq + h;
            if (t >= nt) continue;
            if (slot < 0) Lt[int64_t(tbox[t0 + t]) * k + i] = acc[n8][h];
            else Lpart[(int64_t(slot) + t) * k + i] = acc[n8][h];
        }
}

// Split targets (the first M2L level has up to ~200 offsets per box): the
// offset ranges' partial sums (kHfTile apart) added in range order.
__global__ void hf_m2l_reduce_kernel(const int2* splits, int nparts, const double* Lpart, double* Lt) {
    const int2 sp = splits[blockIdx.x];
    const int i = threadIdx.x;
    if (i >= kHfMaxK) return;
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += Lpart[(int64_t(sp.y) + int64_t(p) * kHfTile) * kHfMaxK + i];
    Lt[int64_t(sp.x) * kHfMaxK + i] = acc;
}

// Warp per near-field chunk: far field from the leaf's Lv (barycentric) plus
// the direct 3x3-leaf K0 sum; out = far + near in the original order.
__global__ void __launch_bounds__(kHfWarps * 32, 2)
hf_l2p_p2p_kernel(HfLevels hl, const P2PChunk* chunks, int64_t nchunks, const int2* ranges,
                  const int32_t* tgt_row, const double2* sxy, const double* q, const double2* txy,
                  const int32_t* tids, const double* tab, const double* Lv, double x0, double y0,
                  double side, double lambda, const double* k0tab, const double2* gtab, double* out,
                  int near_on) {
    extern __shared__ double2 hsm[];
    double2* ltab = hsm;  // log table, 8 copies (common.cuh)
    double (*lvs)[kHfMaxN * kHfMaxN] =
        reinterpret_cast<double (*)[kHfMaxN * kHfMaxN]>(hsm + kLogTableSize * kLogTableCopies);
    log_table_to_smem(ltab, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab_lane = log_table_lane_addr(ltab, lane & (kLogTableCopies - 1));
    const int n = hl.n, n2 = n * n;
    const double* nodes = tab;
    const double* bw = tab + 32;
    double* L = lvs[warp];
    for (int64_t ci = int64_t(blockIdx.x) * kHfWarps + warp; ci < nchunks;
         ci += int64_t(gridDim.x) * kHfWarps) {
        const P2PChunk c = chunks[ci];
        if (c.part != 0) continue;  // split chunks: once, whole
        const int64_t row = tgt_row[c.tbegin];  // leaf row (uniform tree, level L)
        const int64_t leaf = row - (lvl_base(hl.L) - lvl_base(2));
        const double s = side / double(1 << hl.L);
        const double cx = x0 + (squash2(uint32_t(leaf)) + 0.5) * s;
        const double cy = y0 + (squash2(uint32_t(leaf) >> 1) + 0.5) * s;
        const int64_t hrow = hl.base[hl.L] + leaf;
        __syncwarp();
        for (int j = lane; j < n2; j += 32) L[j] = Lv[hrow * n2 + j];
        __syncwarp();
        const bool two = c.tcount > 32;  // warp-uniform: second target per lane
        double2 t[2];
        double far[2] = {0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int li = lane + 32 * u;
            t[u] = txy[c.tbegin + min(li, c.tcount - 1)];
            if (u == 1 && !two) continue;
            // far: sum_ab lx_a ly_b L[a][b] at this target (ly held, lx recomputed)
            double ly[kHfMaxN];
            hf_bary(nodes, bw, n, (t[u].y - cy) * 2.0 / s, ly);
            const double x = (t[u].x - cx) * 2.0 / s;
            int hit = -1;
            double sx = 0.0;
            for (int a = 0; a < n; ++a) {
                const double d = x - nodes[a];
                if (d == 0.0) hit = a;
                sx += bw[a] / (d == 0.0 ? 1.0 : d);
            }
            const double inv = 1.0 / sx;
            for (int a = 0; a < n; ++a) {
                const double d = x - nodes[a];
                const double lxa = hit >= 0 ? (a == hit ? 1.0 : 0.0) : bw[a] / d * inv;
                double inner = 0.0;
#pragma unroll
                for (int b2 = 0; b2 < kHfMaxN; ++b2)
                    if (b2 < n) inner = fma(ly[b2], L[a * n + b2], inner);
                far[u] = fma(lxa, inner, far[u]);
            }
        }
        // near: the 3x3 leaves, sources broadcast 32 at a time, both targets
        // per source; K0 through q = (lambda r / 2)^2 (no square root) while
        // every pair of the batch has lambda r <= 2, else the general K0
        double near[2] = {0.0, 0.0};
        const double l2q = 0.25 * lambda * lambda;
        // K0 = -(ln(x/2) + gamma) I0(q) + S(q), q = (x/2)^2, ln(x/2) =
        // (ln r^2 + ln(lambda^2/4)) / 2 with the table log of the Laplace
        // near field; for q <= 1/4 (the near field: lambda r <= 1) the two
        // series end at q^9 (tail < 3e-17 relative)
        const double c0 = 0.5 * log(l2q) + 0.57721566490153286061;
        // every pair of the chunk lies within the 3x3 leaves: |r| <= 3 sqrt(2) s
        const bool fast = l2q * 18.0 * s * s <= 0.25;
        auto sweep = [&](auto fast_tag) {
            constexpr bool kFast = decltype(fast_tag)::value;
            for (int ri = 0; ri < c.rcount; ++ri) {
                const int2 rg = ranges[c.rfirst + ri];
                for (int base = rg.x; base < rg.x + rg.y; base += 32) {
                    const int cnt = min(32, rg.x + rg.y - base);
                    double2 sp = make_double2(0.0, 0.0);
                    double qj = 0.0;
                    if (lane < cnt) {
                        sp = sxy[base + lane];
                        qj = q[base + lane];
                    }
#pragma unroll kHfNearUnroll
                    for (int j = 0; j < cnt; ++j) {
                        const double px = __shfl_sync(0xffffffffu, sp.x, j);
                        const double py = __shfl_sync(0xffffffffu, sp.y, j);
                        const double pq = __shfl_sync(0xffffffffu, qj, j);
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            if (u == 1 && !two) continue;
                            const double dx = t[u].x - px, dy = t[u].y - py;
                            const double r2 = fma(dy, dy, dx * dx);
                            const double qq = l2q * r2;
                            double v;
                            if (kFast) {
                                double ed;
                                const double tl = fast_log_split(r2, tab_lane, ed);
                                const double lnr2 = fma(ed, kLn2Hi, fma(ed, kLn2Lo, tl));
                                v = fma(-fma(0.5, lnr2, c0), k0_i0_9(qq), k0_h_9(qq));
                                if (__double2hiint(r2) < 0x00100000) v = r2 == 0.0 ? 0.0 : k0_small_q(qq);
                            } else {
                                v = r2 == 0.0 ? 0.0
                                              : (qq <= 1.0 ? k0_small_q(qq) : k0_dev(lambda * sqrt(r2), k0tab));
                            }
                            near[u] = fma(kInv2Pi * pq, v, near[u]);
                        }
                    }
                }
            }
        };
        if (!near_on) {  // symmetric near field: out = far here, the finalize adds the near sums
        } else if (fast) sweep(std::true_type{});
        else sweep(std::false_type{});
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int li = lane + 32 * u;
            if (li < c.tcount) out[tids[c.tbegin + li]] = far[u] + near[u];
        }
    }
}

// The K0 near field as a pair function of the symmetric kernel (sym.cuh):
// K0(lambda r) for one unordered pair of nodes, 0 at r = 0 (summation.cpp:486
// skips coincident pairs).  Fast form (every near pair has lambda r <= 1):
// the two series of degree D through q = (lambda r / 2)^2 and the table log
// of r^2; q is clamped at its plan bound so the padding points of partial
// tiles (1e100 away, zero charge) stay finite.  General form: the series for
// q <= 1, else the fitted K0 of k0.cuh.
template <bool kFast, int D>
struct K0NearK {
    static constexpr int kSymMaxR = 2;
    double l2q, c0, qmax, lambda;
    const double* k0tab;
    __device__ __forceinline__ double operator()(double r2, uint32_t tab_lane) const {
        if (kFast) {
            const double qq = fmin(l2q * r2, qmax);
            double ed;
            const double tl = fast_log_split(r2, tab_lane, ed);
            const double lnr2 = fma(ed, kLn2Hi, fma(ed, kLn2Lo, tl));
            double v = fma(-fma(0.5, lnr2, c0), k0_i0_d<D>(qq), k0_h_d<D>(qq));
            if (__double2hiint(r2) < 0x00100000) v = r2 == 0.0 ? 0.0 : k0_small_q(qq);
            return v;
        }
        const double qq = l2q * r2;
        return r2 == 0.0 ? 0.0 : (qq <= 1.0 ? k0_small_q(qq) : k0_dev(lambda * sqrt(r2), k0tab));
    }
};

// Per leaf (warp per leaf): the matched targets add the leaf's slot partials
// of the symmetric K0 sweep in slot order; unmatched targets (beyond the
// leaf's sources) sum their 3x3 near sources one-sided (lanes stride each
// range, butterfly reduction).  out = far (already written) + near / 2 pi.
constexpr int kHfFinWarps = 8;
template <class K>
__global__ void __launch_bounds__(kHfFinWarps * 32)
hf_sym_finalize_kernel(K kern, const SymLeaf* leaves, int64_t nleaves, const double* part, const int2* ranges,
                       const double2* sxy, const double* q, const double2* txy, const int32_t* tids,
                       const double2* gtab, double* out) {
    extern __shared__ double2 hfin[];
    log_table_to_smem(hfin, gtab);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab_lane = log_table_lane_addr(hfin, lane & (kLogTableCopies - 1));
    for (int64_t w = int64_t(blockIdx.x) * kHfFinWarps + warp; w < nleaves;
         w += int64_t(gridDim.x) * kHfFinWarps) {
        const SymLeaf lf = leaves[w];
        for (int k = lane; k < lf.n; k += 32) {
            const double* pk = part + lf.pbase + k;
            double sum = 0.0;
            int sl = 0;
            for (; sl + 4 <= lf.nslot; sl += 4) {  // four loads in flight, added in slot order
                const double a0 = __ldcg(pk + int64_t(sl) * lf.n), a1 = __ldcg(pk + int64_t(sl + 1) * lf.n);
                const double a2 = __ldcg(pk + int64_t(sl + 2) * lf.n), a3 = __ldcg(pk + int64_t(sl + 3) * lf.n);
                sum += a0;
                sum += a1;
                sum += a2;
                sum += a3;
            }
            for (; sl < lf.nslot; ++sl) sum += __ldcg(pk + int64_t(sl) * lf.n);
            double& o = out[tids[lf.tgt + k]];
            o = o + kInv2Pi * sum;
        }
        for (int t = lf.tgt + lf.n; t < lf.t1; ++t) {
            const double2 tp = txy[t];
            double v = 0.0;
            for (int r = 0; r < lf.rcount; ++r) {
                const int2 rg = ranges[lf.rfirst + r];
                for (int j = lane; j < rg.y; j += 32) {
                    const double2 sp = sxy[rg.x + j];
                    const double dx = tp.x - sp.x, dy = tp.y - sp.y;
                    v = fma(q[rg.x + j], kern(fma(dy, dy, dx * dx), tab_lane), v);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) {
                double& o = out[tids[t]];
                o = o + kInv2Pi * v;
            }
        }
    }
}

}  // namespace

void build_helm_ops(Plan& pl) {
    if (pl.L + 1 > kMaxLevels) throw Error{VPG_ERR_INVALID_ARGUMENT, "tree too deep for treecode"};
    // summation.cpp:367-396
    pl.helm_min_level = 2;
    while (pl.helm_min_level <= pl.L && pl.lambda * (pl.side / double(1 << pl.helm_min_level)) > 5.0)
        ++pl.helm_min_level;
    pl.helm_skip_x = std::log(1.0 / pl.eps) + 12.0;
    const int base = 8 + std::max(0, int(std::ceil(std::log(1.15e-8 / pl.eps) / 1.97)));
    pl.helm_m.assign(size_t(pl.L + 1), 0);
    std::vector<double> nodes(size_t(pl.L + 1) * 32, 0.0), bw(size_t(pl.L + 1) * 32, 0.0);
    const double pi = 3.14159265358979323846;
    pl.helm_w_off.assign(size_t(pl.L + 1), 0);
    int64_t off = 0;
    pl.P = 0;
    for (int l = pl.helm_min_level; l <= pl.L; ++l) {
        const double ls = pl.lambda * (pl.side / double(1 << l));
        const int bump = ls <= 0.5 ? 0 : (ls <= 2.0 ? 2 : 5);
        const int m = std::min(base + bump, kMaxM);
        pl.helm_m[size_t(l)] = m;
        pl.P = std::max(pl.P, m);
        for (int a = 0; a < m; ++a) {
            const double th = (2 * a + 1) * pi / (2 * m);
            nodes[size_t(l) * 32 + a] = std::cos(th);
            bw[size_t(l) * 32 + a] = (a % 2 ? -1.0 : 1.0) * std::sin(th);
        }
        pl.helm_w_off[size_t(l)] = off;
        off += (int64_t(1) << (2 * l)) * m * m;
    }
    pl.helm_w_total = off;
    pl.helm_nodes.alloc(nodes.size());
    pl.helm_bw.alloc(bw.size());
    VPG_CUDA(cudaMemcpy(pl.helm_nodes.p, nodes.data(), pl.helm_nodes.bytes(), cudaMemcpyHostToDevice));
    VPG_CUDA(cudaMemcpy(pl.helm_bw.p, bw.data(), pl.helm_bw.bytes(), cudaMemcpyHostToDevice));
}

void helm_fmm_apply(const Plan& pl, const double* q_dev, double* out_dev, cudaStream_t st, cudaEvent_t* ev,
                    int64_t& launches);

void helm_apply(const Plan& pl, const double* q_dev, double* out_dev,
                cudaStream_t st, cudaEvent_t* ev, int64_t& launches) {
    if (pl.hf) {
        helm_fmm_apply(pl, q_dev, out_dev, st, ev, launches);
        return;
    }
    auto mark = [&](int i) {
        if (ev) VPG_CUDA(cudaEventRecord(ev[i], st));
    };
    const HelmParams hp = make_params(pl);
    double* qs = nullptr;
    double* W = nullptr;
    VPG_CUDA(cudaMallocAsync(&qs, sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1)), st));
    VPG_CUDA(cudaMallocAsync(&W, sizeof(double) * size_t(std::max<int64_t>(pl.helm_w_total, 1)), st));
    struct Free {
        void* p[2];
        cudaStream_t s;
        ~Free() {
            for (void* x : p)
                if (x) cudaFreeAsync(x, s);
        }
    } fr{{qs, W}, st};
    mark(0);
    gather_q_h<<<nblk(pl.ns, 256), 256, 0, st>>>(q_dev, pl.src_ids.p, pl.ns, qs);
    VPG_LAUNCH_CHECK();
    ++launches;
    mark(1);
    for (int l = pl.helm_min_level; l <= pl.L; ++l) {
        const int m = pl.helm_m[size_t(l)];
        const int threads = std::max(((m * m + 31) / 32) * 32, 2 * kAntChunk);
        anterp_kernel<<<unsigned(int64_t(1) << (2 * l)), threads,
                        sizeof(double) * 2 * kAntChunk * kMaxM, st>>>(
            hp, l, pl.src_cnt.p + lvl_base(l), pl.src_off.p, pl.src_sorted.p, qs,
            pl.helm_nodes.p, pl.helm_bw.p, W);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(2);
    mark(3);
    mark(4);
    mark(5);
    if (pl.nt > 0) {
        // targets are independent: a shard traverses its sorted-target range only
        const int64_t t0 = pl.shard_t0, nts = pl.shard_t1 - pl.shard_t0;
        if (nts > 0)
            traverse_kernel<<<nblk(nts, kTravWarps * 32), kTravWarps * 32, 0, st>>>(
                hp, pl.src_cnt.p, pl.src_off.p, pl.src_sorted.p, qs, pl.tgt_sorted.p + t0,
                pl.tgt_ids.p + t0, nts, pl.helm_nodes.p, W, k0_fast_table_dev(), out_dev);
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(6);
}


namespace {

struct CuHandles {
    cusolverDnHandle_t sol = nullptr;
    cublasHandle_t blas = nullptr;
    ~CuHandles() {
        if (sol) cusolverDnDestroy(sol);
        if (blas) cublasDestroy(blas);
    }
};

#define VPG_SOLVER(call)                                                                     \
    do {                                                                                     \
        const int st_ = int(call);                                                           \
        if (st_ != 0) throw ::vpg::Error{VPG_ERR_CUDA, std::string(#call) + " failed: " + std::to_string(st_)}; \
    } while (0)

HfLevels hf_levels(const Plan& pl) {
    HfLevels hl{};
    hl.lmin = pl.hf_lmin;
    hl.L = pl.L;
    hl.n = pl.hf_n;
    hl.k = pl.hf_k;
    for (int l = 0; l <= pl.L && l < 17; ++l) {
        hl.base[l] = pl.hf_row_base[size_t(l)];
        hl.voff[l] = pl.hf_V_off[size_t(l)];
    }
    return hl;
}

}  // namespace

// Native-mode plan build for modified Helmholtz (see the block comment at
// hf_kmat_kernel).  Leaves pl.hf false (treecode fallback) when no level is
// fine enough for the interpolation (lambda s > 5 at every level).
// n (Chebyshev nodes per dimension) as a compile-time constant, 8..20
template <class F>
void hf_dispatch_n(int n, F&& f) {
    switch (n) {
#define VPG_HF_N(v) \
    case v: f(std::integral_constant<int, v>()); break;
        VPG_HF_N(8) VPG_HF_N(9) VPG_HF_N(10) VPG_HF_N(11) VPG_HF_N(12) VPG_HF_N(13) VPG_HF_N(14)
        VPG_HF_N(15) VPG_HF_N(16) VPG_HF_N(17) VPG_HF_N(18) VPG_HF_N(19) VPG_HF_N(20)
#undef VPG_HF_N
        default: throw Error{VPG_ERR_INVALID_ARGUMENT, "Chebyshev order outside 8..20"};
    }
}

// S_0 (parent basis at the lower child half's nodes) for every n, written to
// the constant bank once per device; the values depend on n only.
void hf_const_init() {
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && (done >> dev & 1u)) return;
    const double pi = 3.14159265358979323846;
    std::vector<double> s0(size_t(kHfS0Total), 0.0);
    for (int n = kHfNMin; n <= kHfMaxN; ++n) {
        std::vector<double> t(static_cast<size_t>(n)), bw(static_cast<size_t>(n));
        for (int a = 0; a < n; ++a) {
            const double th = (2 * a + 1) * pi / (2 * n);
            t[size_t(a)] = std::cos(th);
            bw[size_t(a)] = (a % 2 ? -1.0 : 1.0) * std::sin(th);
        }
        for (int ap = 0; ap < n; ++ap) {
            const double x = -0.5 + 0.5 * t[size_t(ap)];
            std::vector<double> w(static_cast<size_t>(n));
            int hit = -1;
            double sum = 0.0;
            for (int a = 0; a < n; ++a) {
                const double d = x - t[size_t(a)];
                if (d == 0.0) hit = a;
                w[size_t(a)] = bw[size_t(a)] / (d == 0.0 ? 1.0 : d);
                sum += w[size_t(a)];
            }
            for (int a = 0; a < n; ++a)
                s0[size_t(hf_s0_off(n)) + size_t(a) * n + ap] = hit >= 0 ? (a == hit ? 1.0 : 0.0) : w[size_t(a)] / sum;
        }
    }
    VPG_CUDA(cudaMemcpyToSymbol(c_hfS0, s0.data(), sizeof(double) * s0.size()));
    if (dev < 64) done |= uint64_t(1) << dev;
}

// The M2L schedule of a Chebyshev-FMM plan for the targets of the leaf range
// [lb, le) (vpg_plan_set_shard; the whole tree by default): target rows CSR
// over all levels, the dense (target, offset) -> source row table and the
// 16-target tiles.  A shard keeps the target boxes that lie over its leaves,
// so M2L, the expansion back to node values and L2L shrink with the shard
// (the upward pass stays whole on every rank, as for the Laplace plans).
void hf_build_m2l(Plan& pl, int64_t lb, int64_t le) {
    const int L = pl.L, lmin = pl.hf_lmin, k = pl.hf_k;
    // M2L lists (target rows CSR over all levels; entries: source row, C block)
    std::vector<int32_t> tbox, toff{0}, esrc, eop;
    pl.hf_lvl_t0.assign(size_t(L + 2), 0);
    for (int l = lmin; l <= L; ++l) {
        pl.hf_lvl_t0[size_t(l)] = int64_t(tbox.size());
        const int nb = 1 << l;
        const auto& of = pl.hf_offs[size_t(l)];
        auto oidx = [&](int dx, int dy) {
            for (size_t i = 0; i < of.size(); ++i)
                if (of[i].x == dx && of[i].y == dy) return int(i);
            return -1;
        };
        const int64_t cblk0 = pl.hf_C_off[size_t(l)] / (int64_t(k) * k);
        for (int64_t tb = 0; tb < (int64_t(1) << (2 * l)); ++tb) {
            if (pl.h_tcnt[size_t(lvl_base(l) + tb)] == 0) continue;
            // shards: only the boxes over the shard's leaves (their locals are all the shard's
            // L2L chain and L2P read)
            const int sh = 2 * (L - l);
            if (((tb + 1) << sh) <= lb || (tb << sh) >= le) continue;
            const int tx = int(squash2(uint32_t(tb))), ty = int(squash2(uint32_t(tb) >> 1));
            auto add = [&](int sx, int sy) {
                if (sx < 0 || sy < 0 || sx >= nb || sy >= nb) return;
                if (std::max(std::abs(tx - sx), std::abs(ty - sy)) < 2) return;
                const uint32_t sb = mort(uint32_t(sx), uint32_t(sy));
                if (pl.h_scnt[size_t(lvl_base(l) + sb)] == 0) return;
                const int o = oidx(tx - sx, ty - sy);
                if (o < 0) return;  // beyond the decay cutoff
                esrc.push_back(int32_t(pl.hf_row_base[size_t(l)] + sb));
                eop.push_back(int32_t(cblk0 + o));
            };
            if (l == lmin) {
                for (int sy = 0; sy < nb; ++sy)
                    for (int sx = 0; sx < nb; ++sx) add(sx, sy);
            } else {
                const int px = tx >> 1, py = ty >> 1;
                for (int qy = std::max(0, py - 1); qy <= std::min((nb >> 1) - 1, py + 1); ++qy)
                    for (int qx = std::max(0, px - 1); qx <= std::min((nb >> 1) - 1, px + 1); ++qx)
                        for (int c = 0; c < 4; ++c) add(2 * qx + (c & 1), 2 * qy + (c >> 1));
            }
            tbox.push_back(int32_t(pl.hf_row_base[size_t(l)] + tb));
            toff.push_back(int32_t(esrc.size()));
        }
    }
    pl.hf_lvl_t0[size_t(L + 1)] = int64_t(tbox.size());
    pl.hf_ntbox = int64_t(tbox.size());
    // dense (target, offset) -> source row table and 16-target tiles per level
    {
        std::vector<int32_t> srcof;
        std::vector<int4> tiles;
        std::vector<int2> splits;
        constexpr int kSplitOffsets = 48;  // offsets per tile above which targets are split
        int parts_per_split = 0;           // one part count for every split level
        for (int l = lmin; l <= L; ++l) {
            const int noff = int(pl.hf_offs[size_t(l)].size());
            if (noff > kSplitOffsets)
                parts_per_split = std::max(parts_per_split, (noff + kSplitOffsets - 1) / kSplitOffsets);
        }
        int64_t slot = 0;
        for (int l = lmin; l <= L; ++l) {
            const int64_t a0 = pl.hf_lvl_t0[size_t(l)], a1 = pl.hf_lvl_t0[size_t(l + 1)];
            const int noff = int(pl.hf_offs[size_t(l)].size());
            const int64_t cblk0 = pl.hf_C_off[size_t(l)] / (int64_t(k) * k);
            const int64_t sbase = int64_t(srcof.size()) - a0 * noff;
            for (int64_t ti = a0; ti < a1; ++ti) {
                const size_t row0 = srcof.size();
                srcof.resize(row0 + size_t(noff), -1);
                for (int e = toff[size_t(ti)]; e < toff[size_t(ti + 1)]; ++e)
                    srcof[row0 + size_t(eop[size_t(e)] - cblk0)] = esrc[size_t(e)];
            }
            if (noff > kSplitOffsets) {
                // target tiles x offset ranges -> partial sums (slot + p * kHfTile + t),
                // reduced per target in range order
                const int np = parts_per_split;
                for (int64_t ti = a0; ti < a1; ti += kHfTile) {
                    const int cnt = int(std::min<int64_t>(kHfTile, a1 - ti));
                    for (int t = 0; t < cnt; ++t) splits.push_back(make_int2(tbox[size_t(ti + t)], int(slot + t)));
                    for (int p = 0; p < np; ++p) {
                        const int o0 = int(int64_t(noff) * p / np), o1 = int(int64_t(noff) * (p + 1) / np);
                        tiles.push_back(make_int4(int(ti), cnt, int(sbase), noff));
                        tiles.push_back(make_int4(o0, o1, int(slot + p * kHfTile), int(cblk0)));
                    }
                    slot += int64_t(np) * kHfTile;
                }
            } else {
                for (int64_t ti = a0; ti < a1; ti += kHfTile) {
                    tiles.push_back(make_int4(int(ti), int(std::min<int64_t>(kHfTile, a1 - ti)), int(sbase), noff));
                    tiles.push_back(make_int4(0, noff, -1, int(cblk0)));
                }
            }
        }
        // every split level uses the same part count (ranges of equal count)
        pl.hf_split_parts = parts_per_split;
        pl.hf_nsplit = int64_t(splits.size());
        pl.hf_nparts = slot;
        pl.hf_ntiles = int64_t(tiles.size()) / 2;
        auto up2 = [](auto& d, const auto& h) {
            d.alloc(std::max<size_t>(h.size(), 1));
            if (!h.empty()) VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
        };
        up2(pl.hf_srcof, srcof);
        up2(pl.hf_tiles, tiles);
        up2(pl.hf_splits, splits);
    }
    pl.hf_nent = int64_t(esrc.size());
    auto up = [](auto& d, const auto& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        if (!h.empty()) VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    };
    up(pl.hf_tbox, tbox);
    up(pl.hf_toff, toff);
    up(pl.hf_esrc, esrc);
    up(pl.hf_eop, eop);
}

void build_helm_fmm(Plan& pl) {
    hf_const_init();
    const int L = pl.L;
    int lmin = 2;
    while (lmin <= L && pl.lambda * (pl.side / double(1 << lmin)) > 5.0) ++lmin;
    if (lmin > L || L > 16) return;
    const int n = std::clamp(int(std::ceil(1.5 * std::log10(1.0 / pl.eps))), 8, kHfMaxN);
    const int n2 = n * n;
    const double pi = 3.14159265358979323846;
    // nodes (first kind), barycentric weights, child-half interpolation S[h][a][a']
    std::vector<double> tab(64 + size_t(2) * n * n, 0.0);
    for (int a = 0; a < n; ++a) {
        const double th = (2 * a + 1) * pi / (2 * n);
        tab[size_t(a)] = std::cos(th);
        tab[size_t(32 + a)] = (a % 2 ? -1.0 : 1.0) * std::sin(th);
    }
    for (int h = 0; h < 2; ++h)
        for (int ap = 0; ap < n; ++ap) {
            const double x = (h ? 0.5 : -0.5) + 0.5 * tab[size_t(ap)];
            std::vector<double> w(static_cast<size_t>(n));
            int hit = -1;
            double sum = 0.0;
            for (int a = 0; a < n; ++a) {
                const double d = x - tab[size_t(a)];
                if (d == 0.0) hit = a;
                w[size_t(a)] = tab[size_t(32 + a)] / (d == 0.0 ? 1.0 : d);
                sum += w[size_t(a)];
            }
            for (int a = 0; a < n; ++a)
                tab[64 + size_t(h) * n * n + size_t(a) * n + ap] =
                    hit >= 0 ? (a == hit ? 1.0 : 0.0) : w[size_t(a)] / sum;
        }
    // rows of levels lmin..L
    pl.hf_row_base.assign(size_t(L + 2), 0);
    int64_t rows = 0;
    for (int l = lmin; l <= L; ++l) {
        pl.hf_row_base[size_t(l)] = rows;
        rows += int64_t(1) << (2 * l);
    }
    pl.hf_row_base[size_t(L + 1)] = rows;
    pl.hf_rows = rows;

    // offsets per level (T - S in box units); pruned beyond the decay cutoff
    const double skip_x = std::log(1.0 / pl.eps) + 12.0;
    std::vector<std::vector<int2>> offs(size_t(L + 1));
    for (int l = lmin; l <= L; ++l) {
        const double s = pl.side / double(1 << l);
        const int R = l == lmin ? (1 << l) - 1 : 3;
        for (int dy = -R; dy <= R; ++dy)
            for (int dx = -R; dx <= R; ++dx) {
                if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
                if (pl.lambda * (std::hypot(double(dx), double(dy)) * s - std::sqrt(2.0) * s) > skip_x) continue;
                offs[size_t(l)].push_back(make_int2(dx, dy));
            }
    }

    DBuf<double> dtab;
    dtab.alloc(tab.size());
    VPG_CUDA(cudaMemcpy(dtab.p, tab.data(), dtab.bytes(), cudaMemcpyHostToDevice));
    CuHandles hd;
    VPG_SOLVER(cusolverDnCreate(&hd.sol));
    VPG_SOLVER(cublasCreate(&hd.blas));
    const double* k0tab = k0_table_dev();

    // per level: SVD of the stacked K_o -> right singular vectors
    std::vector<std::vector<double>> vt_all(size_t(L + 1));  // VT (n2 x n2, column-major) per level
    int k = 1;
    const double tol = pl.eps * 0.1;
    for (int l = lmin; l <= L; ++l) {
        const auto& of = offs[size_t(l)];
        if (of.empty()) continue;
        const int noff = int(of.size());
        const int64_t m = int64_t(noff) * n2;
        DBuf<int2> doff;
        doff.alloc(of.size());
        VPG_CUDA(cudaMemcpy(doff.p, of.data(), doff.bytes(), cudaMemcpyHostToDevice));
        DBuf<double> A, S, VT;
        A.alloc(size_t(m) * n2);
        S.alloc(size_t(n2));
        VT.alloc(size_t(n2) * n2);
        const double s = pl.side / double(1 << l);
        hf_kmat_kernel<<<unsigned((m * n2 + 255) / 256), 256>>>(doff.p, noff, n, dtab.p, s, pl.lambda, k0tab, A.p);
        VPG_LAUNCH_CHECK();
        int lwork = 0;
        VPG_SOLVER(cusolverDnDgesvd_bufferSize(hd.sol, int(m), n2, &lwork));
        DBuf<double> work, rwork;
        DBuf<int> info;
        work.alloc(size_t(std::max(lwork, 1)));
        rwork.alloc(size_t(n2));
        info.alloc(1);
        VPG_SOLVER(cusolverDnDgesvd(hd.sol, 'N', 'A', int(m), n2, A.p, int(m), S.p, nullptr, 1, VT.p, n2,
                                    work.p, lwork, rwork.p, info.p));
        int hinfo = 0;
        VPG_CUDA(cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (hinfo != 0) throw Error{VPG_ERR_CUDA, "helmholtz FMM: SVD failed (" + std::to_string(hinfo) + ")"};
        std::vector<double> sv(static_cast<size_t>(n2));
        VPG_CUDA(cudaMemcpy(sv.data(), S.p, S.bytes(), cudaMemcpyDeviceToHost));
        int r = 0;
        while (r < n2 && sv[size_t(r)] > tol * sv[0]) ++r;
        k = std::max(k, r);
        vt_all[size_t(l)].resize(size_t(n2) * n2);
        VPG_CUDA(cudaMemcpy(vt_all[size_t(l)].data(), VT.p, VT.bytes(), cudaMemcpyDeviceToHost));
    }
    k = kHfMaxK;  // rank r <= 64 needed (~50 at 1e-12); the DMMA M2L tile is 64 rows
    // V per level in both layouts; C_o = V^T K_o V
    pl.hf_V_off.assign(size_t(L + 2), 0);
    pl.hf_C_off.assign(size_t(L + 2), 0);
    std::vector<double> vt_rm, vc_cm;  // [n2][k] and [k][n2]
    int64_t coff = 0;
    for (int l = lmin; l <= L; ++l) {
        pl.hf_V_off[size_t(l)] = int64_t(vt_rm.size());
        pl.hf_C_off[size_t(l)] = coff;
        const auto& VT = vt_all[size_t(l)];
        for (int j = 0; j < n2; ++j)
            for (int i = 0; i < k; ++i) vt_rm.push_back(VT.empty() ? 0.0 : VT[size_t(i) + size_t(j) * n2]);
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < n2; ++j) vc_cm.push_back(VT.empty() ? 0.0 : VT[size_t(i) + size_t(j) * n2]);
        coff += int64_t(offs[size_t(l)].size()) * k * k;
    }
    pl.hf_Vt.alloc(vt_rm.size());
    pl.hf_Vc.alloc(vc_cm.size());
    VPG_CUDA(cudaMemcpy(pl.hf_Vt.p, vt_rm.data(), pl.hf_Vt.bytes(), cudaMemcpyHostToDevice));
    VPG_CUDA(cudaMemcpy(pl.hf_Vc.p, vc_cm.data(), pl.hf_Vc.bytes(), cudaMemcpyHostToDevice));
    pl.hf_C.alloc(size_t(std::max<int64_t>(coff, 1)));
    for (int l = lmin; l <= L; ++l) {
        const auto& of = offs[size_t(l)];
        if (of.empty()) continue;
        const int noff = int(of.size());
        const int64_t m = int64_t(noff) * n2;
        DBuf<int2> doff;
        doff.alloc(of.size());
        VPG_CUDA(cudaMemcpy(doff.p, of.data(), doff.bytes(), cudaMemcpyHostToDevice));
        DBuf<double> A, X;
        A.alloc(size_t(m) * n2);
        X.alloc(size_t(m) * k);
        const double s = pl.side / double(1 << l);
        hf_kmat_kernel<<<unsigned((m * n2 + 255) / 256), 256>>>(doff.p, noff, n, dtab.p, s, pl.lambda, k0tab, A.p);
        VPG_LAUNCH_CHECK();
        const double one = 1.0, zero = 0.0;
        // V (n2 x k) column-major == [k][n2] layout (vc_cm)
        const double* V = pl.hf_Vc.p + pl.hf_V_off[size_t(l)];
        VPG_SOLVER(cublasDgemm(hd.blas, CUBLAS_OP_N, CUBLAS_OP_N, int(m), k, n2, &one, A.p, int(m), V, n2,
                               &zero, X.p, int(m)));
        VPG_SOLVER(cublasDgemmStridedBatched(hd.blas, CUBLAS_OP_T, CUBLAS_OP_N, k, k, n2, &one, V, n2, 0, X.p,
                                             int(m), n2, &zero, pl.hf_C.p + pl.hf_C_off[size_t(l)], k,
                                             int64_t(k) * k, noff));
    }
    VPG_CUDA(cudaDeviceSynchronize());

    pl.hf_offs = offs;
    pl.hf_n = n;
    pl.hf_k = k;
    pl.hf_lmin = lmin;
    hf_build_m2l(pl, pl.shard_lb, pl.shard_le);
    // anterp_kernel layout: nodes / bw per level (32 slots) -> the same n nodes at every level
    std::vector<double> nl(size_t(L + 1) * 32, 0.0), bl(size_t(L + 1) * 32, 0.0);
    for (int l = 0; l <= L; ++l)
        for (int a = 0; a < n; ++a) {
            nl[size_t(l) * 32 + a] = tab[size_t(a)];
            bl[size_t(l) * 32 + a] = tab[size_t(32 + a)];
        }
    pl.helm_nodes.alloc(nl.size());
    pl.helm_bw.alloc(bl.size());
    VPG_CUDA(cudaMemcpy(pl.helm_nodes.p, nl.data(), pl.helm_nodes.bytes(), cudaMemcpyHostToDevice));
    VPG_CUDA(cudaMemcpy(pl.helm_bw.p, bl.data(), pl.helm_bw.bytes(), cudaMemcpyHostToDevice));
    pl.hf_tab.alloc(tab.size());
    VPG_CUDA(cudaMemcpy(pl.hf_tab.p, tab.data(), pl.hf_tab.bytes(), cudaMemcpyHostToDevice));
    pl.hf_n = n;
    pl.hf_k = k;
    pl.hf_lmin = lmin;
    pl.P = n;  // reported expansion order: Chebyshev nodes per dimension
    smem_optin((const void*)hf_m2l_tc_kernel, int(sizeof(double) * kHfMaxK * (kHfMaxK + kHfTile + 8)));
    smem_optin((const void*)hf_l2p_p2p_kernel,
               int(size_t(kLogTableBytes) + sizeof(double) * kHfWarps * kHfMaxN * kHfMaxN));
    pl.hf = true;
    // near-field K0 form: every near pair lies within the 3x3 leaves, |r| <= 3 sqrt(2) s
    {
        const double s = pl.side / double(1 << L);
        pl.hf_k0_qmax = 0.25 * pl.lambda * pl.lambda * 18.0 * s * s;
        pl.hf_k0_fast = pl.hf_k0_qmax <= 0.25;
        pl.hf_k0_deg = k0_series_degree(pl.hf_k0_qmax);
    }
    build_sym_near(pl, pl.shard_lb, pl.shard_le);
}

// Half a warp per chunk (cfg5's level-8 leaves hold ~16 targets, so a warp per
// chunk left half its lanes idle): the two halves take independent chunks,
// broadcast their own sources 16 at a time (width-16 shuffles) and give each
// lane up to U targets (chunks of <= 16 U targets).  Same arithmetic per pair
// as hf_l2p_p2p_kernel.
template <int U>
__global__ void __launch_bounds__(kHfWarps * 32, 2)
hf_l2p_p2p16_kernel(HfLevels hl, const P2PChunk* chunks, int64_t nchunks, const int2* ranges,
                    const int32_t* tgt_row, const double2* sxy, const double* q, const double2* txy,
                    const int32_t* tids, const double* tab, const double* Lv, double x0, double y0,
                    double side, double lambda, const double* k0tab, const double2* gtab, double* out) {
    extern __shared__ double2 hsm[];
    double2* ltab = hsm;  // log table, 8 copies (common.cuh)
    const int n = hl.n, n2 = n * n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane >> 4, l16 = lane & 15;
    const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
    double* L = reinterpret_cast<double*>(hsm + kLogTableSize * kLogTableCopies) + (warp * 2 + half) * n2;
    log_table_to_smem(ltab, gtab);
    __syncthreads();
    const uint32_t tab_lane = log_table_lane_addr(ltab, lane & (kLogTableCopies - 1));
    const double* nodes = tab;
    const double* bw = tab + 32;
    const double l2q = 0.25 * lambda * lambda;
    const double c0 = 0.5 * log(l2q) + 0.57721566490153286061;
    for (int64_t ci = (int64_t(blockIdx.x) * kHfWarps + warp) * 2 + half; ci < nchunks;
         ci += int64_t(gridDim.x) * kHfWarps * 2) {
        const P2PChunk c = chunks[ci];
        if (c.part != 0) continue;  // split chunks: once, whole
        const int64_t row = tgt_row[c.tbegin];
        const int64_t leaf = row - (lvl_base(hl.L) - lvl_base(2));
        const double s = side / double(1 << hl.L);
        const double cx = x0 + (squash2(uint32_t(leaf)) + 0.5) * s;
        const double cy = y0 + (squash2(uint32_t(leaf) >> 1) + 0.5) * s;
        const int64_t hrow = hl.base[hl.L] + leaf;
        __syncwarp(hmask);
        for (int j = l16; j < n2; j += 16) L[j] = Lv[hrow * n2 + j];
        __syncwarp(hmask);
        const bool fast = l2q * 18.0 * s * s <= 0.25;
        // passes of 16 U targets (chunks hold <= 64; most cfg5 leaves <= 32)
        for (int tb = 0; tb < c.tcount; tb += 16 * U) {
        const int tcnt = min(16 * U, c.tcount - tb);
        const int nu = (tcnt + 15) >> 4;  // targets per lane (<= U)
        double2 t[U];
        double far[U], near[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            far[u] = near[u] = 0.0;
            t[u] = txy[c.tbegin + tb + min(l16 + 16 * u, tcnt - 1)];
            if (u >= nu) continue;
            double ly[kHfMaxN];
            hf_bary(nodes, bw, n, (t[u].y - cy) * 2.0 / s, ly);
            const double x = (t[u].x - cx) * 2.0 / s;
            int hit = -1;
            double sx = 0.0;
            for (int a = 0; a < n; ++a) {
                const double d = x - nodes[a];
                if (d == 0.0) hit = a;
                sx += bw[a] / (d == 0.0 ? 1.0 : d);
            }
            const double inv = 1.0 / sx;
            for (int a = 0; a < n; ++a) {
                const double d = x - nodes[a];
                const double lxa = hit >= 0 ? (a == hit ? 1.0 : 0.0) : bw[a] / d * inv;
                double inner = 0.0;
#pragma unroll
                for (int b2 = 0; b2 < kHfMaxN; ++b2)
                    if (b2 < n) inner = fma(ly[b2], L[a * n + b2], inner);
                far[u] = fma(lxa, inner, far[u]);
            }
        }
        auto sweep = [&](auto fast_tag) {
            constexpr bool kFast = decltype(fast_tag)::value;
            for (int ri = 0; ri < c.rcount; ++ri) {
                const int2 rg = ranges[c.rfirst + ri];
                for (int base = rg.x; base < rg.x + rg.y; base += 16) {
                    const int cnt = min(16, rg.x + rg.y - base);
                    double2 sp = make_double2(0.0, 0.0);
                    double qj = 0.0;
                    if (l16 < cnt) {
                        sp = sxy[base + l16];
                        qj = q[base + l16];
                    }
#pragma unroll 2
                    for (int j = 0; j < cnt; ++j) {
                        const double px = __shfl_sync(hmask, sp.x, j, 16);
                        const double py = __shfl_sync(hmask, sp.y, j, 16);
                        const double pq = __shfl_sync(hmask, qj, j, 16);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (u >= nu) continue;
                            const double dx = t[u].x - px, dy = t[u].y - py;
                            const double r2 = fma(dy, dy, dx * dx);
                            const double qq = l2q * r2;
                            double v;
                            if (kFast) {
                                double ed;
                                const double tl = fast_log_split(r2, tab_lane, ed);
                                const double lnr2 = fma(ed, kLn2Hi, fma(ed, kLn2Lo, tl));
                                v = fma(-fma(0.5, lnr2, c0), k0_i0_9(qq), k0_h_9(qq));
                                if (__double2hiint(r2) < 0x00100000) v = r2 == 0.0 ? 0.0 : k0_small_q(qq);
                            } else {
                                v = r2 == 0.0 ? 0.0
                                              : (qq <= 1.0 ? k0_small_q(qq) : k0_dev(lambda * sqrt(r2), k0tab));
                            }
                            near[u] = fma(kInv2Pi * pq, v, near[u]);
                        }
                    }
                }
            }
        };
        if (fast) sweep(std::true_type{});
        else sweep(std::false_type{});
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int li = l16 + 16 * u;
            if (u < nu && li < tcnt) out[tids[c.tbegin + tb + li]] = far[u] + near[u];
        }
        }
    }
}

// The per-level compress (Wt = Vt W) and expand (Lv = Vc Lt) GEMMs on the FP64
// tensor cores: C (M x N) = A (M x K) . B (K x N), column-major, M and K at most
// a few hundred (k, n^2), N the level's box count.  A CTA takes NT columns at a
// time: A staged whole in smem once per CTA (leading dimension == 4 mod 16
// doubles so the m8n8k4 fragment loads are conflict-free), the NT B columns
// staged per tile with the next tile's columns prefetched into registers
// while the current tile's DMMAs run; warp w owns 8-row tiles w, w + 8, ...
// and all NT / 8 column tiles; the accumulators go straight to C (8 rows of a
// column are 64 contiguous bytes per lane group).  Persistent CTAs.
__host__ __device__ inline int ld4mod16(int n) { return n + ((4 - n % 16) + 16) % 16; }
template <int NT>
size_t hf_gemm_smem(int M, int K) {
    const int Mp = (M + 7) & ~7, Kp = (K + 3) & ~3;
    return sizeof(double) * (size_t(Kp) * ld4mod16(Mp) + size_t(NT) * ld4mod16(Kp));
}
constexpr int kGemmPre = 24;  // B elements per thread in flight (NT * Kp <= 256 * kGemmPre)
template <int NT>
__global__ void __launch_bounds__(256)
hf_gemm_kernel(int M, int N, int K, const double* A, int lda, const double* B, int ldb, double* C, int ldc) {
    extern __shared__ __align__(16) double gs[];
    const int Mp = (M + 7) & ~7, Kp = (K + 3) & ~3;
    const int la = ld4mod16(Mp), lb = ld4mod16(Kp);
    double* As = gs;                    // [k][m], column-major, ld la
    double* Bs = gs + size_t(Kp) * la;  // [n][k], ld lb
    // A: batches of 8 independent loads per thread
    for (int e0 = threadIdx.x; e0 < Kp * Mp; e0 += 8 * blockDim.x) {
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x, kk = e / Mp, m = e % Mp;
            v[r] = (e < Kp * Mp && kk < K && m < M) ? A[int64_t(kk) * lda + m] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = e0 + r * blockDim.x;
            if (e < Kp * Mp) As[(e / Mp) * la + e % Mp] = v[r];
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    const int mtiles = Mp / 8;
    constexpr int kNt = NT / 8;
    double pre[kGemmPre];
    auto fetch = [&](int64_t n0) {
#pragma unroll
        for (int r = 0; r < kGemmPre; ++r) {
            const int e = threadIdx.x + 256 * r, j = e / Kp, kk = e % Kp;
            pre[r] = (j < NT && n0 + j < N && kk < K) ? B[(n0 + j) * ldb + kk] : 0.0;
        }
    };
    int64_t n0 = int64_t(blockIdx.x) * NT;
    if (n0 < N) fetch(n0);
    for (; n0 < N; n0 += int64_t(gridDim.x) * NT) {
        const int nc = int(min(int64_t(NT), N - n0));
        __syncthreads();  // A staged / the previous tile's B reads are done
#pragma unroll
        for (int r = 0; r < kGemmPre; ++r) {
            const int e = threadIdx.x + 256 * r, j = e / Kp, kk = e % Kp;
            if (j < NT) Bs[j * lb + kk] = pre[r];
        }
        __syncthreads();
        const int64_t nn = n0 + int64_t(gridDim.x) * NT;
        if (nn < N) fetch(nn);
        for (int mt = warp; mt < mtiles; mt += 8) {
            double acc[kNt][2];
#pragma unroll
            for (int t = 0; t < kNt; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 4
            for (int k4 = 0; k4 < Kp; k4 += 4) {
                const double a = As[(k4 + kq) * la + 8 * mt + rq];
#pragma unroll
                for (int nt = 0; nt < kNt; ++nt) {
                    const double b = Bs[(8 * nt + rq) * lb + k4 + kq];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(acc[nt][0]), "+d"(acc[nt][1])
                                 : "d"(a), "d"(b));
                }
            }
            const int m = 8 * mt + rq;
            if (m < M)
#pragma unroll
                for (int nt = 0; nt < kNt; ++nt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = 8 * nt + 2 * kq + h;
                        if (j < nc) C[(n0 + j) * ldc + m] = acc[nt][h];
                    }
        }
    }
}

void hf_gemm(int M, int N, int K, const double* A, int lda, const double* B, int ldb, double* C, int ldc,
             int sm_count, cudaStream_t st) {
    if (N <= 0) return;
    const int Kp = (K + 3) & ~3;
    // widest column tile whose B prefetch fits the registers and A + B the smem
    auto launch = [&](auto nt_tag) {
        constexpr int NT = decltype(nt_tag)::value;
        const size_t smem = hf_gemm_smem<NT>(M, K);
        smem_optin((const void*)hf_gemm_kernel<NT>, int(smem));
        const int grid = int(std::min<int64_t>((N + NT - 1) / NT, int64_t(sm_count)));
        hf_gemm_kernel<NT><<<grid, 256, smem, st>>>(M, N, K, A, lda, B, ldb, C, ldc);
        VPG_LAUNCH_CHECK();
    };
    if (32 * Kp <= 256 * kGemmPre && hf_gemm_smem<32>(M, K) <= 227 * 1024)
        launch(std::integral_constant<int, 32>());
    else if (16 * Kp <= 256 * kGemmPre && hf_gemm_smem<16>(M, K) <= 227 * 1024)
        launch(std::integral_constant<int, 16>());
    else if (8 * Kp <= 256 * kGemmPre && hf_gemm_smem<8>(M, K) <= 227 * 1024)
        launch(std::integral_constant<int, 8>());
    else  // n <= 18 for every eps >= 1e-12 keeps this unreachable
        throw Error{VPG_ERR_INVALID_ARGUMENT, "Chebyshev FMM operator too large for the GEMM tile"};
}

// The K0 pair function of the plan's symmetric near field (K0NearK): the
// fast series form at the plan's degree when every near pair has
// lambda r <= 1, else the general form.
template <class F>
void hf_with_k0(const Plan& pl, F&& f) {
    const double l2q = 0.25 * pl.lambda * pl.lambda;
    const double c0 = 0.5 * std::log(l2q) + 0.57721566490153286061;
    const double qm = pl.hf_k0_qmax;
    const double* kt = k0_table_dev();
    if (!pl.hf_k0_fast) return f(K0NearK<false, 9>{l2q, c0, qm, pl.lambda, kt});
    switch (pl.hf_k0_deg) {
        case 5: return f(K0NearK<true, 5>{l2q, c0, qm, pl.lambda, kt});
        case 6: return f(K0NearK<true, 6>{l2q, c0, qm, pl.lambda, kt});
        case 7: return f(K0NearK<true, 7>{l2q, c0, qm, pl.lambda, kt});
        case 8: return f(K0NearK<true, 8>{l2q, c0, qm, pl.lambda, kt});
        default: return f(K0NearK<true, 9>{l2q, c0, qm, pl.lambda, kt});
    }
}

// Per-apply scratch of the Chebyshev FMM, carved from one block: sorted
// charges, W / Lv rows (n^2 each), Wt / Lt rows (k each), the split-M2L
// partials, the symmetric near field's slot partials and its ticket.
namespace {
size_t hf_al(size_t b) { return (b + 255) & ~size_t(255); }
struct HfWork {
    double *qs, *W, *Lv, *Wt, *Lt, *Lpart, *sym_part;
    int* ticket;
};
HfWork hf_work_at(const Plan& pl, void* base, size_t* total) {
    const size_t rows = size_t(std::max<int64_t>(pl.hf_rows, 1));
    const size_t n2 = size_t(pl.hf_n) * pl.hf_n, k = size_t(pl.hf_k);
    char* p = static_cast<char*>(base);
    size_t used = 0;
    auto take = [&](size_t bytes) {
        char* r = p ? p + used : nullptr;
        used += hf_al(bytes);
        return r;
    };
    HfWork w;
    w.qs = reinterpret_cast<double*>(take(sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1))));
    w.W = reinterpret_cast<double*>(take(sizeof(double) * rows * n2));
    w.Lv = reinterpret_cast<double*>(take(sizeof(double) * rows * n2));
    w.Wt = reinterpret_cast<double*>(take(sizeof(double) * rows * k));
    w.Lt = reinterpret_cast<double*>(take(sizeof(double) * rows * k));
    w.Lpart = reinterpret_cast<double*>(take(sizeof(double) * size_t(std::max<int64_t>(pl.hf_nparts, 1)) * kHfMaxK));
    w.sym_part = reinterpret_cast<double*>(take(sizeof(double) * size_t(pl.sym ? std::max<int64_t>(pl.sym_nparts, 1) : 1)));
    w.ticket = reinterpret_cast<int*>(take(sizeof(int) * 32));
    if (total) *total = used;
    return w;
}
}  // namespace

size_t helm_work_bytes(const Plan& pl) {
    size_t total = 0;
    (void)hf_work_at(pl, nullptr, &total);
    return total;
}

void helm_fmm_apply(const Plan& pl, const double* q_dev, double* out_dev, cudaStream_t st, cudaEvent_t* ev,
                    int64_t& launches) {
    void* base = nullptr;
    VPG_CUDA(cudaMallocAsync(&base, helm_work_bytes(pl), st));
    struct Free {
        void* p;
        cudaStream_t s;
        ~Free() {
            if (p) cudaFreeAsync(p, s);
        }
    } fr{base, st};
    helm_fmm_issue(pl, q_dev, out_dev, base, st, ev, launches, nullptr, nullptr, nullptr, nullptr);
}

// The kernels of one Chebyshev-FMM apply in stream order on a given
// workspace (no allocation: capturable into a CUDA graph).  With a side
// stream the symmetric near field runs concurrently with the far-field
// chain; L2P writes out = far on the main stream and the finalize (side)
// adds the near sums after it.
void helm_fmm_issue(const Plan& pl, const double* q_dev, double* out_dev, void* work, cudaStream_t st,
                    cudaEvent_t* ev, int64_t& launches, cudaStream_t side, cudaEvent_t fork, cudaEvent_t join,
                    cudaEvent_t far_done) {
    auto mark = [&](int i) {
        if (ev) VPG_CUDA(cudaEventRecord(ev[i], st));
    };
    const int L = pl.L, n = pl.hf_n, n2 = n * n, k = pl.hf_k;
    const HfLevels hl = hf_levels(pl);
    const HfWork w = hf_work_at(pl, work, nullptr);
    double* qs = w.qs;
    double* W = w.W;
    double* Lv = w.Lv;
    double* Wt = w.Wt;
    double* Lt = w.Lt;
    double* sym_part = w.sym_part;
    int* ticket = w.ticket;
    const bool sym_side = side && pl.sym;
    auto sym_sweep = [&](cudaStream_t s) {
        if (!pl.sym || pl.n_sym_tasks == 0) return;
        VPG_CUDA(cudaMemsetAsync(ticket, 0, 2 * sizeof(int), s));
        hf_with_k0(pl, [&](auto kern) {
            using K = decltype(kern);
            constexpr int kSymWarps = SymShape<K>::kWarps;
            constexpr size_t kSymSmem = sym_smem<K>();
            smem_optin((const void*)p2p_sym_kernel<K>, int(kSymSmem));
            int per_sm = 1;
            VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p2p_sym_kernel<K>, kSymWarps * 32,
                                                                   kSymSmem));
            const int64_t want = (pl.n_sym_tasks + kSymWarps - 1) / kSymWarps;
            const unsigned grid = unsigned(std::min<int64_t>(want, int64_t(pl.sm_count) * std::max(per_sm, 1)));
            p2p_sym_kernel<K><<<grid, kSymWarps * 32, kSymSmem, s>>>(kern, pl.sym_tasks.p, pl.n_sym_tasks,
                                                                     pl.sym_ranges.p, pl.src_sorted.p, qs,
                                                                     log_table_dev(), ticket, sym_part);
        });
        VPG_LAUNCH_CHECK();
        ++launches;
    };
    auto sym_finalize = [&](cudaStream_t s) {
        if (!pl.sym || pl.n_sym_leaves == 0) return;
        hf_with_k0(pl, [&](auto kern) {
            using K = decltype(kern);
            smem_optin((const void*)hf_sym_finalize_kernel<K>, kLogTableBytes);
            const unsigned grid = unsigned(std::min<int64_t>(nblk(pl.n_sym_leaves, kHfFinWarps),
                                                             int64_t(pl.sm_count) * 3));
            hf_sym_finalize_kernel<K><<<grid, kHfFinWarps * 32, kLogTableBytes, s>>>(
                kern, pl.sym_leaves.p, pl.n_sym_leaves, sym_part, pl.near_ranges.p, pl.src_sorted.p, qs,
                pl.tgt_sorted.p, pl.tgt_ids.p, log_table_dev(), out_dev);
        });
        VPG_LAUNCH_CHECK();
        ++launches;
    };
    mark(0);
    gather_q_h<<<nblk(pl.ns, 256), 256, 0, st>>>(q_dev, pl.src_ids.p, pl.ns, qs);
    VPG_LAUNCH_CHECK();
    ++launches;
    if (sym_side) {
        VPG_CUDA(cudaEventRecord(fork, st));
        VPG_CUDA(cudaStreamWaitEvent(side, fork, 0));
        sym_sweep(side);
    }
    mark(1);
    // P2M at the leaves (warp per leaf)
    hf_anterp_leaf_kernel<<<unsigned(((int64_t(1) << (2 * L)) + kAntWarps - 1) / kAntWarps), kAntWarps * 32, 0, st>>>(
        L, n, pl.x0, pl.y0, pl.side, pl.src_cnt.p + lvl_base(L), pl.src_off.p, pl.src_sorted.p, qs, pl.hf_tab.p,
        pl.hf_row_base[size_t(L)], W);
    VPG_LAUNCH_CHECK();
    ++launches;
    mark(2);
    for (int l = L - 1; l >= pl.hf_lmin; --l) {
        const int64_t np = int64_t(1) << (2 * l);
        hf_dispatch_n(n, [&](auto nc) {
            constexpr int N = decltype(nc)::value;
            constexpr int P = hf_m2m_parents(N);
            hf_m2m_kernel<N><<<unsigned((np + P - 1) / P), 4 * N * P, 0, st>>>(
                np, pl.src_cnt.p + lvl_base(l), pl.src_cnt.p + lvl_base(l + 1), pl.hf_row_base[size_t(l)],
                pl.hf_row_base[size_t(l + 1)], W);
        });
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    // compress: Wt_l (k x rows, column-major) = Vt_l (k x n2) . W_l (n2 x rows), one GEMM per level
    for (int l = pl.hf_lmin; l <= L; ++l) {
        const int rows_l = 1 << (2 * l);
        const int64_t b0 = pl.hf_row_base[size_t(l)];
        hf_gemm(k, rows_l, n2, pl.hf_Vt.p + pl.hf_V_off[size_t(l)], k, W + b0 * n2, n2, Wt + b0 * k, k,
                pl.sm_count, st);
        ++launches;
    }
    mark(3);
    if (pl.hf_ntbox > 0) {
        double* Lpart = w.Lpart;
        hf_m2l_tc_kernel<<<unsigned(pl.hf_ntiles), 256, sizeof(double) * kHfMaxK * (kHfMaxK + kHfTile + 8), st>>>(
            pl.hf_tiles.p, pl.hf_tbox.p, pl.hf_srcof.p, pl.hf_C.p, Wt, Lt, Lpart);
        VPG_LAUNCH_CHECK();
        ++launches;
        if (pl.hf_nsplit > 0) {
            hf_m2l_reduce_kernel<<<unsigned(pl.hf_nsplit), kHfMaxK, 0, st>>>(pl.hf_splits.p, pl.hf_split_parts,
                                                                            Lpart, Lt);
        }
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(4);
    // expand: Lv_l (n2 x rows) = Vc_l (n2 x k) . Lt_l (k x rows), one GEMM per level over the rows
    // of the boxes above the shard's leaves (Morton-contiguous; the whole level without shards)
    for (int l = pl.hf_lmin; l <= L; ++l) {
        const int sh = 2 * (L - l);
        const int64_t r0 = pl.shard_lb >> sh, r1 = pl.shard_le > pl.shard_lb ? ((pl.shard_le - 1) >> sh) + 1 : r0;
        if (r1 <= r0) continue;
        const int64_t b0 = pl.hf_row_base[size_t(l)] + r0;
        hf_gemm(n2, int(r1 - r0), k, pl.hf_Vc.p + pl.hf_V_off[size_t(l)], n2, Lt + b0 * k, k, Lv + b0 * n2, n2,
                pl.sm_count, st);
        ++launches;
    }
    // L2L, top-down
    for (int l = pl.hf_lmin + 1; l <= L; ++l) {
        const int64_t t0 = pl.hf_lvl_t0[size_t(l)], t1 = pl.hf_lvl_t0[size_t(l + 1)];
        if (t1 == t0) continue;
        hf_dispatch_n(n, [&](auto nc) {
            constexpr int N = decltype(nc)::value;
            constexpr int P = hf_l2l_boxes(N);
            hf_l2l_kernel<N><<<unsigned((t1 - t0 + P - 1) / P), N * P, 0, st>>>(
                t1 - t0, pl.hf_row_base[size_t(l)], pl.hf_row_base[size_t(l - 1)], pl.hf_tbox.p + t0, Lv);
        });
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    mark(5);
    // symmetric near field (plan.cuh SymTask): the K0 of each unordered node
    // pair once, into slot partials; L2P below writes out = far, the
    // finalize adds the near sums
    if (!sym_side) sym_sweep(st);
    if (pl.n_p2p_chunks > 0) {
        const unsigned grid = unsigned(std::min<int64_t>((pl.n_p2p_chunks + kHfWarps - 1) / kHfWarps,
                                                         int64_t(pl.sm_count) * 8));
#ifndef VPG_HF_HALF
#define VPG_HF_HALF 0  // 1: half-warp chunks, slower on cfg5 (K0 near field 2.23 -> 2.98 ms)
#endif
        if (VPG_HF_HALF && !pl.sym) {  // half a warp per chunk, 32 targets per pass (U = 2)
            const unsigned grid16 = unsigned(std::min<int64_t>((pl.n_p2p_chunks + 2 * kHfWarps - 1) / (2 * kHfWarps),
                                                               int64_t(pl.sm_count) * 8));
            const size_t smem16 = size_t(kLogTableBytes) + sizeof(double) * 2 * kHfWarps * n2;
            smem_optin((const void*)hf_l2p_p2p16_kernel<2>, int(smem16));
            hf_l2p_p2p16_kernel<2><<<grid16, kHfWarps * 32, smem16, st>>>(
                hl, pl.p2p_chunks.p, pl.n_p2p_chunks, pl.near_ranges.p, pl.tgt_row.p, pl.src_sorted.p, qs,
                pl.tgt_sorted.p, pl.tgt_ids.p, pl.hf_tab.p, Lv, pl.x0, pl.y0, pl.side, pl.lambda,
                k0_table_dev(), log_table_dev(), out_dev);
        } else {
            const size_t smem = size_t(kLogTableBytes) + sizeof(double) * kHfWarps * kHfMaxN * kHfMaxN;
            hf_l2p_p2p_kernel<<<grid, kHfWarps * 32, smem, st>>>(
                hl, pl.p2p_chunks.p, pl.n_p2p_chunks, pl.near_ranges.p, pl.tgt_row.p, pl.src_sorted.p, qs,
                pl.tgt_sorted.p, pl.tgt_ids.p, pl.hf_tab.p, Lv, pl.x0, pl.y0, pl.side, pl.lambda,
                k0_table_dev(), log_table_dev(), out_dev, pl.sym ? 0 : 1);
        }
        VPG_LAUNCH_CHECK();
        ++launches;
    }
    if (sym_side) {
        VPG_CUDA(cudaEventRecord(far_done, st));
        VPG_CUDA(cudaStreamWaitEvent(side, far_done, 0));
        sym_finalize(side);
        VPG_CUDA(cudaEventRecord(join, side));
        VPG_CUDA(cudaStreamWaitEvent(st, join, 0));
    } else {
        sym_finalize(st);
    }
    mark(6);
}

__global__ void k0_kernel(const double* x, int64_t n, const double* tab, double* out) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = k0_dev(x[i], tab);
}

void k0_device(const double* x, int64_t n, double* out, cudaStream_t st) {
    if (n <= 0) return;
    k0_kernel<<<nblk(n, 256), 256, 0, st>>>(x, n, k0_table_dev(), out);
    VPG_LAUNCH_CHECK();
}

}  // namespace vpg
