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
#include <vector>

#include "k0.cuh"
#include "plan.cuh"

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
                const double* W, const double* k0tab, double* out) {
    __shared__ uint64_t st_ent[kTravWarps][kTravStack];
    __shared__ uint32_t st_mask[kTravWarps][kTravStack];
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
                    acc = fma(wb[a * m + bb], kInv2Pi * k0_dev(lambda * r, k0tab), acc);
                }
            }
            if (on) pot = acc;
        }
        if (dm) {
            const bool on = (dm >> lane) & 1u;
            double acc = pot;
            for (int f = soff[id]; f < soff[id + 1]; ++f) {
                const double2 sp = sxy[f];
                acc = fma(kInv2Pi, k0_pair(t.x, t.y, sp.x, sp.y, q[f], lambda, k0tab), acc);
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

void helm_apply(const Plan& pl, const double* q_dev, double* out_dev,
                cudaStream_t st, cudaEvent_t* ev, int64_t& launches) {
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
        traverse_kernel<<<nblk(pl.nt, kTravWarps * 32), kTravWarps * 32, 0, st>>>(
            hp, pl.src_cnt.p, pl.src_off.p, pl.src_sorted.p, qs, pl.tgt_sorted.p,
            pl.tgt_ids.p, pl.nt, pl.helm_nodes.p, W, k0_table_dev(), out_dev);
        VPG_LAUNCH_CHECK();
        ++launches;
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
