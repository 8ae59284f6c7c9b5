// tree.cu -- on-device quadtree build: bounding box, Morton leaf keys,
// stable radix sort into leaf CSR, per-level occupancy and explicit M2L
// interaction lists.  Reproduces the reference tree bit for bit in
// VPG_MODE_REFERENCE (summation.cpp:81-129, 271-303, 551-591).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "plan.cuh"

namespace vpg {
namespace {

// ---------------------------------------------------------------- bbox --
// Exact min/max (order-independent) in two passes: per-block partials, then
// one block folds them.  summation.cpp:560-575.
constexpr int kBoxThreads = 256;

__global__ void bbox_partial(const double2* a, int64_t na, const double2* b,
                             int64_t nb, double4* part) {
    double xlo = INFINITY, xhi = -INFINITY, ylo = INFINITY, yhi = -INFINITY;
    const int64_t n = na + nb;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double2 p = i < na ? a[i] : b[i - na];
        xlo = fmin(xlo, p.x);
        xhi = fmax(xhi, p.x);
        ylo = fmin(ylo, p.y);
        yhi = fmax(yhi, p.y);
    }
    __shared__ double4 red[kBoxThreads];
    red[threadIdx.x] = make_double4(xlo, xhi, ylo, yhi);
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            double4 u = red[threadIdx.x], v = red[threadIdx.x + s];
            red[threadIdx.x] = make_double4(fmin(u.x, v.x), fmax(u.y, v.y),
                                            fmin(u.z, v.z), fmax(u.w, v.w));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void bbox_final(const double4* part, int n, double4* out) {
    __shared__ double4 red[kBoxThreads];
    double4 acc = make_double4(INFINITY, -INFINITY, INFINITY, -INFINITY);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double4 v = part[i];
        acc = make_double4(fmin(acc.x, v.x), fmax(acc.y, v.y), fmin(acc.z, v.z),
                           fmax(acc.w, v.w));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            double4 u = red[threadIdx.x], v = red[threadIdx.x + s];
            red[threadIdx.x] = make_double4(fmin(u.x, v.x), fmax(u.y, v.y),
                                            fmin(u.z, v.z), fmax(u.w, v.w));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// ------------------------------------------------------------ leaf keys --
// ix = clamp(int((x - x0) / side * n), 0, n-1) -- summation.cpp:85-92.  The
// expression has no multiply-add pair, so no contraction can change it.
__global__ void leaf_keys(const double2* pts, int64_t n, double x0, double y0,
                          double side, int L, uint32_t* keys, int32_t* ids) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int nb = 1 << L;
    const double2 p = pts[j];
    int ix = __double2int_rz(__dmul_rn(__ddiv_rn(__dsub_rn(p.x, x0), side), double(nb)));
    int iy = __double2int_rz(__dmul_rn(__ddiv_rn(__dsub_rn(p.y, y0), side), double(nb)));
    ix = min(max(ix, 0), nb - 1);
    iy = min(max(iy, 0), nb - 1);
    keys[j] = mort(uint32_t(ix), uint32_t(iy));
    ids[j] = int32_t(j);
}

// off[b] = first sorted position with key >= b, b in [0, 4^L].
__global__ void leaf_offsets(const uint32_t* skeys, int64_t n, int64_t nbox,
                             int32_t* off) {
    const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (b > nbox) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (skeys[mid] < uint32_t(b)) lo = mid + 1; else hi = mid;
    }
    off[b] = int32_t(lo);
}

// cnt[l][b] = number of points in the Morton leaf range of box b: the
// closed form of count_levels' child sums (summation.cpp:102-115).
__global__ void level_counts(const int32_t* off, int L, int64_t total,
                             int32_t* cnt) {
    const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (g >= total) return;
    int l = 0;
    while (lvl_base(l + 1) <= g) ++l;
    const int64_t b = g - lvl_base(l);
    const int sh = 2 * (L - l);
    cnt[g] = off[(b + 1) << sh] - off[b << sh];
}

__global__ void gather_points(const double2* pts, const int32_t* ids,
                              int64_t n, double2* out) {
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e < n) out[e] = pts[ids[e]];
}

// ----------------------------------------------------- M2L interaction --
// Children of the parent's 3x3 neighbours that are not neighbours of the
// box, with a non-empty source box (summation.cpp:271-303).  Boxes of
// levels 2..L are addressed by g = lvl_base(l) + b - lvl_base(2).
__device__ inline int box_level(int64_t g, int lmin) {
    int l = lmin;
    while (lvl_base(l + 1) - lvl_base(lmin) <= g) ++l;
    return l;
}

template <bool kFill>
__global__ void m2l_list_kernel(const int32_t* src_cnt, const int32_t* tgt_cnt,
                                int64_t nbox, const int64_t* tpos,
                                const int64_t* epos, int32_t* ecount,
                                int32_t* tflag, int32_t* tbox, int32_t* toff,
                                int32_t* esrc, int32_t* eoidx) {
    const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (g >= nbox) return;
    const int l = box_level(g, 2);
    const int64_t b = g + lvl_base(2) - lvl_base(l);
    const bool active = tgt_cnt[lvl_base(l) + b] > 0;
    if (!kFill) {
        tflag[g] = active ? 1 : 0;
        if (!active) {
            ecount[g] = 0;
            return;
        }
    } else if (!active) {
        return;
    }
    const int nb = 1 << l;
    const int ix = int(squash2(uint32_t(b))), iy = int(squash2(uint32_t(b) >> 1));
    const int px = ix >> 1, py = iy >> 1;
    const int32_t* sc = src_cnt + lvl_base(l);
    int cnt = 0;
    int64_t e = kFill ? epos[g] : 0;
    for (int qy = py - 1; qy <= py + 1; ++qy) {
        if (qy < 0 || qy > (nb >> 1) - 1) continue;
        for (int qx = px - 1; qx <= px + 1; ++qx) {
            if (qx < 0 || qx > (nb >> 1) - 1) continue;
            for (int c = 0; c < 4; ++c) {
                const int jx = 2 * qx + (c & 1), jy = 2 * qy + ((c & 2) >> 1);
                const int dx = jx - ix, dy = jy - iy;
                if (max(abs(dx), abs(dy)) < 2) continue;
                const uint32_t sid = mort(uint32_t(jx), uint32_t(jy));
                if (sc[sid] == 0) continue;
                if (kFill) {
                    // expansion row of the source box (levels 2..L dense)
                    esrc[e] = int32_t(lvl_base(l) - lvl_base(2) + sid);
                    eoidx[e] = (dx + 3) + 7 * (dy + 3);
                    ++e;
                } else {
                    ++cnt;
                }
            }
        }
    }
    if (!kFill) {
        ecount[g] = cnt;
    } else {
        const int64_t t = tpos[g];
        tbox[t] = int32_t(g);  // expansion row of the target box
        toff[t] = int32_t(epos[g]);
    }
}

inline unsigned blocks_for(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// Stable (key, index) sort of one point set into leaf CSR.
void sort_points(const double2* pts, int64_t n, const Plan& pl, int32_t* off,
                 int32_t* ids_out, double2* sorted, cudaStream_t st) {
    const int64_t nbox = int64_t(1) << (2 * pl.L);
    DBuf<uint32_t> keys, skeys;
    DBuf<int32_t> ids;
    keys.alloc(size_t(std::max<int64_t>(n, 1)));
    skeys.alloc(size_t(std::max<int64_t>(n, 1)));
    ids.alloc(size_t(std::max<int64_t>(n, 1)));
    if (n > 0) {
        leaf_keys<<<blocks_for(n, 256), 256, 0, st>>>(pts, n, pl.x0, pl.y0, pl.side,
                                                      pl.L, keys.p, ids.p);
        VPG_LAUNCH_CHECK();
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, skeys.p, ids.p,
                                        ids_out, int(n), 0, 2 * pl.L, st);
        DBuf<unsigned char> tmp;
        tmp.alloc(std::max<size_t>(tmp_bytes, 1));
        VPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, skeys.p,
                                                 ids.p, ids_out, int(n), 0, 2 * pl.L,
                                                 st));
        gather_points<<<blocks_for(n, 256), 256, 0, st>>>(pts, ids_out, n, sorted);
        VPG_LAUNCH_CHECK();
    }
    leaf_offsets<<<blocks_for(nbox + 1, 256), 256, 0, st>>>(skeys.p, n, nbox, off);
    VPG_LAUNCH_CHECK();
    VPG_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
std::vector<T> to_host(const DBuf<T>& d, cudaStream_t st) {
    std::vector<T> h(d.n);
    if (d.n) VPG_CUDA(cudaMemcpyAsync(h.data(), d.p, d.bytes(), cudaMemcpyDeviceToHost, st));
    VPG_CUDA(cudaStreamSynchronize(st));
    return h;
}
template <typename T>
void to_device(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
    d.alloc(h.size());
    if (!h.empty())
        VPG_CUDA(cudaMemcpyAsync(d.p, h.data(), d.bytes(), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void build_tree(Plan& pl) {
    cudaStream_t st;
    VPG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{st};

    // ---- bounding box over sources and targets (summation.cpp:560-576)
    const int64_t ntot = pl.ns + pl.nt;
    double4 bb = make_double4(0, 0, 0, 0);
    if (ntot > 0) {
        const int nblk = int(std::min<int64_t>(blocks_for(ntot, kBoxThreads), 1184));
        DBuf<double4> part, fin;
        part.alloc(size_t(nblk));
        fin.alloc(1);
        bbox_partial<<<nblk, kBoxThreads, 0, st>>>(pl.src.p, pl.ns, pl.tgt.p, pl.nt, part.p);
        VPG_LAUNCH_CHECK();
        bbox_final<<<1, kBoxThreads, 0, st>>>(part.p, nblk, fin.p);
        VPG_LAUNCH_CHECK();
        VPG_CUDA(cudaMemcpyAsync(&bb, fin.p, sizeof(bb), cudaMemcpyDeviceToHost, st));
        VPG_CUDA(cudaStreamSynchronize(st));
    }
    const double side = std::max(bb.y - bb.x, bb.w - bb.z);
    // Pairwise threshold (summation.cpp:578).  NATIVE mode keeps the same
    // threshold: below 4e6 pairs one all-pairs launch beats any tree.
    pl.direct = (ntot == 0) || side <= 0.0 || double(pl.ns) * double(pl.nt) <= 4e6;
    if (pl.direct) return;

    const double big = double(std::max(pl.ns, pl.nt));
    pl.x0 = bb.x;
    pl.y0 = bb.z;
    pl.side = side * (1.0 + 1e-12);
    if (pl.mode == VPG_MODE_NATIVE && pl.family == VPG_LAPLACE) {
        build_adaptive(pl, st);  // adaptive quadtree + U/V/W/X lists (adaptive.cu)
        return;
    }
    pl.L = std::clamp(int(std::ceil(std::log(big / 32.0) / std::log(4.0))), 2, 7);
    if (pl.mode == VPG_MODE_NATIVE && pl.family == VPG_MODIFIED_HELMHOLTZ)
        // Chebyshev FMM (helm.cu): ~16 points per leaf -- the K0 near field
        // dominates, the compressed M2L is cheap
        pl.L = std::clamp(int(std::ceil(std::log(big / 16.0) / std::log(4.0))), 2, 8);
    const int L = pl.L;
    const int64_t nleaf = int64_t(1) << (2 * L);
    const int64_t nall = lvl_base(L + 1);

    // ---- leaf CSR for sources and targets (summation.cpp:81-100, 124-125)
    pl.src_off.alloc(size_t(nleaf + 1));
    pl.tgt_off.alloc(size_t(nleaf + 1));
    pl.src_ids.alloc(size_t(std::max<int64_t>(pl.ns, 1)));
    pl.tgt_ids.alloc(size_t(std::max<int64_t>(pl.nt, 1)));
    pl.src_sorted.alloc(size_t(std::max<int64_t>(pl.ns, 1)));
    pl.tgt_sorted.alloc(size_t(std::max<int64_t>(pl.nt, 1)));
    sort_points(pl.src.p, pl.ns, pl, pl.src_off.p, pl.src_ids.p, pl.src_sorted.p, st);
    sort_points(pl.tgt.p, pl.nt, pl, pl.tgt_off.p, pl.tgt_ids.p, pl.tgt_sorted.p, st);

    // ---- per-level occupancy (summation.cpp:102-115, 126-127)
    pl.src_cnt.alloc(size_t(nall));
    pl.tgt_cnt.alloc(size_t(nall));
    level_counts<<<blocks_for(nall, 256), 256, 0, st>>>(pl.src_off.p, L, nall, pl.src_cnt.p);
    VPG_LAUNCH_CHECK();
    level_counts<<<blocks_for(nall, 256), 256, 0, st>>>(pl.tgt_off.p, L, nall, pl.tgt_cnt.p);
    VPG_LAUNCH_CHECK();

    // ---- explicit M2L lists for levels 2..L (summation.cpp:271-303)
    const int64_t nbox = nall - lvl_base(2);
    {
        DBuf<int32_t> ecount, tflag;
        DBuf<int64_t> epos, tpos;
        ecount.alloc(size_t(nbox));
        tflag.alloc(size_t(nbox));
        epos.alloc(size_t(nbox + 1));
        tpos.alloc(size_t(nbox + 1));
        m2l_list_kernel<false><<<blocks_for(nbox, 128), 128, 0, st>>>(
            pl.src_cnt.p, pl.tgt_cnt.p, nbox, nullptr, nullptr, ecount.p, tflag.p,
            nullptr, nullptr, nullptr, nullptr);
        VPG_LAUNCH_CHECK();
        size_t tb1 = 0, tb2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb1, ecount.p, epos.p, int(nbox), st);
        cub::DeviceScan::ExclusiveSum(nullptr, tb2, tflag.p, tpos.p, int(nbox), st);
        DBuf<unsigned char> tmp;
        tmp.alloc(std::max<size_t>(std::max(tb1, tb2), 1));
        VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb1, ecount.p, epos.p, int(nbox), st));
        VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, tflag.p, tpos.p, int(nbox), st));
        std::vector<int32_t> h_ecount = to_host(ecount, st);
        std::vector<int32_t> h_tflag = to_host(tflag, st);
        std::vector<int64_t> h_epos = to_host(epos, st);
        std::vector<int64_t> h_tpos = to_host(tpos, st);
        pl.n_m2l = h_epos[size_t(nbox - 1)] + h_ecount[size_t(nbox - 1)];
        pl.n_tbox = h_tpos[size_t(nbox - 1)] + h_tflag[size_t(nbox - 1)];
        if (pl.n_m2l > INT32_MAX) throw Error{VPG_ERR_INVALID_ARGUMENT, "M2L list too large"};
        pl.m2l_tbox.alloc(size_t(std::max<int64_t>(pl.n_tbox, 1)));
        pl.m2l_toff.alloc(size_t(pl.n_tbox + 1));
        pl.m2l_src.alloc(size_t(std::max<int64_t>(pl.n_m2l, 1)));
        pl.m2l_oidx.alloc(size_t(std::max<int64_t>(pl.n_m2l, 1)));
        m2l_list_kernel<true><<<blocks_for(nbox, 128), 128, 0, st>>>(
            pl.src_cnt.p, pl.tgt_cnt.p, nbox, tpos.p, epos.p, nullptr, nullptr,
            pl.m2l_tbox.p, pl.m2l_toff.p, pl.m2l_src.p, pl.m2l_oidx.p);
        VPG_LAUNCH_CHECK();
        const int32_t total = int32_t(pl.n_m2l);
        VPG_CUDA(cudaMemcpyAsync(pl.m2l_toff.p + pl.n_tbox, &total, sizeof(total),
                                 cudaMemcpyHostToDevice, st));
        VPG_CUDA(cudaStreamSynchronize(st));

        pl.lvl_tfirst.assign(size_t(L + 2), 0);
        for (int l = 2; l <= L + 1; ++l) {
            const int64_t g = lvl_base(l) - lvl_base(2);
            pl.lvl_tfirst[size_t(l)] = g < nbox ? h_tpos[size_t(g)] : pl.n_tbox;
        }
        pl.h_tflag = std::move(h_tflag);
        pl.h_ecount = std::move(h_ecount);
        pl.h_epos = std::move(h_epos);
        pl.h_tpos = std::move(h_tpos);
    }
    pl.h_scnt = to_host(pl.src_cnt, st);
    pl.h_tcnt = to_host(pl.tgt_cnt, st);
    pl.h_soff = to_host(pl.src_off, st);
    pl.h_toff = to_host(pl.tgt_off, st);
    {
        // expansion rows: levels 2..L dense, row = lvl_base(l) - lvl_base(2) + Morton
        const int64_t rb2 = lvl_base(2);
        pl.n_rows = lvl_base(L + 1) - rb2;
        std::vector<int32_t> rl(size_t(pl.n_rows)), rm(size_t(pl.n_rows)), rp(size_t(pl.n_rows));
        for (int l = 2; l <= L; ++l)
            for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
                const int64_t r = lvl_base(l) - rb2 + b;
                rl[size_t(r)] = l;
                rm[size_t(r)] = int32_t(b);
                rp[size_t(r)] = l > 2 ? int32_t(lvl_base(l - 1) - rb2 + (b >> 2)) : -1;
            }
        to_device(pl.row_level, rl, st);
        to_device(pl.row_morton, rm, st);
        to_device(pl.row_parent, rp, st);
        std::vector<int32_t> tl(size_t(std::max<int64_t>(pl.nt, 1)), 0);
        for (int64_t b = 0; b < nleaf; ++b)
            for (int32_t e = pl.h_toff[size_t(b)]; e < pl.h_toff[size_t(b) + 1]; ++e)
                tl[size_t(e)] = int32_t(lvl_base(L) - rb2 + b);
        to_device(pl.tgt_row, tl, st);
    }
    choose_passes(pl);
    {
        // P2M items: every box with <= up_cap sources, and oversized leaves
        // (split into items + an ordered reduction)
        std::vector<P2MItem> items;
        std::vector<P2MSplit> splits;
        for (int l = 2; l <= L; ++l) {
            const int sh = 2 * (L - l);
            for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
                const int32_t cnt = pl.h_scnt[size_t(lvl_base(l) + b)];
                if (cnt == 0 || (l < L && cnt > pl.up_cap)) continue;
                const int32_t e0 = pl.h_soff[size_t(b << sh)], e1 = pl.h_soff[size_t((b + 1) << sh)];
                const int32_t pieces = (e1 - e0 + kP2MItemCap - 1) / kP2MItemCap;
                const int32_t row = int32_t(lvl_base(l) - lvl_base(2) + b);
                if (pieces > 1) splits.push_back(P2MSplit{row, int32_t(items.size()), pieces});
                for (int32_t e = e0; e < e1; e += kP2MItemCap)
                    items.push_back(P2MItem{l, int32_t(b), row, e, std::min(e1, e + kP2MItemCap), pieces == 1 ? 1 : 0});
            }
        }
        pl.n_p2m_items = int64_t(items.size());
        pl.n_p2m_splits = int64_t(splits.size());
        to_device(pl.p2m_items, items, st);
        to_device(pl.p2m_splits, splits, st);
    }
    build_schedules(pl, 0, nleaf);
}

// Pass selection for uniform trees: per direction, the threshold (see
// Plan::up_cap) minimising a cost model fitted to B200 measurements
// (tools/cap_sweep.sh on cfg1/cfg2/cfg4):
//   direct P2M: max(critical path ~90 ns x points of the largest item,
//               4 ns per item + 45 ps per (point, row));
//   direct L2P: 1.1 ns per (64-target chunk, chain row);
//   M2M / L2L (DMMA shift kernel): ~7.5 us per level with any shifted
//               parent + 1 ns per child.
// VPG_MULTILEVEL=0/1 forces the classical chain / the multilevel passes;
// VPG_PASS_CAP=N forces N in both directions (tests).
void choose_passes(Plan& pl) {
    const int L = pl.L;
    const int32_t kInf = INT32_MAX;
    const char* env = std::getenv("VPG_MULTILEVEL");
    const char* cap_env = std::getenv("VPG_PASS_CAP");
    if (env && (env[0] == '0' || env[0] == '1')) {
        pl.up_cap = pl.dn_cap = env[0] == '1' ? kInf : 0;
    } else if (cap_env && cap_env[0]) {
        pl.up_cap = pl.dn_cap = int32_t(std::atoi(cap_env));
    } else {
        const int32_t caps[] = {0, 16, 32, 64, 128, 256, 1024, 4096, kInf};
        auto shifts = [&](const std::vector<int32_t>& cnt, int32_t cap) {
            double children = 0.0;
            int levels = 0;
            for (int l = 2; l < L; ++l) {
                bool any = false;
                for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
                    if (cnt[size_t(lvl_base(l) + b)] <= cap) continue;
                    any = true;
                    for (int q = 0; q < 4; ++q) children += cnt[size_t(lvl_base(l + 1) + (b << 2) + q)] > 0;
                }
                levels += any;
            }
            return levels * 7.5e-6 + children * 1e-9;
        };
        auto up_cost = [&](int32_t cap) {
            double items = 0.0, rows = 0.0, longest = 0.0;
            for (int l = 2; l <= L; ++l)
                for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
                    const int32_t c = pl.h_scnt[size_t(lvl_base(l) + b)];
                    if (c == 0 || (l < L && c > cap)) continue;
                    items += (c + kP2MItemCap - 1) / kP2MItemCap;
                    rows += c;
                    longest = std::max(longest, double(std::min(c, kP2MItemCap)));
                }
            return std::max(90e-9 * longest, items * 4e-9 + rows * 45e-12) + shifts(pl.h_scnt, cap);
        };
        auto down_cost = [&](int32_t cap) {
            double chunk_rows = 0.0;
            const int64_t nleaf = int64_t(1) << (2 * L);
            for (int64_t b = 0; b < nleaf; ++b) {
                const int32_t t = pl.h_tcnt[size_t(lvl_base(L) + b)];
                if (t == 0) continue;
                int chain = 1;
                for (int l = L - 1; l >= 2 && pl.h_tcnt[size_t(lvl_base(l) + (b >> (2 * (L - l))))] <= cap; --l)
                    ++chain;
                chunk_rows += double((t + 63) / 64) * chain;
            }
            return chunk_rows * 1.1e-9 + shifts(pl.h_tcnt, cap);
        };
        double bu = 1e30, bd = 1e30;
        for (const int32_t cap : caps) {
            const double cu = up_cost(cap), cd = down_cost(cap);
            if (cu < bu) {
                bu = cu;
                pl.up_cap = cap;
            }
            if (cd < bd) {
                bd = cd;
                pl.dn_cap = cap;
            }
        }
    }
    pl.multilevel_up = pl.up_cap == kInf;
    pl.multilevel_down = pl.dn_cap == kInf;
}

// Near-field task list (both trees).  A chunk (<= 64 targets of one leaf)
// worth more than a quarter of a warp's fair share of the near field (~24
// resident warps per SM) and with a large neighbourhood is split into parts
// -- contiguous shares of its flat source list, one warp each -- whose
// partial sums the last finishing warp adds in part order; all other chunks
// are one warp task.  Costliest first (dynamic ticket), stable (equal costs
// keep Morton order).
void schedule_near_chunks(Plan& pl, std::vector<P2PChunk>& chunks) {
    if (pl.near_fair <= 0.0)  // first (whole-tree) schedule of the plan
        pl.near_fair = double(std::max<int64_t>(pl.p2p_pairs, 1)) / (double(pl.sm_count) * 24.0);
    const double fair = pl.near_fair;
    std::vector<P2PChunk> tasks;
    tasks.reserve(chunks.size());
    int32_t slots = 0, parts = 0;
    for (P2PChunk c : chunks) {
        const double pairs = double(c.pad) * c.tcount;
        int np = 1;
        if (c.pad >= kP2PCoopSources && c.tcount > 32 && pairs >= 0.25 * fair)
            np = int(std::min(16.0, std::max(2.0, std::ceil(pairs / (0.25 * fair)))));
        c.nparts = np;
        c.slot = np > 1 ? slots++ : -1;
        c.pbase = np > 1 ? parts : -1;
        for (int i = 0; i < np; ++i) {
            c.part = i;
            tasks.push_back(c);
        }
        if (np > 1) parts += np;
    }
    auto cost = [](const P2PChunk& c) {
        if (c.nparts > 1) return int64_t(c.pad) * 32 / c.nparts;  // 2 targets per lane, one group
        const int nth = (c.tcount + 1) / 2;
        return int64_t(c.pad) * nth / std::max(1, 32 / nth);
    };
    std::stable_sort(tasks.begin(), tasks.end(),
                     [&](const P2PChunk& x, const P2PChunk& y) { return cost(x) > cost(y); });
    chunks.swap(tasks);
    pl.n_p2p_heavy = slots;
    pl.n_p2p_parts = parts;
    pl.n_p2p_chunks = int64_t(chunks.size());
}

// Target-side schedules restricted to the Morton leaf range [lb, le): M2L
// batches and L2L parents of every box overlapping the range, P2P chunks of
// the leaves inside it.  The upward pass (P2M, M2M) always covers the whole
// tree.  [0, 4^L) is the single-GPU plan; a proper sub-range is one shard of
// a multi-GPU run (vpg_plan_set_shard).
void build_schedules(Plan& pl, int64_t lb, int64_t le) {
    const int L = pl.L;
    const int64_t nleaf = int64_t(1) << (2 * L);
    const int64_t nbox = lvl_base(L + 1) - lvl_base(2);
    cudaStream_t st = 0;
    auto overlaps = [&](int l, int64_t b) {
        const int sh = 2 * (L - l);
        return (b << sh) < le && ((b + 1) << sh) > lb;
    };
    pl.shard_lb = lb;
    pl.shard_le = le;
    pl.shard_t0 = pl.h_toff[size_t(lb)];
    pl.shard_t1 = pl.h_toff[size_t(le)];
    {
        // M2L batches of <= kM2LPairs entries that never split a target box
        // (each target's local expansion is reduced by one CTA, fixed order).
        std::vector<M2LBatch> batches;
        M2LBatch cur{};
        bool open = false;
        int cur_level = -1;
        int l = 2;
        for (int64_t g = 0; g < nbox; ++g) {
            while (lvl_base(l + 1) - lvl_base(2) <= g) ++l;
            const bool take = pl.h_tflag[size_t(g)] && overlaps(l, g + lvl_base(2) - lvl_base(l));
            if (!take) {
                if (open) batches.push_back(cur);
                open = false;
                continue;
            }
            const int32_t ne = pl.h_ecount[size_t(g)];
            if (open && (l != cur_level || cur.ecount + ne > kM2LPairs)) {
                batches.push_back(cur);
                open = false;
            }
            if (!open) {
                cur = M2LBatch{l, int32_t(pl.h_tpos[size_t(g)]), 0, int32_t(pl.h_epos[size_t(g)]), 0};
                cur_level = l;
                open = true;
            }
            cur.tcount += 1;
            cur.ecount += ne;
        }
        if (open) batches.push_back(cur);
        pl.n_m2l_batches = int64_t(batches.size());
        to_device(pl.m2l_batches, batches, st);
    }
    build_m2l_grid(pl, lb, le);  // the same entries batched by offset (uniform Laplace trees)
    {
        std::vector<int32_t> boxes;  // parent rows
        std::vector<int4> kids;      // child rows per quadrant, -1 = none
        pl.m2m_first.assign(size_t(L + 1), 0);
        pl.m2m_count.assign(size_t(L + 1), 0);
        pl.l2l_first.assign(size_t(L + 1), 0);
        pl.l2l_count.assign(size_t(L + 1), 0);
        pl.m2m_children = pl.l2l_children = 0;
        auto children = [&](int l, int64_t b, const std::vector<int32_t>& cnt, int64_t& nk) {
            int k4[4];
            for (int c = 0; c < 4; ++c) {
                const int64_t cb = (b << 2) | c;
                k4[c] = cnt[size_t(lvl_base(l + 1) + cb)] > 0 ? int32_t(lvl_base(l + 1) - lvl_base(2) + cb) : -1;
                nk += k4[c] >= 0;
            }
            return make_int4(k4[0], k4[1], k4[2], k4[3]);
        };
        for (int l = 2; l < L; ++l) {
            // M2M: parents at level l above up_cap sources (summation.cpp:257-267
            // with up_cap = 0), children with src_cnt > 0
            pl.m2m_first[size_t(l)] = int64_t(boxes.size());
            for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b)
                if (pl.h_scnt[size_t(lvl_base(l) + b)] > pl.up_cap) {
                    boxes.push_back(int32_t(lvl_base(l) - lvl_base(2) + b));
                    kids.push_back(children(l, b, pl.h_scnt, pl.m2m_children));
                }
            pl.m2m_count[size_t(l)] = int64_t(boxes.size()) - pl.m2m_first[size_t(l)];
        }
        for (int l = 2; l < L; ++l) {
            // L2L: parents at level l above dn_cap targets (summation.cpp:305-312
            // with dn_cap = 0), children with tgt_cnt > 0
            pl.l2l_first[size_t(l)] = int64_t(boxes.size());
            for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b)
                if (pl.h_tcnt[size_t(lvl_base(l) + b)] > pl.dn_cap && overlaps(l, b)) {
                    boxes.push_back(int32_t(lvl_base(l) - lvl_base(2) + b));
                    kids.push_back(children(l, b, pl.h_tcnt, pl.l2l_children));
                }
            pl.l2l_count[size_t(l)] = int64_t(boxes.size()) - pl.l2l_first[size_t(l)];
        }
        to_device(pl.updown_kids, kids, st);
        to_device(pl.updown_boxes, boxes, st);
    }
    {
        const std::vector<int32_t>& h_soff = pl.h_soff;
        const std::vector<int32_t>& h_toff = pl.h_toff;
        const int nb = 1 << L;
        int64_t occupied = 0;
        for (int64_t b = 0; b < nleaf; ++b) occupied += h_toff[size_t(b) + 1] > h_toff[size_t(b)];
        (void)occupied;
        pl.p2p_tpt = 2;
        const int chunk = 64;  // kP2PChunk: two targets per lane
        std::vector<P2PChunk> chunks;
        std::vector<int2> ranges;
        std::vector<int32_t> lrows;
        pl.p2p_pairs = 0;
        pl.h_leafnear.clear();
        for (int64_t b = lb; b < le; ++b) {
            const int32_t t0 = h_toff[size_t(b)], t1 = h_toff[size_t(b) + 1];
            if (t1 == t0) continue;
            // L2P chain: the leaf's local expansion after the L2L pass, or
            // in the multilevel downward pass the leaf's and every ancestor's
            const int32_t lfirst = int32_t(lrows.size());
            for (int l = L; l >= 2; --l) {
                lrows.push_back(int32_t(lvl_base(l) - lvl_base(2) + (b >> (2 * (L - l)))));
                // stop below a parent that pushed its local down by L2L
                if (l > 2 && pl.h_tcnt[size_t(lvl_base(l - 1) + (b >> (2 * (L - l + 1))))] > pl.dn_cap) break;
            }
            const int32_t lcount = int32_t(lrows.size()) - lfirst;
            const int ix = int(squash2(uint32_t(b))), iy = int(squash2(uint32_t(b) >> 1));
            // 3x3 neighbour leaves in the reference order (summation.cpp:330-334)
            const int32_t rfirst = int32_t(ranges.size());
            int32_t rself = 0;
            int64_t nsrc = 0;
            for (int jy = std::max(0, iy - 1); jy <= std::min(nb - 1, iy + 1); ++jy)
                for (int jx = std::max(0, ix - 1); jx <= std::min(nb - 1, ix + 1); ++jx) {
                    const uint32_t sid = mort(uint32_t(jx), uint32_t(jy));
                    if (jx == ix && jy == iy) rself = int32_t(ranges.size()) - rfirst;
                    ranges.push_back(make_int2(h_soff[sid], h_soff[sid + 1] - h_soff[sid]));
                    nsrc += h_soff[sid + 1] - h_soff[sid];
                }
            const int32_t rcount = int32_t(ranges.size()) - rfirst;
            pl.p2p_pairs += int64_t(t1 - t0) * nsrc;
            pl.h_leafnear.push_back(LeafNear{int32_t(b), t0, t1, rfirst, rcount, rself, lfirst, lcount});
            for (int32_t t = t0; t < t1; t += chunk)
                chunks.push_back(P2PChunk{t, std::min(chunk, t1 - t), int32_t(std::min<int64_t>(nsrc, INT32_MAX)),
                                          rfirst, rcount, rself, lfirst, lcount, 0, 1, -1, -1});
        }
        to_device(pl.near_ranges, ranges, st);
        to_device(pl.l2p_rows, lrows, st);
        schedule_near_chunks(pl, chunks);
        to_device(pl.p2p_chunks, chunks, st);
    }
    {
        int64_t m2l = 0;
        int l = 2;
        for (int64_t g = 0; g < nbox; ++g) {
            while (lvl_base(l + 1) - lvl_base(2) <= g) ++l;
            if (pl.h_tflag[size_t(g)] && overlaps(l, g + lvl_base(2) - lvl_base(l)))
                m2l += pl.h_ecount[size_t(g)];
        }
        pl.shard_m2l = m2l;
    }
    if (pl.hf) hf_build_m2l(pl, lb, le);                     // the Chebyshev FMM's far field follows the shard
    if (pl.coin_ready || pl.hf) build_sym_near(pl, lb, le);  // Laplace ops / Chebyshev FMM built
}

// The symmetric near-field schedule (SymTask, plan.cuh) for the targets of
// the leaf range [lb, le): the subtasks of every leaf owning a pair {A, B}
// of near leaves touching the range, the per-leaf slot layout (SymLeaf) for
// the final sums, which also cover the unmatched targets (those beyond a
// leaf's first n_src targets) one-sided.  Taken when the first ns
// targets are the sources (so leaf A's first n_src sorted targets are its
// sorted sources, both sorts being stable), the tree is uniform, the
// kernel Laplace (or modified Helmholtz with the Chebyshev FMM: every pair
// symmetric, no hybrid) and no leaf holds more than kSymMaxN sources.
void build_sym_near(Plan& pl, int64_t lb, int64_t le) {
    pl.sym = false;
    const char* fv = std::getenv("VPG_SYM");  // 0: never, 1: always (when applicable), unset: by cost
    const int force = fv ? std::atoi(fv) : -1;
    if (force == 0 || !pl.matched || pl.adaptive || pl.direct || (pl.family != VPG_LAPLACE && !pl.hf)) return;
    pl.lat = false;
    if (pl.family == VPG_LAPLACE && pl.coin_ready && build_lattice_near(pl, lb, le)) return;  // leaves are translates of one pattern
    const int L = pl.L;
    const int nb = 1 << L;
    const int64_t nleaf = int64_t(1) << (2 * L);
    const bool whole = lb == 0 && le == nleaf;
    const std::vector<int32_t>& so = pl.h_soff;
    const std::vector<int32_t>& to = pl.h_toff;
    auto nsrc = [&](int64_t b) { return so[size_t(b) + 1] - so[size_t(b)]; };
    for (int64_t b = 0; b < nleaf; ++b)
        if (nsrc(b) > kSymMaxN) return;
    auto in = [&](int64_t b) { return b >= lb && b < le; };
    auto neighbour = [&](int64_t a, int slot) -> int64_t {  // slot = (dy+1)*3 + (dx+1), -1 outside
        const int bx = int(squash2(uint32_t(a))) + slot % 3 - 1, by = int(squash2(uint32_t(a) >> 1)) + slot / 3 - 1;
        if (bx < 0 || by < 0 || bx >= nb || by >= nb) return -1;
        return int64_t(mort(uint32_t(bx), uint32_t(by)));
    };
    // rows per lane R = 1 << rsel: 1 for leaves of <= 32 sources, 2 up to
    // 64, for Laplace 4 up to 128 and 8 above (cfg4: near field 5.57 -> 5.31
    // ms at R = 4, the column tile's smem loads and shuffles amortised over
    // the rows and more independent pair chains per warp; VPG_SYM_R4=0: 2,
    // VPG_SYM_R8=0: at most 4; 8 needs a -DVPG_SYM_MAXR=8 build, plan.cuh)
    const char* r4v = std::getenv("VPG_SYM_R4");
    const bool r4 = !(r4v && std::atoi(r4v) == 0) && pl.family == VPG_LAPLACE;
    const char* r8v = std::getenv("VPG_SYM_R8");
    const bool r8 = r4 && kSymLapMaxR >= 8 && !(r8v && std::atoi(r8v) == 0);
    auto rows2_of = [&](int32_t n) { return n > 32 ? 1 : 0; };
    auto rsel_of = [&](int32_t n) { return r8 && n > 128 ? 3 : r4 && n > 64 ? 2 : rows2_of(n); };
    auto nrt_of = [&](int32_t n) { return (n + (32 << rsel_of(n)) - 1) / (32 << rsel_of(n)); };
    // Which pairs go symmetric: all of them (T = 0), or in the hybrid form only
    // pairs of "big" leaves (>= T sources each); the other pairs of a target
    // stay one-sided.  Decided once on the whole tree.
    if (whole) {
        const char* mv = std::getenv("VPG_SYM_MIN");
        const int tmin = mv ? std::atoi(mv) : -1;
        double cost_sym = 0.0, cost_one = 0.0, total = 0.0, big_pairs = 0.0, all_pairs = 0.0;
        constexpr int kBig = 64;
        for (int64_t a = 0; a < nleaf; ++a) {
            const int32_t na = nsrc(a);
            if (!na) continue;
            int32_t nc = na;
            for (int sl = 0; sl < 9; ++sl) {
                const int64_t b = neighbour(a, sl);
                if (b < 0 || !nsrc(b)) continue;
                all_pairs += double(na) * nsrc(b);
                if (std::min(na, nsrc(b)) >= kBig) big_pairs += double(na) * nsrc(b);
                if (sl == 4) continue;
                const int32_t y = nsrc(b);
                if (!(na > y || (na == y && a < b))) continue;
                nc += y;
                cost_one += 2.0 * double(na) * y * 31.0 / 32.0;
            }
            cost_one += double(na) * na * 31.0 / 32.0;
            total += double(na) * nc;
            cost_sym += double((na + (rows2_of(na) ? 63 : 31)) / (rows2_of(na) ? 64 : 32)) * ((nc + 31) / 32) * 32.0 * (rows2_of(na) ? 56.0 : 31.0) + 150.0;
        }
        // measured: cfg4 (256 per leaf) model 0.50 -> near field 0.64x; cfg2
        // (16..337 per leaf) model 0.76 -> 1.37x when every pair goes
        // symmetric (staging latency, tile quantisation of the small leaves)
        // The hybrid form (VPG_SYM_MIN=T) measured slower on cfg2 too (near field
        // 0.204 ms one-sided vs 0.225 / 0.243 / 0.252 ms at T = 32 / 64 / 96,
        // with 82% / 79% / 54% of the pairs symmetric), so it is opt-in only.
        (void)big_pairs;
        (void)all_pairs;
        if (pl.family != VPG_LAPLACE) pl.sym_min = 0;  // K0 pairs (~40 FP64 instructions) dwarf the tile overheads
        else if (tmin >= 0) pl.sym_min = tmin;
        else if (cost_sym < 0.6 * cost_one) pl.sym_min = 0;
        else pl.sym_min = -1;
        // subtasks of about half one warp's fair share (16 warps per SM)
        pl.sym_fair = std::max(4096.0, total / (double(pl.sm_count) * 16.0 * 2.0));
        pl.sym_chunk = int32_t(std::clamp(std::floor(pl.sym_fair / 64.0 / 32.0) * 32.0, 32.0, 8192.0));
        if (const char* cv = std::getenv("VPG_SYM_CHUNK")) pl.sym_chunk = std::max(32, std::atoi(cv) / 32 * 32);
    }
    if (pl.sym_min < 0 && force != 1) return;
    const int32_t T = std::max(0, pl.sym_min);
    const bool hybrid = T > 0;
    auto big = [&](int64_t a) { return nsrc(a) > 0 && nsrc(a) >= T; };
    // the owner of a symmetric pair {A, B}: the larger leaf, ties to the smaller Morton id
    auto owns = [&](int64_t a, int64_t b) {
        const int32_t x = nsrc(a), y = nsrc(b);
        return big(a) && big(b) && (x > y || (x == y && a < b));
    };
    std::vector<int32_t> ncol(size_t(nleaf), 0);
    for (int64_t a = 0; a < nleaf; ++a) {
        if (!big(a)) continue;
        int32_t nc = nsrc(a);
        for (int sl = 0; sl < 9; ++sl) {
            const int64_t b = sl == 4 ? -1 : neighbour(a, sl);
            if (b >= 0 && owns(a, b)) nc += nsrc(b);
        }
        ncol[size_t(a)] = nc;
    }
    const int32_t C = std::max(32, pl.sym_chunk);
    auto ncc_of = [&](int64_t a) { return (ncol[size_t(a)] + C - 1) / C; };
    // a leaf's chunks are balanced: ncc chunks of ceil(ncol / ncc) columns rounded up to tiles
    // (cfg4: 1280 columns as 448 + 448 + 384, not 544 + 544 + 192: near field 4.89 -> 4.83 ms)
    auto cw_of = [&](int64_t a) {
        const int32_t k = std::max(1, ncc_of(a));
        return std::min(C, ((ncol[size_t(a)] + k - 1) / k + 31) / 32 * 32);
    };
    // row tiles per group: as many as keep group rows x chunk columns near the share
    auto gsz_of = [&](int64_t a) {
        const int32_t na = nsrc(a);
        const double tile = double(32 << rsel_of(na)) * std::min(C, ncol[size_t(a)]);
        return std::clamp(int32_t(pl.sym_fair / tile), 1, nrt_of(na));
    };
    auto nrg_of = [&](int64_t a) { return (nrt_of(nsrc(a)) + gsz_of(a) - 1) / gsz_of(a); };
    // slot layout per big leaf (own chunks, own row groups, then per owning
    // neighbour in slot order its row groups) and partial bases
    std::vector<int32_t> nslot(size_t(nleaf), 0);
    std::vector<int64_t> pbase(size_t(nleaf) + 1, 0);
    for (int64_t a = 0; a < nleaf; ++a) {
        const int32_t na = nsrc(a);
        if (big(a)) {
            int32_t k = ncc_of(a) + nrg_of(a);
            for (int sl = 0; sl < 9; ++sl) {
                const int64_t b = sl == 4 ? -1 : neighbour(a, sl);
                if (b >= 0 && owns(b, a)) k += nrg_of(b);
            }
            nslot[size_t(a)] = k;
        }
        pbase[size_t(a) + 1] = pbase[size_t(a)] + int64_t(na) * nslot[size_t(a)];
    }
    // first column slot of owner a in leaf b (b's own slots, then its owners in slot order)
    auto col_slot = [&](int64_t b, int64_t a) {
        int32_t k = ncc_of(b) + nrg_of(b);
        for (int sl = 0; sl < 9; ++sl) {
            const int64_t o = sl == 4 ? -1 : neighbour(b, sl);
            if (o < 0 || !owns(o, b)) continue;
            if (o == a) return k;
            k += nrg_of(o);
        }
        return -1;
    };
    std::vector<SymTask> tasks;
    std::vector<SymRange> ranges;
    std::vector<SymLeaf> leaves;
    for (int64_t a = 0; a < nleaf; ++a) {
        const int32_t na = nsrc(a);
        if (!big(a)) continue;
        std::vector<SymRange> mine{SymRange{so[size_t(a)], 0, na, 0,
                                            pbase[size_t(a)] + int64_t(ncc_of(a)) * na}};
        bool touches = in(a);
        int32_t off = na;
        for (int sl = 0; sl < 9; ++sl) {
            const int64_t b = sl == 4 ? -1 : neighbour(a, sl);
            if (b < 0 || !owns(a, b)) continue;
            mine.push_back(SymRange{so[size_t(b)], off, nsrc(b), 0,
                                    pbase[size_t(b)] + int64_t(col_slot(b, a)) * nsrc(b)});
            off += nsrc(b);
            touches = touches || in(b);
        }
        if (!touches) continue;
        const int r2 = rsel_of(na);
        const int32_t rows = (32 << r2) * gsz_of(a);
        const int32_t rfirst = int32_t(ranges.size());
        ranges.insert(ranges.end(), mine.begin(), mine.end());
        for (int32_t rg = 0; rg < nrg_of(a); ++rg)
            for (int32_t cc = 0; cc < ncc_of(a); ++cc)
                tasks.push_back(SymTask{so[size_t(a)], na, rg * rows, std::min(na, (rg + 1) * rows), cc * cw_of(a),
                                        std::min(ncol[size_t(a)], (cc + 1) * cw_of(a)), rfirst, int32_t(mine.size()),
                                        pbase[size_t(a)] + int64_t(cc) * na, rg, r2});
    }
    // full form: every leaf of the range with targets -- matched ones from
    // the slots, unmatched ones one-sided (sym_finalize_kernel).  Hybrid: the
    // big leaves' matched targets add their slots to what the one-sided
    // kernel wrote (out +=); that kernel takes every target, over the 3x3
    // ranges minus the symmetric pairs (big leaves' matched targets) or all
    // of them (small leaves, unmatched targets).
    std::vector<P2PChunk> hyb;
    std::vector<int2> hranges;
    pl.sym_unmatched = false;
    for (const LeafNear& ln : pl.h_leafnear) {
        const int64_t x = ln.leaf;
        const int32_t na = nsrc(x);
        if (!hybrid && ln.t0 + na < ln.t1) pl.sym_unmatched = true;
        if (!hybrid || big(x))
            leaves.push_back(SymLeaf{pbase[size_t(x)], ln.t0, hybrid ? na : na, nslot[size_t(x)], ln.t1, ln.rfirst,
                                     ln.rcount, ln.lfirst, ln.lcount});
        if (!hybrid) continue;
        for (int part = 0; part < 2; ++part) {  // 0: matched targets, 1: unmatched
            const int32_t t0 = part == 0 ? ln.t0 : ln.t0 + na, t1 = part == 0 ? ln.t0 + na : ln.t1;
            if (t1 <= t0) continue;
            const int32_t rfirst = int32_t(hranges.size());
            int32_t rself = 0;
            int64_t near_src = 0;
            const int ix = int(squash2(uint32_t(x))), iy = int(squash2(uint32_t(x) >> 1));
            for (int jy = std::max(0, iy - 1); jy <= std::min(nb - 1, iy + 1); ++jy)  // summation.cpp:330-334
                for (int jx = std::max(0, ix - 1); jx <= std::min(nb - 1, ix + 1); ++jx) {
                    const int64_t y = mort(uint32_t(jx), uint32_t(jy));
                    if (part == 0 && big(x) && big(y)) continue;  // symmetric pair
                    if (jx == ix && jy == iy) rself = int32_t(hranges.size()) - rfirst;
                    hranges.push_back(make_int2(so[size_t(y)], nsrc(y)));
                    near_src += nsrc(y);
                }
            const int32_t rcount = int32_t(hranges.size()) - rfirst;
            for (int32_t t = t0; t < t1; t += 64)
                hyb.push_back(P2PChunk{t, std::min(64, t1 - t), int32_t(std::min<int64_t>(near_src, INT32_MAX)), rfirst,
                                       rcount, rself, ln.lfirst, ln.lcount, 0, 1, -1, -1});
        }
    }
    if (hybrid) {
        auto ccost = [](const P2PChunk& c) { return int64_t(c.pad) * c.tcount; };
        std::stable_sort(hyb.begin(), hyb.end(),
                         [&](const P2PChunk& a, const P2PChunk& b) { return ccost(a) > ccost(b); });
        to_device(pl.hyb_chunks, hyb, 0);
        to_device(pl.hyb_ranges, hranges, 0);
    }
    pl.n_hyb_chunks = hybrid ? int64_t(hyb.size()) : 0;
    pl.sym_hybrid = hybrid;
    auto cost = [](const SymTask& t) { return int64_t(t.c1 - t.c0) * (t.r1 - t.r0); };
    std::stable_sort(tasks.begin(), tasks.end(),
                     [&](const SymTask& x, const SymTask& y) { return cost(x) > cost(y); });
    pl.sym_nparts = pbase.back();
    cudaStream_t st = 0;
    to_device(pl.sym_tasks, tasks, st);
    to_device(pl.sym_ranges, ranges, st);
    to_device(pl.sym_leaves, leaves, st);
    pl.n_sym_tasks = int64_t(tasks.size());
    pl.n_sym_leaves = int64_t(leaves.size());
    pl.sym_l2p_single = true;
    // (and no leaf so large that a warp per leaf unbalances the Horner work: cfg3's 4,096-point
    // leaves measured 20.2 -> 20.5 ms fused)
    for (const SymLeaf& lf : leaves) pl.sym_l2p_single = pl.sym_l2p_single && lf.lcount == 1 && lf.n <= 512;
    pl.sym = true;
}

}  // namespace vpg
