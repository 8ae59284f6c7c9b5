// adaptive.cu -- adaptive quadtree (VPG_MODE_NATIVE) built on the device.
//
// The reference tree is uniform (summation.cpp:580-585, depth capped at 7),
// so point sets concentrated in a small region (BASELINE cfg3: refinement
// to level 10 around a sharp source) put thousands of points in one leaf
// and the near field explodes.  This is the new
// adaptive build (no reference counterpart; parity is to the requested
// tolerance against direct sums):
//
//   1. Morton keys at depth 16 for sources and targets (same bounding box
//      rule as the reference, summation.cpp:560-585); stable radix sort.
//   2. Level-by-level refinement on the device: a box is split while it
//      holds more than kLeafCap sources or targets (and always above level
//      2); its point ranges are binary searches in the sorted keys, so every
//      box owns a contiguous range.  Empty children are not created.
//   3. Interaction lists (Carrier-Greengard-Rokhlin), one device thread per
//      box, two passes (count, fill), then sorted by (owner, partner) so the
//      order -- and therefore every sum -- is deterministic:
//        V(B)  children of the parent's colleagues not adjacent to B (M2L),
//        U(B)  leaves adjacent to leaf B, any level, B itself included (P2P),
//        W(B)  boxes below B's colleagues that are not adjacent to B but
//              whose parent is (M2P: their multipole at B's targets),
//        X(B)  the dual of W (P2L: a coarser leaf's sources into B's local).
//   4. Host schedules from the lists (M2L batches, near-field chunks, M2P and
//      P2L work, multilevel P2M items).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "plan.cuh"

namespace vpg {
namespace {

constexpr int kDepth = 16;     // 32-bit Morton keys
constexpr int kLeafCap = 96;   // points per leaf (sources or targets); VPG_LEAF_CAP overrides
                               // (sweep: 96 best on cfg2, ties 64 on cfg3 / cfg4)
constexpr int kL2PChainCap = 256;  // rows with more targets push their local down (L2L)

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

__global__ void keys16(const double2* pts, int64_t n, double x0, double y0, double side,
                       uint32_t* keys, int32_t* ids) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int nb = 1 << kDepth;
    const double2 p = pts[j];
    int ix = __double2int_rz(__dmul_rn(__ddiv_rn(__dsub_rn(p.x, x0), side), double(nb)));
    int iy = __double2int_rz(__dmul_rn(__ddiv_rn(__dsub_rn(p.y, y0), side), double(nb)));
    ix = min(max(ix, 0), nb - 1);
    iy = min(max(iy, 0), nb - 1);
    keys[j] = mort(uint32_t(ix), uint32_t(iy));
    ids[j] = int32_t(j);
}

__device__ inline int lbound(const uint32_t* k, int n, uint64_t v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uint64_t(k[mid]) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// One level of refinement: point ranges, split decision, non-empty children.
__global__ void level_pass(const uint32_t* sk, int ns, const uint32_t* tk, int nt,
                           const int32_t* morton, int nbox, int level, int4* rng,
                           int32_t* cmask, int32_t* nchild, int cap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbox) return;
    const uint64_t m = uint32_t(morton[i]);
    const int sh = 2 * (kDepth - level);
    const uint64_t lo = m << sh, hi = (m + 1) << sh;
    const int sb = lbound(sk, ns, lo), se = lbound(sk, ns, hi);
    const int tb = lbound(tk, nt, lo), te = lbound(tk, nt, hi);
    rng[i] = make_int4(sb, se, tb, te);
    const bool split = level < kDepth && (level < 2 || se - sb > cap || te - tb > cap);
    int mask = 0, cnt = 0;
    if (split) {
        for (int c = 0; c < 4; ++c) {
            const uint64_t clo = ((m << 2) | uint64_t(c)) << (sh - 2), chi = clo + (uint64_t(1) << (sh - 2));
            const int a = lbound(sk, ns, clo), b = lbound(sk, ns, chi);
            const int x = lbound(tk, nt, clo), y = lbound(tk, nt, chi);
            if (b > a || y > x) {
                mask |= 1 << c;
                ++cnt;
            }
        }
    }
    cmask[i] = mask;
    nchild[i] = cnt;
}

__global__ void emit_children(const int32_t* morton, const int32_t* cmask, const int64_t* cpos,
                              int nbox, int32_t* next_morton) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbox) return;
    const int mask = cmask[i];
    int64_t o = cpos[i];
    for (int c = 0; c < 4; ++c)
        if (mask & (1 << c)) next_morton[o++] = int32_t((uint32_t(morton[i]) << 2) | uint32_t(c));
}

// ------------------------------------------------------------ list kernels --
struct TreeView {
    const int32_t* level;
    const int32_t* morton;
    const int32_t* first_child;  // row of the first child, -1 for leaves
    const int32_t* cmask;
    const int4* rng;             // (src b, src e, tgt b, tgt e)
    const int64_t* lvl_first;    // [depth + 2]
    int depth;
};

__device__ inline int find_row(const TreeView& tv, int level, int ix, int iy) {
    if (level > tv.depth) return -1;
    const int n = 1 << level;
    if (ix < 0 || iy < 0 || ix >= n || iy >= n) return -1;
    const uint32_t m = mort(uint32_t(ix), uint32_t(iy));
    int lo = int(tv.lvl_first[level]), hi = int(tv.lvl_first[level + 1]);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uint32_t(tv.morton[mid]) < m) lo = mid + 1; else hi = mid;
    }
    return (lo < tv.lvl_first[level + 1] && uint32_t(tv.morton[lo]) == m) ? lo : -1;
}

__device__ inline int child_row(const TreeView& tv, int r, int c) {
    const int mask = tv.cmask[r];
    if (!(mask & (1 << c))) return -1;
    return tv.first_child[r] + __popc(mask & ((1 << c) - 1));
}

__device__ inline bool nsrc(const TreeView& tv, int r) { return tv.rng[r].y > tv.rng[r].x; }
__device__ inline bool ntgt(const TreeView& tv, int r) { return tv.rng[r].w > tv.rng[r].z; }

// Boxes (l1, a) and (l2, e) with l2 >= l1 touch (share an edge or corner)?
__device__ inline bool touches(int l1, int ax, int ay, int l2, int ex, int ey) {
    const int k = 1 << (l2 - l1);
    return ex >= ax * k - 1 && ex <= (ax + 1) * k && ey >= ay * k - 1 && ey <= (ay + 1) * k;
}

// V lists: children of the parent's colleagues, not adjacent (same level).
template <bool kFill>
__global__ void vlist_kernel(TreeView tv, int nrows, int32_t* vcount, const int64_t* vpos,
                             int32_t* vsrc, int32_t* voidx) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int l = tv.level[r];
    int cnt = 0;
    int64_t e = kFill ? vpos[r] : 0;
    if (l >= 2 && ntgt(tv, r)) {
        const uint32_t m = uint32_t(tv.morton[r]);
        const int ix = int(squash2(m)), iy = int(squash2(m >> 1));
        const int px = ix >> 1, py = iy >> 1;
        for (int qy = py - 1; qy <= py + 1; ++qy)
            for (int qx = px - 1; qx <= px + 1; ++qx) {
                const int q = find_row(tv, l - 1, qx, qy);
                if (q < 0 || tv.first_child[q] < 0) continue;
                for (int c = 0; c < 4; ++c) {
                    const int jx = 2 * qx + (c & 1), jy = 2 * qy + ((c & 2) >> 1);
                    const int dx = jx - ix, dy = jy - iy;
                    if (max(abs(dx), abs(dy)) < 2) continue;
                    const int s = child_row(tv, q, c);
                    if (s < 0 || !nsrc(tv, s)) continue;
                    if (kFill) {
                        vsrc[e] = s;
                        voidx[e] = (dx + 3) + 7 * (dy + 3);
                        ++e;
                    } else {
                        ++cnt;
                    }
                }
            }
    }
    if (!kFill) vcount[r] = cnt;
}

// U / W / X pair generation from leaf B's point of view (descent into the
// colleagues' subtrees); inverse U pairs (finer adjacent leaf -> B) and X
// pairs (W dual) are emitted here too, so every pair is produced once.
constexpr int kKindU = 0, kKindW = 1, kKindX = 2;

template <bool kFill>
__global__ void uwx_kernel(TreeView tv, int nrows, int32_t* count, const int64_t* pos,
                           unsigned long long* rec) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nrows) return;
    int cnt = 0;
    int64_t o = kFill ? pos[b] : 0;
    auto emit = [&](int kind, int owner, int partner) {
        if (kFill) rec[o++] = (static_cast<unsigned long long>(kind) << 62) |
                              (static_cast<unsigned long long>(owner) << 31) |
                              static_cast<unsigned long long>(partner);
        else ++cnt;
    };
    if (tv.first_child[b] < 0) {  // leaf
        const int l = tv.level[b];
        const uint32_t m = uint32_t(tv.morton[b]);
        const int ix = int(squash2(m)), iy = int(squash2(m >> 1));
        const bool bt = ntgt(tv, b), bs = nsrc(tv, b);
        if (bt && bs) emit(kKindU, b, b);
        int stack[4 * 18];
        for (int cy = iy - 1; cy <= iy + 1; ++cy)
            for (int cx = ix - 1; cx <= ix + 1; ++cx) {
                if (cx == ix && cy == iy) continue;
                const int c = find_row(tv, l, cx, cy);
                if (c < 0) continue;
                if (tv.first_child[c] < 0) {  // same-level leaf: symmetric, emit own side only
                    if (bt && nsrc(tv, c)) emit(kKindU, b, c);
                    continue;
                }
                int top = 0;
                for (int k = 3; k >= 0; --k) {
                    const int e = child_row(tv, c, k);
                    if (e >= 0) stack[top++] = e;
                }
                while (top > 0) {
                    const int e = stack[--top];
                    const int el = tv.level[e];
                    const uint32_t em = uint32_t(tv.morton[e]);
                    const int ex = int(squash2(em)), ey = int(squash2(em >> 1));
                    if (touches(l, ix, iy, el, ex, ey)) {
                        if (tv.first_child[e] < 0) {
                            if (bt && nsrc(tv, e)) emit(kKindU, b, e);
                            if (bs && ntgt(tv, e)) emit(kKindU, e, b);  // inverse (finer side)
                        } else {
                            for (int k = 3; k >= 0; --k) {
                                const int f = child_row(tv, e, k);
                                if (f >= 0) stack[top++] = f;
                            }
                        }
                    } else {
                        if (bt && nsrc(tv, e)) emit(kKindW, b, e);  // M2P: e's multipole at b
                        if (bs && ntgt(tv, e)) emit(kKindX, e, b);  // P2L: b's sources into e
                    }
                }
            }
    }
    if (!kFill) count[b] = cnt;
}

__global__ void gather_xy(const double2* pts, const int32_t* ids, int64_t n, double2* out) {
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e < n) out[e] = pts[ids[e]];
}

void gather_sorted(const double2* pts, const int32_t* ids, int64_t n, double2* out, cudaStream_t st) {
    gather_xy<<<nblk(n, 256), 256, 0, st>>>(pts, ids, n, out);
    VPG_LAUNCH_CHECK();
}

template <typename T>
std::vector<T> d2h(const T* p, size_t n, cudaStream_t st) {
    std::vector<T> h(n);
    if (n) VPG_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    VPG_CUDA(cudaStreamSynchronize(st));
    return h;
}
template <typename T>
void h2d(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
    d.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty()) VPG_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    VPG_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void exclusive_scan(const T* in, int64_t* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, int(n), st);
    DBuf<unsigned char> tmp;
    tmp.alloc(std::max<size_t>(bytes, 1));
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, int(n), st));
}

void sort_by_key16(const double2* pts, int64_t n, const Plan& pl, DBuf<uint32_t>& skeys,
                   DBuf<int32_t>& ids_out, DBuf<double2>& sorted, cudaStream_t st) {
    DBuf<uint32_t> keys;
    DBuf<int32_t> ids;
    const size_t m = size_t(std::max<int64_t>(n, 1));
    keys.alloc(m);
    ids.alloc(m);
    skeys.alloc(m);
    ids_out.alloc(m);
    sorted.alloc(m);
    if (n == 0) return;
    keys16<<<nblk(n, 256), 256, 0, st>>>(pts, n, pl.x0, pl.y0, pl.side, keys.p, ids.p);
    VPG_LAUNCH_CHECK();
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, skeys.p, ids.p, ids_out.p, int(n), 0, 32, st);
    DBuf<unsigned char> tmp;
    tmp.alloc(std::max<size_t>(bytes, 1));
    VPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, skeys.p, ids.p, ids_out.p, int(n), 0, 32, st));
    gather_sorted(pts, ids_out.p, n, sorted.p, st);
}

}  // namespace

int leaf_cap() {
    static const int cap = [] {
        const char* v = std::getenv("VPG_LEAF_CAP");
        const int c = v ? std::atoi(v) : 0;
        return c > 0 ? c : kLeafCap;
    }();
    return cap;
}

void build_adaptive(Plan& pl, cudaStream_t st) {
    pl.adaptive = true;
    pl.multilevel_up = pl.multilevel_down = false;  // hybrid passes (schedules below)
    DBuf<uint32_t> sk, tk;
    sort_by_key16(pl.src.p, pl.ns, pl, sk, pl.src_ids, pl.src_sorted, st);
    sort_by_key16(pl.tgt.p, pl.nt, pl, tk, pl.tgt_ids, pl.tgt_sorted, st);

    // ---- level-by-level refinement
    std::vector<int32_t> h_morton, h_level, h_cmask, h_first;
    std::vector<int4> h_rng;
    std::vector<int64_t> lvl_first{0};
    DBuf<int32_t> cur;
    h2d(cur, std::vector<int32_t>{0}, st);
    int64_t ncur = 1;
    int depth = 0;
    for (int level = 0; ncur > 0; ++level) {
        DBuf<int4> rng;
        DBuf<int32_t> cmask, nchild;
        DBuf<int64_t> cpos;
        rng.alloc(size_t(ncur));
        cmask.alloc(size_t(ncur));
        nchild.alloc(size_t(ncur));
        cpos.alloc(size_t(ncur));
        level_pass<<<nblk(ncur, 128), 128, 0, st>>>(sk.p, int(pl.ns), tk.p, int(pl.nt), cur.p, int(ncur),
                                                     level, rng.p, cmask.p, nchild.p, leaf_cap());
        VPG_LAUNCH_CHECK();
        exclusive_scan(nchild.p, cpos.p, ncur, st);
        const std::vector<int32_t> m = d2h(cur.p, size_t(ncur), st);
        const std::vector<int4> r = d2h(rng.p, size_t(ncur), st);
        const std::vector<int32_t> cm = d2h(cmask.p, size_t(ncur), st);
        const std::vector<int32_t> nc = d2h(nchild.p, size_t(ncur), st);
        const std::vector<int64_t> cp = d2h(cpos.p, size_t(ncur), st);
        const int64_t nnext = cp.back() + nc.back();
        const int64_t next_first = lvl_first.back() + ncur;
        for (int64_t i = 0; i < ncur; ++i) {
            h_morton.push_back(m[size_t(i)]);
            h_level.push_back(level);
            h_rng.push_back(r[size_t(i)]);
            h_cmask.push_back(cm[size_t(i)]);
            h_first.push_back(cm[size_t(i)] ? int32_t(next_first + cp[size_t(i)]) : -1);
        }
        lvl_first.push_back(next_first);
        depth = level;
        if (nnext == 0) break;
        DBuf<int32_t> next;
        next.alloc(size_t(nnext));
        emit_children<<<nblk(ncur, 128), 128, 0, st>>>(cur.p, cmask.p, cpos.p, int(ncur), next.p);
        VPG_LAUNCH_CHECK();
        VPG_CUDA(cudaStreamSynchronize(st));
        std::swap(cur.p, next.p);
        std::swap(cur.n, next.n);
        ncur = nnext;
    }
    const int64_t nrows = int64_t(h_morton.size());
    if (nrows > INT32_MAX / 2) throw Error{VPG_ERR_INVALID_ARGUMENT, "adaptive tree too large"};
    pl.L = depth;
    pl.n_rows = nrows;
    lvl_first.push_back(lvl_first.back());  // sentinel for find_row at depth + 1
    std::vector<int32_t> h_parent(size_t(nrows), -1);
    for (int64_t r = 0; r < nrows; ++r)
        if (h_first[size_t(r)] >= 0)
            for (int c = 0, k = 0; c < 4; ++c)
                if (h_cmask[size_t(r)] & (1 << c))
                    h_parent[size_t(h_first[size_t(r)] + k++)] = h_level[size_t(r)] >= 2 ? int32_t(r) : -1;
    h2d(pl.row_level, h_level, st);
    h2d(pl.row_morton, h_morton, st);
    h2d(pl.row_parent, h_parent, st);
    DBuf<int32_t> first_child, cmask_d;
    DBuf<int4> rng_d;
    DBuf<int64_t> lvl_first_d;
    h2d(first_child, h_first, st);
    h2d(cmask_d, h_cmask, st);
    h2d(rng_d, h_rng, st);
    h2d(lvl_first_d, lvl_first, st);
    const TreeView tv{pl.row_level.p, pl.row_morton.p, first_child.p, cmask_d.p, rng_d.p, lvl_first_d.p, depth};

    // target leaf row of every sorted target
    {
        std::vector<int32_t> trow(size_t(std::max<int64_t>(pl.nt, 1)), 0);
        for (int64_t r = 0; r < nrows; ++r)
            if (h_first[size_t(r)] < 0)
                for (int e = h_rng[size_t(r)].z; e < h_rng[size_t(r)].w; ++e) trow[size_t(e)] = int32_t(r);
        h2d(pl.tgt_row, trow, st);
    }

    // ---- V lists (M2L), two passes
    {
        DBuf<int32_t> vcount;
        DBuf<int64_t> vpos;
        vcount.alloc(size_t(nrows));
        vpos.alloc(size_t(nrows));
        vlist_kernel<false><<<nblk(nrows, 128), 128, 0, st>>>(tv, int(nrows), vcount.p, nullptr, nullptr, nullptr);
        VPG_LAUNCH_CHECK();
        exclusive_scan(vcount.p, vpos.p, nrows, st);
        const std::vector<int32_t> vc = d2h(vcount.p, size_t(nrows), st);
        const std::vector<int64_t> vp = d2h(vpos.p, size_t(nrows), st);
        const int64_t nv = vp.back() + vc.back();
        DBuf<int32_t> vsrc, voidx;
        vsrc.alloc(size_t(std::max<int64_t>(nv, 1)));
        voidx.alloc(size_t(std::max<int64_t>(nv, 1)));
        vlist_kernel<true><<<nblk(nrows, 128), 128, 0, st>>>(tv, int(nrows), nullptr, vpos.p, vsrc.p, voidx.p);
        VPG_LAUNCH_CHECK();
        // target-box CSR over rows with targets at levels >= 2, batches
        std::vector<int32_t> tbox;
        std::vector<M2LBatch> batches;
        M2LBatch curb{};
        bool open = false;
        for (int64_t r = 0; r < nrows; ++r) {
            const int l = h_level[size_t(r)];
            if (l < 2 || h_rng[size_t(r)].w <= h_rng[size_t(r)].z) continue;
            const int32_t ne = vc[size_t(r)];
            if (open && (l != curb.level || curb.ecount + ne > kM2LPairs)) {
                batches.push_back(curb);
                open = false;
            }
            if (!open) {
                curb = M2LBatch{l, int32_t(tbox.size()), 0, int32_t(vp[size_t(r)]), 0};
                open = true;
            }
            tbox.push_back(int32_t(r));
            curb.tcount += 1;
            curb.ecount += ne;
        }
        if (open) batches.push_back(curb);
        // toff must be the CSR of the kept boxes: entries of skipped rows are
        // empty (no targets -> no V entries), so vp is contiguous over them
        pl.n_tbox = int64_t(tbox.size());
        pl.n_m2l = nv;
        pl.shard_m2l = nv;
        h2d(pl.m2l_tbox, tbox, st);
        std::vector<int32_t> toff_fixed(tbox.size() + 1);
        for (size_t i = 0; i < tbox.size(); ++i) toff_fixed[i] = int32_t(vp[size_t(tbox[i])]);
        toff_fixed[tbox.size()] = int32_t(nv);
        h2d(pl.m2l_toff, toff_fixed, st);
        pl.m2l_src.alloc(vsrc.n);
        pl.m2l_oidx.alloc(voidx.n);
        std::swap(pl.m2l_src.p, vsrc.p);
        std::swap(pl.m2l_oidx.p, voidx.p);
        pl.n_m2l_batches = int64_t(batches.size());
        h2d(pl.m2l_batches, batches, st);
        pl.ad_vc = vc;
        pl.ad_vp = vp;
        pl.ad_nv = nv;
    }

    // ---- U / W / X pairs, sorted by (kind, owner, partner)
    std::vector<int64_t> uoff, woff, xoff;
    std::vector<int32_t> upart, wpart, xpart;
    {
        DBuf<int32_t> cnt;
        DBuf<int64_t> pos;
        cnt.alloc(size_t(nrows));
        pos.alloc(size_t(nrows));
        uwx_kernel<false><<<nblk(nrows, 128), 128, 0, st>>>(tv, int(nrows), cnt.p, nullptr, nullptr);
        VPG_LAUNCH_CHECK();
        exclusive_scan(cnt.p, pos.p, nrows, st);
        const std::vector<int32_t> c = d2h(cnt.p, size_t(nrows), st);
        const std::vector<int64_t> p = d2h(pos.p, size_t(nrows), st);
        const int64_t nrec = p.back() + c.back();
        DBuf<unsigned long long> rec, srec;
        rec.alloc(size_t(std::max<int64_t>(nrec, 1)));
        srec.alloc(size_t(std::max<int64_t>(nrec, 1)));
        uwx_kernel<true><<<nblk(nrows, 128), 128, 0, st>>>(tv, int(nrows), nullptr, pos.p, rec.p);
        VPG_LAUNCH_CHECK();
        if (nrec > 0) {
            size_t bytes = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, bytes, rec.p, srec.p, int(nrec), 0, 64, st);
            DBuf<unsigned char> tmp;
            tmp.alloc(std::max<size_t>(bytes, 1));
            VPG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, rec.p, srec.p, int(nrec), 0, 64, st));
        }
        const std::vector<unsigned long long> h = d2h(srec.p, size_t(nrec), st);
        auto csr = [&](int kind, std::vector<int64_t>& off, std::vector<int32_t>& part) {
            off.assign(size_t(nrows + 1), 0);
            for (const unsigned long long v : h)
                if (int(v >> 62) == kind) ++off[size_t((v >> 31) & 0x7FFFFFFFull) + 1];
            for (int64_t r = 0; r < nrows; ++r) off[size_t(r + 1)] += off[size_t(r)];
            part.resize(size_t(off.back()));
            std::vector<int64_t> cur2(off.begin(), off.end() - 1);
            for (const unsigned long long v : h)
                if (int(v >> 62) == kind)
                    part[size_t(cur2[size_t((v >> 31) & 0x7FFFFFFFull)]++)] = int32_t(v & 0x7FFFFFFFull);
        };
        csr(kKindU, uoff, upart);
        csr(kKindW, woff, wpart);
        csr(kKindX, xoff, xpart);
    }

    // ---- schedules
    std::vector<int32_t> chain;  // L2P chain: next row a target evaluates (-1: done)
    {
        // Upward pass, hybrid: a row with at most kP2MItemCap sources gets its
        // multipole by P2M straight from its points (one warp item); a larger
        // non-leaf row by M2M from its children, level by level bottom-up
        // (cooperative shift kernel).  Each point then feeds ~2 rows instead
        // of every ancestor.  Oversized leaves (depth cap) are split into
        // items and reduced.
        std::vector<P2MItem> items;
        std::vector<P2MSplit> splits;
        for (int64_t r = 0; r < nrows; ++r) {
            const int l = h_level[size_t(r)];
            const int4 g = h_rng[size_t(r)];
            if (l < 2 || g.y <= g.x) continue;
            if (h_first[size_t(r)] >= 0 && g.y - g.x > kP2MItemCap) continue;  // M2M
            const int32_t pieces = (g.y - g.x + kP2MItemCap - 1) / kP2MItemCap;
            if (pieces > 1) splits.push_back(P2MSplit{int32_t(r), int32_t(items.size()), pieces});
            for (int32_t e = g.x; e < g.y; e += kP2MItemCap)
                items.push_back(P2MItem{l, h_morton[size_t(r)], int32_t(r), e, std::min(g.y, e + kP2MItemCap),
                                        pieces == 1 ? 1 : 0});
        }
        // M2M parents (bottom-up) then L2L parents (top-down), per level
        std::vector<int32_t> boxes;
        std::vector<int4> kids;
        pl.m2m_first.assign(size_t(depth + 1), 0);
        pl.m2m_count.assign(size_t(depth + 1), 0);
        pl.l2l_first.assign(size_t(depth + 1), 0);
        pl.l2l_count.assign(size_t(depth + 1), 0);
        pl.m2m_children = pl.l2l_children = 0;
        auto children = [&](int64_t r, bool tgt, int64_t& nkids) {
            int k4[4] = {-1, -1, -1, -1};
            for (int c = 0, k = 0; c < 4; ++c)
                if (h_cmask[size_t(r)] & (1 << c)) {
                    const int32_t cr = h_first[size_t(r)] + k++;
                    const int4 gc = h_rng[size_t(cr)];
                    if (tgt ? gc.w > gc.z : gc.y > gc.x) {
                        k4[c] = cr;
                        ++nkids;
                    }
                }
            return make_int4(k4[0], k4[1], k4[2], k4[3]);
        };
        for (int l = 2; l < depth; ++l) {
            pl.m2m_first[size_t(l)] = int64_t(boxes.size());
            for (int64_t r = lvl_first[size_t(l)]; r < lvl_first[size_t(l + 1)]; ++r) {
                const int4 g = h_rng[size_t(r)];
                if (h_first[size_t(r)] < 0 || g.y - g.x <= kP2MItemCap) continue;
                boxes.push_back(int32_t(r));
                kids.push_back(children(r, false, pl.m2m_children));
            }
            pl.m2m_count[size_t(l)] = int64_t(boxes.size()) - pl.m2m_first[size_t(l)];
        }
        std::vector<char> pushed(size_t(nrows), 0);
        for (int l = 2; l < depth; ++l) {
            pl.l2l_first[size_t(l)] = int64_t(boxes.size());
            for (int64_t r = lvl_first[size_t(l)]; r < lvl_first[size_t(l + 1)]; ++r) {
                const int4 g = h_rng[size_t(r)];
                if (h_first[size_t(r)] < 0 || g.w - g.z <= kL2PChainCap) continue;
                pushed[size_t(r)] = 1;
                boxes.push_back(int32_t(r));
                kids.push_back(children(r, true, pl.l2l_children));
            }
            pl.l2l_count[size_t(l)] = int64_t(boxes.size()) - pl.l2l_first[size_t(l)];
        }
        chain.assign(size_t(nrows), -1);
        for (int64_t r = 0; r < nrows; ++r) {
            const int32_t p = h_parent[size_t(r)];
            chain[size_t(r)] = (p >= 0 && !pushed[size_t(p)]) ? p : -1;
        }
        h2d(pl.updown_boxes, boxes, st);
        h2d(pl.updown_kids, kids, st);
        h2d(pl.row_chain, chain, st);
        pl.ad_ud_boxes = boxes;
        pl.ad_ud_kids = kids;
        pl.ad_m2m_first = pl.m2m_first;
        pl.ad_m2m_count = pl.m2m_count;
        pl.ad_l2l_first = pl.l2l_first;
        pl.ad_l2l_count = pl.l2l_count;
        pl.n_p2m_items = int64_t(items.size());
        pl.n_p2m_splits = int64_t(splits.size());
        h2d(pl.p2m_items, items, st);
        h2d(pl.p2m_splits, splits, st);
    }
    {
        // near field: U lists as source ranges
        std::vector<P2PChunk> chunks;
        std::vector<int2> ranges;
        std::vector<int32_t> lrows;
        pl.p2p_pairs = 0;
        int max_ranges = 0;
        for (int64_t r = 0; r < nrows; ++r) {
            const int4 g = h_rng[size_t(r)];
            if (h_first[size_t(r)] >= 0 || g.w <= g.z) continue;
            // U leaves as sorted-source ranges; Morton-adjacent leaves are
            // adjacent in the sorted arrays, so contiguous ranges merge (the
            // self fix-up then spans the merged range -- exact for any pair)
            std::vector<int2> rl;
            int64_t nsrc = 0;
            int32_t self_start = -1;
            for (int64_t k = uoff[size_t(r)]; k < uoff[size_t(r + 1)]; ++k) {
                const int32_t e = upart[size_t(k)];
                const int4 ge = h_rng[size_t(e)];
                if (ge.y <= ge.x) continue;
                if (e == r) self_start = ge.x;
                rl.push_back(make_int2(ge.x, ge.y - ge.x));
                nsrc += ge.y - ge.x;
            }
            // (a target leaf without near sources still gets a chunk: the
            // P2P pass is what writes out = far + near)
            std::sort(rl.begin(), rl.end(), [](const int2& a, const int2& b) { return a.x < b.x; });
            const int32_t rfirst = int32_t(ranges.size());
            int32_t rself = -1;
            for (const int2& v : rl) {
                if (ranges.size() > size_t(rfirst) && ranges.back().x + ranges.back().y == v.x)
                    ranges.back().y += v.y;
                else
                    ranges.push_back(v);
                if (v.x == self_start) rself = int32_t(ranges.size()) - 1 - rfirst;
            }
            const int32_t rcount = int32_t(ranges.size()) - rfirst;
            max_ranges = std::max(max_ranges, int(rcount));
            if (rself < 0) {  // target leaf without sources: no coincident pair possible
                ranges.push_back(make_int2(0, 0));
                rself = rcount;
            }
            pl.p2p_pairs += int64_t(g.w - g.z) * nsrc;
            const int32_t lfirst = int32_t(lrows.size());
            for (int32_t c = int32_t(r); c >= 0; c = chain[size_t(c)]) lrows.push_back(c);
            const int32_t lcount = int32_t(lrows.size()) - lfirst;
            for (int32_t t = g.z; t < g.w; t += 64)
                chunks.push_back(P2PChunk{t, std::min(64, g.w - t), int32_t(std::min<int64_t>(nsrc, INT32_MAX)),
                                          rfirst, int32_t(ranges.size()) - rfirst, rself, lfirst, lcount, 0, 1,
                                          -1, -1});
        }
        if (max_ranges + 1 > kMaxNearRanges)
            throw Error{VPG_ERR_INVALID_ARGUMENT,
                        "adaptive tree: a leaf has " + std::to_string(max_ranges) + " near leaves (max " +
                            std::to_string(kMaxNearRanges - 1) + ")"};
        pl.ad_chunks = chunks;
        schedule_near_chunks(pl, chunks);
        h2d(pl.p2p_chunks, chunks, st);
        h2d(pl.near_ranges, ranges, st);
        h2d(pl.l2p_rows, lrows, st);
    }
    {
        // M2P (W lists): chunks of 32 targets of a leaf
        std::vector<int4> work;  // (tbegin, tcount, wfirst, wcount)
        std::vector<int32_t> wrows;
        int64_t nw = 0;
        for (int64_t r = 0; r < nrows; ++r) {
            const int4 g = h_rng[size_t(r)];
            const int64_t w0 = woff[size_t(r)], w1 = woff[size_t(r + 1)];
            if (h_first[size_t(r)] >= 0 || g.w <= g.z || w1 == w0) continue;
            const int32_t first = int32_t(wrows.size());
            for (int64_t k = w0; k < w1; ++k) wrows.push_back(wpart[size_t(k)]);
            for (int32_t t = g.z; t < g.w; t += 32)
                work.push_back(make_int4(t, std::min(32, g.w - t), first, int32_t(w1 - w0)));
            nw += (w1 - w0) * (g.w - g.z);
        }
        pl.m2p_evals = nw;
        pl.n_m2p_work = int64_t(work.size());
        h2d(pl.m2p_work, work, st);
        pl.ad_m2p = work;
        h2d(pl.m2p_rows, wrows, st);
    }
    {
        // P2L (X lists): per receiving box, its X leaves as source ranges
        std::vector<int4> work;  // (row, rfirst, rcount, 0)
        std::vector<int2> ranges;
        int64_t np2l = 0;
        for (int64_t r = 0; r < nrows; ++r) {
            const int64_t x0 = xoff[size_t(r)], x1 = xoff[size_t(r + 1)];
            if (x1 == x0 || h_level[size_t(r)] < 2) continue;
            const int32_t first = int32_t(ranges.size());
            for (int64_t k = x0; k < x1; ++k) {
                const int4 ge = h_rng[size_t(xpart[size_t(k)])];
                ranges.push_back(make_int2(ge.x, ge.y - ge.x));
                np2l += ge.y - ge.x;
            }
            work.push_back(make_int4(int32_t(r), first, int32_t(ranges.size()) - first, 0));
        }
        pl.p2l_sources = np2l;
        pl.n_p2l_work = int64_t(work.size());
        h2d(pl.p2l_work, work, st);
        pl.ad_p2l = work;
        h2d(pl.p2l_ranges, ranges, st);
    }
    pl.ad_rng = h_rng;
    pl.ad_level = h_level;
    // shard units: leaves with targets, in target (Morton) order
    pl.ad_leaves.clear();
    for (int64_t r = 0; r < nrows; ++r)
        if (h_first[size_t(r)] < 0 && h_rng[size_t(r)].w > h_rng[size_t(r)].z) pl.ad_leaves.push_back(int32_t(r));
    std::sort(pl.ad_leaves.begin(), pl.ad_leaves.end(),
              [&](int32_t a, int32_t b) { return h_rng[size_t(a)].z < h_rng[size_t(b)].z; });
    pl.shard_lb = 0;
    pl.shard_le = int64_t(pl.ad_leaves.size());
    pl.shard_t0 = 0;
    pl.shard_t1 = pl.nt;
}

// Restricts the target side of an adaptive plan to the targets of the
// leaves [leaf_begin, leaf_end) of ad_leaves (a contiguous sorted-target
// range): near-field chunks and L2P chains, M2P work of those targets, M2L /
// P2L / L2L of every box whose target range meets it.  The upward pass stays
// whole.  The per-target arithmetic is unchanged, so the shards' outputs
// (0.0 elsewhere) sum to the single-plan result bit for bit.
void adaptive_set_targets(Plan& pl, int64_t leaf_begin, int64_t leaf_end) {
    cudaStream_t st = 0;
    const int64_t nl = int64_t(pl.ad_leaves.size());
    int32_t T0 = 0, T1 = 0;
    if (leaf_begin < leaf_end) {
        T0 = pl.ad_rng[size_t(pl.ad_leaves[size_t(leaf_begin)])].z;
        T1 = pl.ad_rng[size_t(pl.ad_leaves[size_t(leaf_end - 1)])].w;
    }
    if (leaf_begin == 0 && leaf_end == nl) {
        T0 = 0;
        T1 = int32_t(pl.nt);
    }
    auto meets = [&](int64_t r) {
        const int4 g = pl.ad_rng[size_t(r)];
        return g.w > g.z && g.z < T1 && g.w > T0;
    };
    // near field + L2P
    {
        std::vector<P2PChunk> chunks;
        pl.p2p_pairs = 0;
        for (const P2PChunk& c : pl.ad_chunks)
            if (c.tbegin >= T0 && c.tbegin < T1) {
                chunks.push_back(c);
                pl.p2p_pairs += int64_t(c.pad) * c.tcount;
            }
        schedule_near_chunks(pl, chunks);
        h2d(pl.p2p_chunks, chunks, st);
    }
    // M2L target boxes and batches (same packing rule as build_adaptive)
    {
        std::vector<int32_t> tbox, toff;
        std::vector<M2LBatch> batches;
        M2LBatch curb{};
        bool open = false;
        int64_t nent = 0;
        const int64_t nrows = int64_t(pl.ad_rng.size());
        for (int64_t r = 0; r < nrows; ++r) {
            const int l = pl.ad_level[size_t(r)];
            if (l < 2 || !meets(r)) continue;
            const int32_t ne = pl.ad_vc[size_t(r)];
            if (open && (l != curb.level || curb.ecount + ne > kM2LPairs)) {
                batches.push_back(curb);
                open = false;
            }
            if (!open) {
                curb = M2LBatch{l, int32_t(tbox.size()), 0, int32_t(pl.ad_vp[size_t(r)]), 0};
                open = true;
            }
            // a batch's entries must be contiguous: close it when this box's
            // entries do not follow the previous box's
            if (curb.tcount > 0 && int64_t(curb.efirst) + curb.ecount != pl.ad_vp[size_t(r)]) {
                batches.push_back(curb);
                curb = M2LBatch{l, int32_t(tbox.size()), 0, int32_t(pl.ad_vp[size_t(r)]), 0};
            }
            tbox.push_back(int32_t(r));
            toff.push_back(int32_t(pl.ad_vp[size_t(r)]));
            curb.tcount += 1;
            curb.ecount += ne;
            nent += ne;
        }
        if (open) batches.push_back(curb);
        // toff: CSR over the kept boxes (entry positions are the global ones)
        toff.push_back(tbox.empty() ? 0 : int32_t(pl.ad_vp[size_t(tbox.back())] + pl.ad_vc[size_t(tbox.back())]));
        pl.n_tbox = int64_t(tbox.size());
        pl.shard_m2l = nent;
        h2d(pl.m2l_tbox, tbox, st);
        h2d(pl.m2l_toff, toff, st);
        pl.n_m2l_batches = int64_t(batches.size());
        h2d(pl.m2l_batches, batches, st);
    }
    // L2L parents meeting the range (the M2M part is unchanged)
    {
        std::vector<int32_t> boxes;
        std::vector<int4> kids;
        const int L = pl.L;
        for (int l = 2; l < L; ++l) {
            pl.m2m_first[size_t(l)] = int64_t(boxes.size());
            const int64_t f = pl.ad_m2m_first[size_t(l)];
            for (int64_t i = f; i < f + pl.ad_m2m_count[size_t(l)]; ++i) {
                boxes.push_back(pl.ad_ud_boxes[size_t(i)]);
                kids.push_back(pl.ad_ud_kids[size_t(i)]);
            }
            pl.m2m_count[size_t(l)] = int64_t(boxes.size()) - pl.m2m_first[size_t(l)];
        }
        for (int l = 2; l < L; ++l) {
            pl.l2l_first[size_t(l)] = int64_t(boxes.size());
            const int64_t f = pl.ad_l2l_first[size_t(l)];
            for (int64_t i = f; i < f + pl.ad_l2l_count[size_t(l)]; ++i)
                if (meets(pl.ad_ud_boxes[size_t(i)])) {
                    boxes.push_back(pl.ad_ud_boxes[size_t(i)]);
                    kids.push_back(pl.ad_ud_kids[size_t(i)]);
                }
            pl.l2l_count[size_t(l)] = int64_t(boxes.size()) - pl.l2l_first[size_t(l)];
        }
        h2d(pl.updown_boxes, boxes, st);
        h2d(pl.updown_kids, kids, st);
    }
    // M2P and P2L
    {
        std::vector<int4> m2p, p2l;
        for (const int4& w : pl.ad_m2p)
            if (w.x >= T0 && w.x < T1) m2p.push_back(w);
        for (const int4& w : pl.ad_p2l)
            if (meets(w.x)) p2l.push_back(w);
        pl.n_m2p_work = int64_t(m2p.size());
        pl.n_p2l_work = int64_t(p2l.size());
        h2d(pl.m2p_work, m2p, st);
        h2d(pl.p2l_work, p2l, st);
    }
    pl.shard_lb = leaf_begin;
    pl.shard_le = leaf_end;
    pl.shard_t0 = T0;
    pl.shard_t1 = T1;
}

}  // namespace vpg
