// corr.cu -- the two dense-small steps either side of the FMM in
// VolumePotentialOperator::apply (potential.cpp:431-470):
//
//   correction apply (potential.cpp:446-462): out[t] += sum over the
//     target's blocks of pool_row . f[node_off[cell] ..].  Block-sparse CSR
//     over targets; one warp per target, lanes stride the row entries
//     (coalesced 8-byte loads of the row and of the f segment), fixed
//     butterfly reduction (deterministic).  Shared box-lattice rows
//     (potential.cpp:256-267) are stored once and stay L2-resident.
//   build_charges (potential.cpp:397-412): charges = src_wj o (O_type f_cell)
//     per cell; one CTA per cell, the cell's f samples in smem, one thread
//     per oversampled source node.
#include <algorithm>
#include <memory>
#include <map>
#include <vector>

#include "plan.cuh"

#include "maps.cuh"

namespace vpg {
namespace {

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

constexpr int kCorrWarps = 8;

__global__ void __launch_bounds__(kCorrWarps * 32)
corr_apply_kernel(int64_t nt, const int32_t* tlist, const int32_t* blk_off, const int32_t* blk_cell,
                  const int32_t* blk_pool, const int64_t* pool_off,
                  const double* pool_vals, const int32_t* node_off,
                  const double* f, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t ti = int64_t(blockIdx.x) * kCorrWarps + (threadIdx.x >> 5);
    if (ti >= nt) return;
    const int64_t t = tlist ? tlist[ti] : ti;
    double acc = 0.0;
    const int k0 = blk_off[t], k1 = blk_off[t + 1];
    for (int k = k0; k < k1; ++k) {
        const int pr = blk_pool[k];
        const int64_t r0 = pool_off[pr], len = pool_off[pr + 1] - r0;
        const double* row = pool_vals + r0;
        const double* fc = f + node_off[blk_cell[k]];
        for (int64_t e = lane; e < len; e += 32) acc = fma(__ldg(row + e), __ldg(fc + e), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[t] += acc;
}

// Lattice groups on the FP64 tensor cores: a CTA takes 64 groups (64
// targets each) and walks the shared 64 x 64 row blocks M_q: out[64g + u] +=
// sum_q sum_i M_q[u][i] f[cell(g, q) + i] as Y = M_q F_q (mma.sync m8n8k4),
// M_q and the tile's f segments staged in smem (strides == 4 mod 16).
template <int kLatTile>  // groups per CTA (64; 16 or 8 for small maps: more CTAs)
__global__ void __launch_bounds__(256)
corr_lattice_kernel(int64_t ngroups, int nmat, const int32_t* group, const int32_t* cellof,
                    const int64_t* moff, const double* pool_vals, const double* f, double* out) {
    constexpr int K = 64, kS = K + 4, kNT = kLatTile / 8;
    extern __shared__ __align__(16) double lsm[];
    double* ms = lsm;            // [u][i]
    double* fs = lsm + K * kS;   // [i][g]
    const int64_t g0 = int64_t(blockIdx.x) * kLatTile;
    const int ng = int(min(int64_t(kLatTile), ngroups - g0));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    double acc[kNT][2];
#pragma unroll
    for (int q = 0; q < kNT; ++q) acc[q][0] = acc[q][1] = 0.0;
    // register double buffer: the loads of block q+1 are in flight while
    // the DMMAs of block q run
    constexpr int kMR = K * K / 2 / 256, kFR = K * kLatTile / 256;
    double2 mreg[kMR];
    double freg[kFR];
    auto fetch = [&](int q) {
        const double2* mg = reinterpret_cast<const double2*>(pool_vals + moff[q]);
#pragma unroll
        for (int r = 0; r < kMR; ++r) mreg[r] = mg[threadIdx.x + 256 * r];
#pragma unroll
        for (int r = 0; r < kFR; ++r) {
            const int e = threadIdx.x + 256 * r, g = e / K, i = e % K;
            const int c = g < ng ? cellof[(g0 + g) * nmat + q] : -1;
            freg[r] = c >= 0 ? f[int64_t(c) + i] : 0.0;
        }
    };
    if (nmat > 0) fetch(0);
    for (int q = 0; q < nmat; ++q) {
        __syncthreads();  // the previous block's DMMAs are done with ms / fs
#pragma unroll
        for (int r = 0; r < kMR; ++r) {
            const int e = 2 * (threadIdx.x + 256 * r);
            *reinterpret_cast<double2*>(ms + (e / K) * kS + (e % K)) = mreg[r];
        }
#pragma unroll
        for (int r = 0; r < kFR; ++r) {
            const int e = threadIdx.x + 256 * r, g = e / K, i = e % K;
            fs[i * (kLatTile + 4) + g] = freg[r];
        }
        __syncthreads();
        if (q + 1 < nmat) fetch(q + 1);
#pragma unroll 4
        for (int k4 = 0; k4 < K; k4 += 4) {
            const double a = ms[(8 * warp + rq) * kS + k4 + kq];
#pragma unroll
            for (int n8 = 0; n8 < kNT; ++n8) {
                const double b = fs[(k4 + kq) * (kLatTile + 4) + 8 * n8 + rq];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(acc[n8][0]), "+d"(acc[n8][1])
                             : "d"(a), "d"(b));
            }
        }
    }
    // lane holds rows u = 8 warp + rq, groups 8 n8 + 2 kq + {0, 1}
    const int u = 8 * warp + rq;
#pragma unroll
    for (int n8 = 0; n8 < kNT; ++n8)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = 8 * n8 + 2 * kq + h;
            if (g < ng) out[int64_t(group[g0 + g]) * K + u] += acc[n8][h];
        }
}

__global__ void charges_kernel(const int32_t* cell_type, const int32_t* node_off,
                               const int32_t* src_off, const double* over0, int np0,
                               int nq0, const double* over1, int np1, int nq1,
                               const double* src_wj, const double* f, double* charges) {
    extern __shared__ double fsm[];
    const int64_t c = blockIdx.x;
    const bool t0 = cell_type[c] == 0;
    const int np = t0 ? np0 : np1, nq = t0 ? nq0 : nq1;
    const double* O = t0 ? over0 : over1;
    const int fb = node_off[c];
    for (int i = threadIdx.x; i < np; i += blockDim.x) fsm[i] = f[fb + i];
    __syncthreads();
    const int base = src_off[c];
    for (int s = threadIdx.x; s < nq; s += blockDim.x) {
        const double* row = O + int64_t(s) * np;
        double v = 0.0;
        for (int i = 0; i < np; ++i) v = fma(__ldg(row + i), fsm[i], v);
        charges[base + s] = src_wj[base + s] * v;
    }
}

template <typename T>
void upload(DBuf<T>& d, const T* h, size_t n) {
    d.alloc(n);
    if (n) VPG_CUDA(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
}

template <typename F>
int guarded_c(F&& f) {
    try {
        f();
        return VPG_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::exception& e) {
        set_error(e.what());
        return VPG_ERR_CUDA;
    }
}

struct OwnStream {
    cudaStream_t s = nullptr;
    bool owned = false;
    explicit OwnStream(void* u) {
        if (u) {
            s = static_cast<cudaStream_t>(u);
        } else {
            // blocking: orders after work already queued on the legacy
            // default stream (e.g. a q written there by the caller)
            VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamDefault));
            owned = true;
        }
    }
    ~OwnStream() {
        if (owned) cudaStreamDestroy(s);
    }
};

}  // namespace
}  // namespace vpg

using namespace vpg;

extern "C" {

int vpg_corr_create(int64_t nt, const int32_t* blk_off, int64_t nblocks,
                    const int32_t* blk_cell, const int32_t* blk_pool, int64_t npool,
                    const int64_t* pool_off, const double* pool_vals, int64_t ncell,
                    const int32_t* node_off, int device, vpg_corr** corr) {
    return guarded_c([&] {
        vpg::corr_create_impl(nt, blk_off, nblocks, blk_cell, blk_pool, npool, pool_off, pool_vals, false, ncell,
                              node_off, device, corr);
    });
}

}  // extern "C"

// The map from host structure arrays; pool_vals on the host, or already on
// the device (dev_pool: the rows built by vpg_corr_build, copied device to device).
void vpg::corr_create_impl(int64_t nt, const int32_t* blk_off, int64_t nblocks, const int32_t* blk_cell,
                           const int32_t* blk_pool, int64_t npool, const int64_t* pool_off,
                           const double* pool_vals, bool dev_pool, int64_t ncell, const int32_t* node_off,
                           int device, vpg_corr** corr) {
    {
        if (!corr) throw Error{VPG_ERR_INVALID_ARGUMENT, "corr is NULL"};
        *corr = nullptr;
        if (nt < 0 || nblocks < 0 || npool < 0 || ncell < 0 || !blk_off || !pool_off || !node_off ||
            (nblocks && (!blk_cell || !blk_pool)))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad correction arrays"};
        if (blk_off[0] != 0 || blk_off[nt] != nblocks)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "blk_off must run from 0 to nblocks"};
        for (int64_t t = 0; t < nt; ++t)
            if (blk_off[t + 1] < blk_off[t]) throw Error{VPG_ERR_INVALID_ARGUMENT, "blk_off not monotone"};
        const int64_t nvals = pool_off[npool];
        for (int64_t k = 0; k < nblocks; ++k) {
            if (blk_pool[k] < 0 || blk_pool[k] >= npool || blk_cell[k] < 0 || blk_cell[k] >= ncell)
                throw Error{VPG_ERR_INVALID_ARGUMENT, "block index out of range"};
            const int64_t len = pool_off[blk_pool[k] + 1] - pool_off[blk_pool[k]];
            if (node_off[blk_cell[k]] + len > node_off[ncell])
                throw Error{VPG_ERR_INVALID_ARGUMENT, "correction row overruns the cell's samples"};
        }
        if (nvals > 0 && !pool_vals) throw Error{VPG_ERR_INVALID_ARGUMENT, "pool_vals is NULL"};
        use_device(device);
        auto c = std::make_unique<vpg_corr>();
        c->device = device;
        c->nt = nt;
        c->nblocks = nblocks;
        c->npool = npool;
        c->ncell = ncell;
        c->ndofs = node_off[ncell];
        upload(c->blk_off, blk_off, size_t(nt + 1));
        upload(c->blk_cell, blk_cell, size_t(nblocks));
        upload(c->blk_pool, blk_pool, size_t(nblocks));
        upload(c->pool_off, pool_off, size_t(npool + 1));
        if (dev_pool) {
            c->pool_vals.alloc(size_t(nvals));
            if (nvals) VPG_CUDA(cudaMemcpy(c->pool_vals.p, pool_vals, size_t(nvals) * sizeof(double),
                                           cudaMemcpyDeviceToDevice));
        } else {
            upload(c->pool_vals, pool_vals, size_t(nvals));
        }
        upload(c->node_off, node_off, size_t(ncell + 1));
        // lattice groups: 64 consecutive targets with identical block-cell
        // sequences whose rows are base_r + u of contiguous 64 x 64 blocks
        {
            std::map<int64_t, int> mat_of;  // pool_off of the block -> matrix index
            std::vector<int64_t> moff;
            std::vector<int32_t> groups, cells_tmp, other;
            std::vector<std::vector<std::pair<int, int32_t>>> gcells;  // per group: (matrix, cell f offset)
            for (int64_t g = 0; g * 64 < nt; ++g) {
                const int64_t t0 = g * 64;
                bool ok = t0 + 64 <= nt;
                const int m = ok ? blk_off[t0 + 1] - blk_off[t0] : 0;
                std::vector<std::pair<int, int32_t>> mine;
                for (int64_t u = 0; ok && u < 64; ++u) ok = blk_off[t0 + u + 1] - blk_off[t0 + u] == m;
                for (int r = 0; ok && r < m; ++r) {
                    const int64_t k0 = blk_off[t0] + r;
                    const int32_t cell = blk_cell[k0], base = blk_pool[k0];
                    if (base + 63 >= npool) { ok = false; break; }
                    const int64_t p0 = pool_off[base];
                    // the kernel stages M_q with 16-byte loads: an odd p0 would
                    // be a misaligned access -- such groups take the CSR path
                    if (p0 & 1) { ok = false; break; }
                    for (int64_t u = 0; ok && u < 64; ++u) {
                        const int64_t ku = blk_off[t0 + u] + r;
                        ok = blk_cell[ku] == cell && blk_pool[ku] == base + u && pool_off[base + u] == p0 + 64 * u &&
                             pool_off[base + u + 1] == p0 + 64 * (u + 1) && node_off[cell] + 64 <= node_off[ncell];
                    }
                    if (!ok) break;
                    auto it = mat_of.find(p0);
                    int q;
                    if (it == mat_of.end()) {
                        q = int(moff.size());
                        mat_of[p0] = q;
                        moff.push_back(p0);
                    } else {
                        q = it->second;
                    }
                    for (const auto& e : mine) ok = ok && e.first != q;  // one cell per matrix
                    mine.emplace_back(q, node_off[cell]);
                }
                if (ok && m > 0) {
                    groups.push_back(int32_t(t0 / 64));
                    gcells.push_back(std::move(mine));
                } else {
                    for (int64_t u = t0; u < std::min<int64_t>(t0 + 64, nt); ++u) other.push_back(int32_t(u));
                }
            }
            // only blocks shared by many groups (the lattice table) pay off as
            // GEMMs: groups touching a rarely used block go to the CSR kernel
            std::vector<int> uses(moff.size(), 0);
            for (const auto& gc : gcells)
                for (const auto& e : gc) ++uses[size_t(e.first)];
            std::vector<int> remap(moff.size(), -1);
            std::vector<int64_t> shared_off;
            for (size_t q = 0; q < moff.size(); ++q)
                if (uses[q] >= 32 && shared_off.size() < 64) {
                    remap[q] = int(shared_off.size());
                    shared_off.push_back(moff[q]);
                }
            {
                std::vector<int32_t> g2;
                std::vector<std::vector<std::pair<int, int32_t>>> c2;
                for (size_t g = 0; g < groups.size(); ++g) {
                    bool all = true;
                    for (auto& e : gcells[g]) all = all && remap[size_t(e.first)] >= 0;
                    if (all) {
                        for (auto& e : gcells[g]) e.first = remap[size_t(e.first)];
                        g2.push_back(groups[g]);
                        c2.push_back(std::move(gcells[g]));
                    } else {
                        for (int64_t u = int64_t(groups[g]) * 64; u < int64_t(groups[g]) * 64 + 64; ++u)
                            other.push_back(int32_t(u));
                    }
                }
                groups.swap(g2);
                gcells.swap(c2);
                moff.swap(shared_off);
                std::sort(other.begin(), other.end());
            }
            const int nmat = int(moff.size());
            if (groups.size() < 16) {  // not worth it: everything through the CSR kernel
                groups.clear();
                other.resize(size_t(nt));
                for (int64_t u = 0; u < nt; ++u) other[size_t(u)] = int32_t(u);
            }
            std::vector<int32_t> cellof(groups.size() * size_t(std::max(nmat, 1)), -1);
            for (size_t g = 0; g < groups.size(); ++g)
                for (const auto& e : gcells[g]) cellof[g * size_t(nmat) + size_t(e.first)] = e.second;
            c->nlat = int64_t(groups.size());
            c->nmat = groups.empty() ? 0 : nmat;
            c->nother = int64_t(other.size());
            upload(c->lat_group, groups.data(), groups.size());
            upload(c->lat_cell, cellof.data(), groups.empty() ? 0 : cellof.size());
            upload(c->lat_moff, moff.data(), groups.empty() ? 0 : moff.size());
            upload(c->other_t, other.data(), other.size());
            if (c->nlat) {
                smem_optin((const void*)corr_lattice_kernel<64>, int(sizeof(double) * 64 * (68 + 68)));
                smem_optin((const void*)corr_lattice_kernel<16>, int(sizeof(double) * 64 * (68 + 20)));
                smem_optin((const void*)corr_lattice_kernel<8>, int(sizeof(double) * 64 * (68 + 12)));
            }
        }
        *corr = c.release();
    }
}

extern "C" {

int vpg_corr_apply(const vpg_corr* c, const double* f, int64_t nf, double* out,
                   unsigned flags, void* stream) {
    return guarded_c([&] {
        if (!c) throw Error{VPG_ERR_INVALID_ARGUMENT, "corr is NULL"};
        if (nf != c->ndofs)  // potential.cpp:434-438
            throw Error{VPG_ERR_INVALID_ARGUMENT, "apply: expected " + std::to_string(c->ndofs) +
                                                      " samples, got " + std::to_string(nf)};
        VPG_CUDA(cudaSetDevice(c->device));
        OwnStream os(stream);
        const bool dev = flags & VPG_DEVICE_POINTERS;
        double* fd = nullptr;
        double* od = nullptr;
        if (!dev) {
            VPG_CUDA(cudaMallocAsync(&fd, sizeof(double) * size_t(std::max<int64_t>(nf, 1)), os.s));
            VPG_CUDA(cudaMallocAsync(&od, sizeof(double) * size_t(std::max<int64_t>(c->nt, 1)), os.s));
            if (nf) VPG_CUDA(cudaMemcpyAsync(fd, f, sizeof(double) * size_t(nf), cudaMemcpyHostToDevice, os.s));
            if (c->nt)
                VPG_CUDA(cudaMemcpyAsync(od, out, sizeof(double) * size_t(c->nt), cudaMemcpyHostToDevice, os.s));
        }
        if (c->nlat > 0) {
            int sms = 148;
            VPG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
            if (c->nlat >= int64_t(64) * 2 * sms) {
                corr_lattice_kernel<64><<<nblk(c->nlat, 64), 256, sizeof(double) * 64 * (68 + 68), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_moff.p, c->pool_vals.p,
                    dev ? f : fd, dev ? out : od);
            } else if (c->nlat >= int64_t(16) * 2 * sms) {
                corr_lattice_kernel<16><<<nblk(c->nlat, 16), 256, sizeof(double) * 64 * (68 + 20), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_moff.p, c->pool_vals.p,
                    dev ? f : fd, dev ? out : od);
            } else {
                corr_lattice_kernel<8><<<nblk(c->nlat, 8), 256, sizeof(double) * 64 * (68 + 12), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_moff.p, c->pool_vals.p,
                    dev ? f : fd, dev ? out : od);
            }
            VPG_LAUNCH_CHECK();
        }
        if (c->nother) {
            corr_apply_kernel<<<nblk(c->nother, kCorrWarps), kCorrWarps * 32, 0, os.s>>>(
                c->nother, c->other_t.p, c->blk_off.p, c->blk_cell.p, c->blk_pool.p, c->pool_off.p,
                c->pool_vals.p, c->node_off.p, dev ? f : fd, dev ? out : od);
            VPG_LAUNCH_CHECK();
        }
        if (!dev) {
            if (c->nt)
                VPG_CUDA(cudaMemcpyAsync(out, od, sizeof(double) * size_t(c->nt), cudaMemcpyDeviceToHost, os.s));
            VPG_CUDA(cudaFreeAsync(fd, os.s));
            VPG_CUDA(cudaFreeAsync(od, os.s));
        }
        if (!(flags & VPG_NO_SYNC) || os.owned || !dev) VPG_CUDA(cudaStreamSynchronize(os.s));
    });
}

int vpg_corr_destroy(vpg_corr* c) {
    return guarded_c([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        delete c;
    });
}

int vpg_charges_create(int64_t ncell, const int32_t* cell_type, const int32_t* node_off,
                       const int32_t* src_off, const double* over0, int np0, int nq0,
                       const double* over1, int np1, int nq1, const double* src_wj,
                       int device, vpg_charges** ch) {
    return guarded_c([&] {
        if (!ch) throw Error{VPG_ERR_INVALID_ARGUMENT, "charges is NULL"};
        *ch = nullptr;
        if (ncell < 0 || !cell_type || !node_off || !src_off || !src_wj || np0 < 0 || nq0 < 0 ||
            np1 < 0 || nq1 < 0 || (np0 * nq0 && !over0) || (np1 * nq1 && !over1))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad charge-map arrays"};
        for (int64_t c = 0; c < ncell; ++c) {
            const bool t0 = cell_type[c] == 0;
            if (node_off[c + 1] - node_off[c] != (t0 ? np0 : np1) ||
                src_off[c + 1] - src_off[c] != (t0 ? nq0 : nq1))
                throw Error{VPG_ERR_INVALID_ARGUMENT, "cell layout does not match its type"};
        }
        use_device(device);
        auto h = std::make_unique<vpg_charges>();
        h->device = device;
        h->ncell = ncell;
        h->ndofs = node_off[ncell];
        h->nsrc = src_off[ncell];
        h->np[0] = np0;
        h->np[1] = np1;
        h->nq[0] = nq0;
        h->nq[1] = nq1;
        upload(h->cell_type, cell_type, size_t(ncell));
        upload(h->node_off, node_off, size_t(ncell + 1));
        upload(h->src_off, src_off, size_t(ncell + 1));
        upload(h->over0, over0, size_t(np0) * nq0);
        upload(h->over1, over1, size_t(np1) * nq1);
        upload(h->src_wj, src_wj, size_t(h->nsrc));
        *ch = h.release();
    });
}

int vpg_charges_apply(const vpg_charges* h, const double* f, int64_t nf, double* charges,
                      unsigned flags, void* stream) {
    return guarded_c([&] {
        if (!h) throw Error{VPG_ERR_INVALID_ARGUMENT, "charges is NULL"};
        if (nf != h->ndofs)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "apply: expected " + std::to_string(h->ndofs) +
                                                      " samples, got " + std::to_string(nf)};
        VPG_CUDA(cudaSetDevice(h->device));
        OwnStream os(stream);
        const bool dev = flags & VPG_DEVICE_POINTERS;
        double* fd = nullptr;
        double* cd = nullptr;
        if (!dev) {
            VPG_CUDA(cudaMallocAsync(&fd, sizeof(double) * size_t(std::max<int64_t>(nf, 1)), os.s));
            VPG_CUDA(cudaMallocAsync(&cd, sizeof(double) * size_t(std::max<int64_t>(h->nsrc, 1)), os.s));
            if (nf) VPG_CUDA(cudaMemcpyAsync(fd, f, sizeof(double) * size_t(nf), cudaMemcpyHostToDevice, os.s));
        }
        if (h->ncell) {
            const int npmax = std::max(h->np[0], h->np[1]);
            charges_kernel<<<unsigned(h->ncell), 128, sizeof(double) * size_t(std::max(npmax, 1)), os.s>>>(
                h->cell_type.p, h->node_off.p, h->src_off.p, h->over0.p, h->np[0], h->nq[0], h->over1.p,
                h->np[1], h->nq[1], h->src_wj.p, dev ? f : fd, dev ? charges : cd);
            VPG_LAUNCH_CHECK();
        }
        if (!dev) {
            if (h->nsrc)
                VPG_CUDA(cudaMemcpyAsync(charges, cd, sizeof(double) * size_t(h->nsrc),
                                         cudaMemcpyDeviceToHost, os.s));
            VPG_CUDA(cudaFreeAsync(fd, os.s));
            VPG_CUDA(cudaFreeAsync(cd, os.s));
        }
        if (!(flags & VPG_NO_SYNC) || os.owned || !dev) VPG_CUDA(cudaStreamSynchronize(os.s));
    });
}

int vpg_charges_destroy(vpg_charges* h) {
    return guarded_c([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        delete h;
    });
}

}  // extern "C"

extern "C" int vpg_corr_export(const vpg_corr* c, int32_t* blk_off, int32_t* blk_cell, int32_t* blk_pool,
                               int64_t* pool_off, double* pool_vals, int64_t* sizes) {
    return guarded_c([&] {
        if (!c) throw Error{VPG_ERR_INVALID_ARGUMENT, "corr is NULL"};
        VPG_CUDA(cudaSetDevice(c->device));
        if (sizes) {
            sizes[0] = c->nt;
            sizes[1] = c->nblocks;
            sizes[2] = c->npool;
            sizes[3] = int64_t(c->pool_vals.n);
            sizes[4] = c->ndofs;
        }
        auto dl = [](void* h, const void* d, size_t bytes) {
            if (h && bytes) VPG_CUDA(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost));
        };
        dl(blk_off, c->blk_off.p, c->blk_off.bytes());
        dl(blk_cell, c->blk_cell.p, c->blk_cell.bytes());
        dl(blk_pool, c->blk_pool.p, c->blk_pool.bytes());
        dl(pool_off, c->pool_off.p, c->pool_off.bytes());
        dl(pool_vals, c->pool_vals.p, c->pool_vals.bytes());
    });
}
