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
#include <set>
#include <unordered_map>
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

// CSR apply over per-block descriptors (row offset, f offset, length built
// at map creation): lane j of a target's warp loads block j's descriptor, so
// the three dependent index loads of a block (blk_pool -> pool_off, blk_cell
// -> node_off) are gone and the data loads of successive blocks are
// independent (the loop is unrolled); one butterfly per target.
__global__ void __launch_bounds__(kCorrWarps * 32)
corr_desc_kernel(int64_t nt, const int32_t* tlist, const int32_t* blk_off, const BlkDesc* desc,
                 const double* pool_vals, const double* f, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t ti = int64_t(blockIdx.x) * kCorrWarps + (threadIdx.x >> 5);
    if (ti >= nt) return;
    const int64_t t = tlist ? tlist[ti] : ti;
    const int k0 = blk_off[t], n = blk_off[t + 1] - k0;
    double acc = 0.0;
    for (int b0 = 0; b0 < n; b0 += 32) {
        BlkDesc d{0, 0, 0};
        if (b0 + lane < n) d = desc[k0 + b0 + lane];
        const int m = min(32, n - b0);
        // four blocks at a time: all their loads are issued before the FMAs
        for (int j = 0; j < m; j += 4) {
            double rv[8], fv[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int jj = min(j + u, 31);
                const int64_t row = __shfl_sync(0xffffffffu, d.row, jj);
                const int fo = __shfl_sync(0xffffffffu, d.f, jj);
                const int len = j + u < m ? __shfl_sync(0xffffffffu, d.len, jj) : 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int e = lane + 32 * h;
                    const bool ok = e < len;
                    rv[2 * u + h] = ok ? __ldg(pool_vals + row + e) : 0.0;
                    fv[2 * u + h] = ok ? __ldg(f + fo + e) : 0.0;
                }
                // rows longer than 64 (p > 8 boxes): the rest, in order
                for (int e = lane + 64; e < len; e += 32) acc = fma(__ldg(pool_vals + row + e), __ldg(f + fo + e), acc);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = fma(rv[k], fv[k], acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[t] += acc;
}

// The residual blocks with half a warp per target (two targets per warp):
// a lane covers entries l, l + 16, l + 32, l + 48 of each row (rows <= 64;
// longer rows finish in order), four blocks' loads issued before their FMAs.
__global__ void __launch_bounds__(kCorrWarps * 32)
corr_desc16_kernel(int64_t nt, const int32_t* tlist, const int32_t* blk_off, const BlkDesc* desc,
                   const double* pool_vals, const double* f, double* out) {
    const int lane = threadIdx.x & 31, half = lane >> 4, l = lane & 15;
    const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
    const int64_t ti = (int64_t(blockIdx.x) * kCorrWarps + (threadIdx.x >> 5)) * 2 + half;
    const bool live = ti < nt;
    const int64_t t = live ? (tlist ? tlist[ti] : ti) : 0;
    const int k0 = live ? blk_off[t] : 0, n = live ? blk_off[t + 1] - k0 : 0;
    double acc = 0.0;
    for (int b0 = 0; b0 < n; b0 += 16) {
        BlkDesc d{0, 0, 0};
        if (b0 + l < n) d = desc[k0 + b0 + l];
        const int m = min(16, n - b0);
        for (int j = 0; j < m; j += 4) {
            double rv[16], fv[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int src = (half << 4) + min(j + u, 15);
                const int64_t row = __shfl_sync(hmask, d.row, src);
                const int fo = __shfl_sync(hmask, d.f, src);
                const int len = j + u < m ? __shfl_sync(hmask, d.len, src) : 0;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int e = l + 16 * h;
                    const bool ok = e < len;
                    rv[4 * u + h] = ok ? __ldg(pool_vals + row + e) : 0.0;
                    fv[4 * u + h] = ok ? __ldg(f + fo + e) : 0.0;
                }
                for (int e = l + 64; e < len; e += 16) acc = fma(__ldg(pool_vals + row + e), __ldg(f + fo + e), acc);
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = fma(rv[k], fv[k], acc);
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (live && l == 0) out[t] += acc;
}

__global__ void gather_rows_kernel(const int64_t* rowsrc, const double* pool_vals, double* mats) {
    const int64_t r = blockIdx.x;
    const int64_t src = rowsrc[r];
    mats[r * 64 + threadIdx.x] = src >= 0 ? pool_vals[src + threadIdx.x] : 0.0;
}

// Lattice groups on the FP64 tensor cores: a CTA takes 64 groups (64
// targets each) and walks the shared 64 x 64 row blocks M_q: out[64g + u] +=
// sum_q sum_i M_q[u][i] f[cell(g, q) + i] as Y = M_q F_q (mma.sync m8n8k4),
// M_q and the tile's f segments staged in smem (strides == 4 mod 16).
template <int kLatTile>  // groups per CTA (64; 16 or 8 for small maps: more CTAs)
__global__ void __launch_bounds__(256)
corr_lattice_kernel(int64_t ngroups, int nmat, const int32_t* group, const int32_t* cellof,
                    const int32_t* tile_off, const int32_t* tile_mats, const double* mats, const double* f,
                    double* out) {
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
    const int q0 = tile_off[blockIdx.x], q1 = tile_off[blockIdx.x + 1];  // this tile's matrices
    auto fetch = [&](int q) {
        const double2* mg = reinterpret_cast<const double2*>(mats + int64_t(q) * K * K);
#pragma unroll
        for (int r = 0; r < kMR; ++r) mreg[r] = mg[threadIdx.x + 256 * r];
#pragma unroll
        for (int r = 0; r < kFR; ++r) {
            const int e = threadIdx.x + 256 * r, g = e / K, i = e % K;
            const int c = g < ng ? cellof[(g0 + g) * nmat + q] : -1;
            freg[r] = c >= 0 ? f[int64_t(c) + i] : 0.0;
        }
    };
    if (q1 > q0) fetch(tile_mats[q0]);
    for (int qi = q0; qi < q1; ++qi) {
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
        if (qi + 1 < q1) fetch(tile_mats[qi + 1]);
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
            if (g < ng) out[int64_t(group[g0 + g]) + u] += acc[n8][h];
        }
}

// build_charges on the FP64 tensor cores: per cell kind, Q = O F with O the
// kind's oversampling matrix (nq x np, staged once per CTA in smem as A
// fragments, row stride == 4 mod 16 doubles) and F the f segments of a tile
// of 32 cells (np x 32, B fragments); mma.sync m8n8k4 (DMMA), each warp owns
// every 8th 8-row tile of O for the 4 column tiles; results go straight from
// the accumulators to charges[src_off[c] + s] * src_wj (a lane's 8 rows of
// one cell are 64 contiguous bytes).  Persistent CTAs walk the cell tiles.
constexpr int kChTile = 32;  // largest cell tile (4 column tiles of 8 cells)
struct ChKind {
    int64_t ncell;
    const int32_t* cells;
    const double* O;
    int np, nq;
    int ntl;    // 8-cell column tiles per CTA tile (1, 2 or 4)
    int grid;   // CTAs of this kind
};
// Both cell kinds in one launch: CTAs [0, k0.grid) take the box tiles, the
// rest the triangle tiles (split by flops), tiles of 8 ntl cells so that
// small maps still spread over every SM.
template <int kMT>  // 8-row tiles per warp: ceil(ceil(nq / 8) / 8), max over the kinds
__global__ void __launch_bounds__(256)
charges_mma_kernel(ChKind k0, ChKind k1, const int32_t* node_off, const int32_t* src_off, const double* src_wj,
                   const double* f, double* charges) {
    extern __shared__ __align__(16) double csm[];
    const bool second = int(blockIdx.x) >= k0.grid;
    const ChKind K = second ? k1 : k0;
    const int bid = second ? int(blockIdx.x) - k0.grid : int(blockIdx.x);
    const int np = K.np, nq = K.nq, ntl = K.ntl, tile = 8 * ntl;
    const int Kp = (np + 3) & ~3, Mp = (nq + 7) & ~7;
    const int As = Kp + ((4 - Kp % 16) + 16) % 16;  // row stride == 4 mod 16
    constexpr int Bs = kChTile + 4;                  // == 4 mod 16
    double* A = csm;              // [Mp][As]
    double* B = csm + Mp * As;    // [Kp][Bs]
    for (int e = threadIdx.x; e < Mp * Kp; e += blockDim.x) {
        const int r = e / Kp, k = e % Kp;
        A[r * As + k] = (r < nq && k < np) ? K.O[int64_t(r) * np + k] : 0.0;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, rq = lane >> 2;
    const int mtiles = Mp / 8;
    for (int64_t t0 = int64_t(bid) * tile; t0 < K.ncell; t0 += int64_t(K.grid) * tile) {
        const int nc = int(min(int64_t(tile), K.ncell - t0));
        __syncthreads();  // A staged / the previous tile's B reads are done
        for (int e = threadIdx.x; e < tile * Kp; e += blockDim.x) {
            const int j = e / Kp, i = e % Kp;
            double v = 0.0;
            if (j < nc && i < np) v = f[int64_t(node_off[K.cells[t0 + j]]) + i];
            B[i * Bs + j] = v;
        }
        __syncthreads();
        double acc[kMT][4][2];
#pragma unroll
        for (int m = 0; m < kMT; ++m)
#pragma unroll
            for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
        for (int k4 = 0; k4 < Kp; k4 += 4) {
            double b[4];
#pragma unroll
            for (int n = 0; n < 4; ++n) b[n] = n < ntl ? B[(k4 + kq) * Bs + 8 * n + rq] : 0.0;
#pragma unroll
            for (int m = 0; m < kMT; ++m) {
                const int mt = warp + 8 * m;
                if (mt < mtiles) {
                    const double a = A[(8 * mt + rq) * As + k4 + kq];
#pragma unroll
                    for (int n = 0; n < 4; ++n)
                        if (n < ntl)
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                         : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                                         : "d"(a), "d"(b[n]));
                }
            }
        }
        // lane: row 8 mt + rq, cells 8 n + 2 kq + {0, 1}
#pragma unroll
        for (int m = 0; m < kMT; ++m) {
            const int s = 8 * (warp + 8 * m) + rq;
            if (warp + 8 * m >= mtiles || s >= nq) continue;
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 8 * n + 2 * kq + h;
                    if (n < ntl && j < nc) {
                        const int64_t o = int64_t(src_off[K.cells[t0 + j]]) + s;
                        charges[o] = src_wj[o] * acc[m][n][h];
                    }
                }
        }
    }
}

size_t charges_mma_smem(int np, int nq) {
    const int Kp = (np + 3) & ~3, Mp = (nq + 7) & ~7;
    const int As = Kp + ((4 - Kp % 16) + 16) % 16;
    return sizeof(double) * (size_t(Mp) * As + size_t(Kp) * (kChTile + 4));
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

        // Shared-row groups on the tensor cores.  A group is a run of 64
        // consecutive targets whose first (self) blocks share one cell -- the
        // nodes of one box when targets are nodes.  Per group and cell, the
        // blocks whose pool row is shared (length 64, used by >= 8 blocks: the
        // box lattice rows, potential.cpp:256-267) form a 64 x 64 matrix, row u
        // = target u's row for that cell (zero if it has none); groups with the
        // same row pattern share one dense matrix M_q (materialised once), so
        // out[group + u] += sum_q M_q[u] . f[cell(g, q)] runs as DMMA GEMMs
        // (corr_lattice_kernel).  Every other block -- private triangle rows,
        // blocks of targets outside a group -- goes through the CSR kernel.
        {
            std::vector<int32_t> uses(size_t(npool), 0);
            for (int64_t k = 0; k < nblocks; ++k) ++uses[size_t(blk_pool[k])];
            auto shared = [&](int32_t r) { return pool_off[r + 1] - pool_off[r] == 64 && uses[size_t(r)] >= 8; };
            std::vector<char> covered(size_t(nblocks), 0);
            struct VecHash {
                size_t operator()(const std::vector<int32_t>& v) const {
                    uint64_t h = 1469598103934665603ull;
                    for (int32_t x : v) h = (h ^ uint64_t(uint32_t(x))) * 1099511628211ull;
                    return size_t(h);
                }
            };
            std::unordered_map<std::vector<int32_t>, int, VecHash> mat_of;
            std::vector<std::vector<int32_t>> mats;   // per matrix: the 64 pool rows (-1 = zero)
            std::vector<int32_t> uses_q;
            std::vector<int32_t> gstart;                               // first target of each group
            std::vector<std::vector<std::pair<int, int32_t>>> gcells;  // per group: (matrix, f offset)
            std::vector<std::vector<std::vector<int64_t>>> gblocks;    // per group and entry: its blocks
            int64_t t = 0;
            while (t + 64 <= nt) {
                const int64_t k0 = blk_off[t];
                if (blk_off[t + 1] == k0) { ++t; continue; }
                const int32_t self_cell = blk_cell[k0];
                int64_t run = 1;
                while (t + run < nt && blk_off[t + run + 1] > blk_off[t + run] && blk_cell[blk_off[t + run]] == self_cell)
                    ++run;
                for (int64_t g0 = t; g0 + 64 <= t + run; g0 += 64) {
                    std::map<int32_t, std::vector<int32_t>> rows_of;  // cell -> 64 rows
                    std::map<int32_t, std::vector<int64_t>> blks_of;
                    std::set<int32_t> clash;
                    for (int u = 0; u < 64; ++u)
                        for (int64_t k = blk_off[g0 + u]; k < blk_off[g0 + u + 1]; ++k) {
                            const int32_t r = blk_pool[k], cl = blk_cell[k];
                            if (!shared(r)) continue;
                            auto& v = rows_of[cl];
                            if (v.empty()) v.assign(64, -1);
                            if (v[size_t(u)] >= 0) clash.insert(cl);
                            v[size_t(u)] = r;
                            blks_of[cl].push_back(k);
                        }
                    std::vector<std::pair<int, int32_t>> mine;
                    std::vector<std::vector<int64_t>> cov;
                    std::set<int> used_q;
                    for (auto& e : rows_of) {
                        if (clash.count(e.first) || node_off[e.first] + 64 > node_off[ncell]) continue;
                        auto it = mat_of.find(e.second);
                        int q;
                        if (it == mat_of.end()) {
                            q = int(mats.size());
                            mat_of.emplace(e.second, q);
                            mats.push_back(e.second);
                            uses_q.push_back(0);
                        } else {
                            q = it->second;
                        }
                        if (used_q.count(q)) continue;  // one cell per matrix and group
                        used_q.insert(q);
                        ++uses_q[size_t(q)];
                        mine.emplace_back(q, node_off[e.first]);
                        cov.push_back(blks_of[e.first]);
                    }
                    if (!mine.empty()) {
                        gstart.push_back(int32_t(g0));
                        gcells.push_back(std::move(mine));
                        gblocks.push_back(std::move(cov));
                    }
                }
                t += run;
            }
            // keep the matrices shared by enough groups (at most 128); groups keep
            // only those, their other blocks fall back to the CSR kernel
            std::vector<int> order(mats.size());
            for (size_t q = 0; q < mats.size(); ++q) order[q] = int(q);
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return uses_q[size_t(a)] > uses_q[size_t(b)]; });
            std::vector<int> remap(mats.size(), -1);
            std::vector<std::vector<int32_t>> kept;
            for (int q : order)
                if (uses_q[size_t(q)] >= 4 && kept.size() < 128) {
                    remap[size_t(q)] = int(kept.size());
                    kept.push_back(mats[size_t(q)]);
                }
            const int nmat = int(kept.size());
            std::vector<int32_t> groups, cellof;
            for (size_t g = 0; g < gstart.size(); ++g) {
                std::vector<std::pair<int, int32_t>> mine;
                for (auto& e : gcells[g])
                    if (remap[size_t(e.first)] >= 0) mine.emplace_back(remap[size_t(e.first)], e.second);
                if (mine.empty()) continue;
                groups.push_back(gstart[g]);
                const size_t base = cellof.size();
                cellof.resize(base + size_t(nmat), -1);
                for (auto& e : mine) cellof[base + size_t(e.first)] = e.second;
            }
            // covered blocks: those of the kept (group, matrix) entries (each
            // matrix is exactly the rows of its entry's blocks)
            for (size_t g = 0; g < gstart.size(); ++g)
                for (size_t e = 0; e < gcells[g].size(); ++e)
                    if (remap[size_t(gcells[g][e].first)] >= 0)
                        for (int64_t k : gblocks[g][e]) covered[size_t(k)] = 1;
            if (groups.size() < 4) {  // not worth it
                groups.clear();
                cellof.clear();
                std::fill(covered.begin(), covered.end(), 0);
            }
            // residual CSR: the targets' uncovered blocks
            std::vector<int32_t> res_off(size_t(nt) + 1, 0), other;
            std::vector<BlkDesc> rdesc;
            for (int64_t tt = 0; tt < nt; ++tt) {
                for (int64_t k = blk_off[tt]; k < blk_off[tt + 1]; ++k)
                    if (!covered[size_t(k)]) {
                        const int32_t pr = blk_pool[k];
                        rdesc.push_back(BlkDesc{pool_off[pr], node_off[blk_cell[k]], int32_t(pool_off[pr + 1] - pool_off[pr])});
                    }
                res_off[size_t(tt) + 1] = int32_t(rdesc.size());
                if (res_off[size_t(tt) + 1] > res_off[size_t(tt)]) other.push_back(int32_t(tt));
            }
            upload(c->res_off, res_off.data(), res_off.size());
            upload(c->blk_desc, rdesc.data(), rdesc.size());
            c->nlat = int64_t(groups.size());
            c->nmat = groups.empty() ? 0 : nmat;
            c->nother = int64_t(other.size());
            int sms = 148;
            VPG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
            c->lat_tile = c->nlat >= int64_t(64) * 2 * sms ? 64 : c->nlat >= int64_t(16) * 2 * sms ? 16 : 8;
            // per CTA tile: the matrices any of its groups uses
            std::vector<int32_t> toff(1, 0), tmats;
            for (int64_t g0 = 0; g0 < c->nlat; g0 += c->lat_tile) {
                for (int q = 0; q < c->nmat; ++q) {
                    bool any = false;
                    for (int64_t g = g0; g < std::min<int64_t>(g0 + c->lat_tile, c->nlat) && !any; ++g)
                        any = cellof[size_t(g) * size_t(nmat) + size_t(q)] >= 0;
                    if (any) tmats.push_back(q);
                }
                toff.push_back(int32_t(tmats.size()));
            }
            upload(c->lat_group, groups.data(), groups.size());
            upload(c->lat_cell, cellof.data(), cellof.size());
            upload(c->lat_toff, toff.data(), toff.size());
            upload(c->lat_tmats, tmats.data(), tmats.size());
            upload(c->other_t, other.data(), other.size());
            // the dense matrices, gathered from the pool on the device
            if (c->nlat) {
                std::vector<int64_t> rowsrc(size_t(nmat) * 64);
                for (int q = 0; q < nmat; ++q)
                    for (int u = 0; u < 64; ++u) {
                        const int32_t r = kept[size_t(q)][size_t(u)];
                        rowsrc[size_t(q) * 64 + size_t(u)] = r >= 0 ? pool_off[r] : -1;
                    }
                DBuf<int64_t> rs;
                upload(rs, rowsrc.data(), rowsrc.size());
                c->lat_mats.alloc(size_t(nmat) * 4096);
                gather_rows_kernel<<<unsigned(nmat * 64), 64>>>(rs.p, c->pool_vals.p, c->lat_mats.p);
                VPG_LAUNCH_CHECK();
                VPG_CUDA(cudaDeviceSynchronize());
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
            const double* fin = dev ? f : fd;
            double* o = dev ? out : od;
            if (c->lat_tile == 64)
                corr_lattice_kernel<64><<<nblk(c->nlat, 64), 256, sizeof(double) * 64 * (68 + 68), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_toff.p, c->lat_tmats.p,
                    c->lat_mats.p, fin, o);
            else if (c->lat_tile == 16)
                corr_lattice_kernel<16><<<nblk(c->nlat, 16), 256, sizeof(double) * 64 * (68 + 20), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_toff.p, c->lat_tmats.p,
                    c->lat_mats.p, fin, o);
            else
                corr_lattice_kernel<8><<<nblk(c->nlat, 8), 256, sizeof(double) * 64 * (68 + 12), os.s>>>(
                    c->nlat, int(c->nmat), c->lat_group.p, c->lat_cell.p, c->lat_toff.p, c->lat_tmats.p,
                    c->lat_mats.p, fin, o);
            VPG_LAUNCH_CHECK();
        }
        if (c->nother) {
            corr_desc16_kernel<<<nblk(c->nother, 2 * kCorrWarps), kCorrWarps * 32, 0, os.s>>>(
                c->nother, c->other_t.p, c->res_off.p, c->blk_desc.p, c->pool_vals.p, dev ? f : fd,
                dev ? out : od);
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
        for (int kind = 0; kind < 2; ++kind) {
            std::vector<int32_t> cl;
            for (int64_t c = 0; c < ncell; ++c)
                if ((cell_type[c] == 0) == (kind == 0)) cl.push_back(int32_t(c));
            h->ncells_kind[kind] = int64_t(cl.size());
            upload(h->cells_kind[kind], cl.data(), cl.size());
        }
        if (charges_mma_smem(np0, nq0) > 227 * 1024 || charges_mma_smem(np1, nq1) > 227 * 1024 || nq0 > 256 ||
            nq1 > 256)
            h->ncells_kind[0] = h->ncells_kind[1] = 0, h->fallback = true;
        VPG_CUDA(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device));
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
        if (h->fallback && h->ncell) {
            const int npmax = std::max(h->np[0], h->np[1]);
            charges_kernel<<<unsigned(h->ncell), 128, sizeof(double) * size_t(std::max(npmax, 1)), os.s>>>(
                h->cell_type.p, h->node_off.p, h->src_off.p, h->over0.p, h->np[0], h->nq[0], h->over1.p,
                h->np[1], h->nq[1], h->src_wj.p, dev ? f : fd, dev ? charges : cd);
            VPG_LAUNCH_CHECK();
        }
        if (h->ncells_kind[0] + h->ncells_kind[1] > 0) {
            ChKind kk[2];
            double w[2];
            int mtmax = 1;
            for (int kind = 0; kind < 2; ++kind) {
                kk[kind] = ChKind{h->ncells_kind[kind], h->cells_kind[kind].p, kind ? h->over1.p : h->over0.p,
                                  h->np[kind], h->nq[kind], 4, 0};
                w[kind] = double(h->ncells_kind[kind]) * h->np[kind] * h->nq[kind];
                mtmax = std::max(mtmax, ((h->nq[kind] + 7) / 8 + 7) / 8);
            }
            // CTAs split by tile count (a tile's cost is dominated by staging and
            // the k-loop length, not by its exact flops)
            const int sms = h->sm_count;
            for (int kind = 0; kind < 2; ++kind) w[kind] = double((h->ncells_kind[kind] + kChTile - 1) / kChTile);
            int g0 = w[0] > 0 ? std::max(1, int(std::lround(sms * w[0] / (w[0] + w[1])))) : 0;
            if (w[1] > 0) g0 = std::min(g0, sms - 1);
            const int gr[2] = {g0, w[1] > 0 ? sms - g0 : 0};
            for (int kind = 0; kind < 2; ++kind) {
                int ntl = 4;
                while (ntl > 1 && (kk[kind].ncell + 8 * ntl - 1) / (8 * ntl) < gr[kind]) ntl /= 2;
                kk[kind].ntl = ntl;
                kk[kind].grid = int(std::min<int64_t>(gr[kind], (kk[kind].ncell + 8 * ntl - 1) / (8 * ntl)));
            }
            const size_t smem = std::max(kk[0].ncell ? charges_mma_smem(kk[0].np, kk[0].nq) : 0,
                                         kk[1].ncell ? charges_mma_smem(kk[1].np, kk[1].nq) : 0);
            const unsigned grid = unsigned(kk[0].grid + kk[1].grid);
            const double* fin = dev ? f : fd;
            double* cout = dev ? charges : cd;
            if (mtmax <= 2) {
                smem_optin((const void*)charges_mma_kernel<2>, int(smem));
                charges_mma_kernel<2><<<grid, 256, smem, os.s>>>(kk[0], kk[1], h->node_off.p, h->src_off.p,
                                                               h->src_wj.p, fin, cout);
            } else {
                smem_optin((const void*)charges_mma_kernel<4>, int(smem));
                charges_mma_kernel<4><<<grid, 256, smem, os.s>>>(kk[0], kk[1], h->node_off.p, h->src_off.p,
                                                               h->src_wj.p, fin, cout);
            }
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
