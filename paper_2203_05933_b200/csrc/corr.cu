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
#include <vector>

#include "plan.cuh"

#include "maps.cuh"

namespace vpg {
namespace {

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

constexpr int kCorrWarps = 8;

__global__ void __launch_bounds__(kCorrWarps * 32)
corr_apply_kernel(int64_t nt, const int32_t* blk_off, const int32_t* blk_cell,
                  const int32_t* blk_pool, const int64_t* pool_off,
                  const double* pool_vals, const int32_t* node_off,
                  const double* f, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t t = int64_t(blockIdx.x) * kCorrWarps + (threadIdx.x >> 5);
    if (t >= nt) return;
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
            VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
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
        upload(c->pool_vals, pool_vals, size_t(nvals));
        upload(c->node_off, node_off, size_t(ncell + 1));
        *corr = c.release();
    });
}

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
        if (c->nt) {
            corr_apply_kernel<<<nblk(c->nt, kCorrWarps), kCorrWarps * 32, 0, os.s>>>(
                c->nt, c->blk_off.p, c->blk_cell.p, c->blk_pool.p, c->pool_off.p, c->pool_vals.p,
                c->node_off.p, dev ? f : fd, dev ? out : od);
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
