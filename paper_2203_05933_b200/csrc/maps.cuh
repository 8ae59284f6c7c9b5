// maps.cuh -- device-resident correction and charge maps (corr.cu), shared
// with the operator-level apply (api.cu).
#pragma once

#include "plan.cuh"

struct BlkDesc {  // a correction block: its pool row, its cell's first sample, the row length
    int64_t row;
    int32_t f;
    int32_t len;
};

struct vpg_corr {
    int device = 0;
    int64_t nt = 0, nblocks = 0, npool = 0, ncell = 0, ndofs = 0;
    vpg::DBuf<int32_t> blk_off, blk_cell, blk_pool, node_off;
    vpg::DBuf<int64_t> pool_off;
    vpg::DBuf<double> pool_vals;
    vpg::DBuf<BlkDesc> blk_desc;    // residual blocks (not on the tensor-core path), CSR res_off
    vpg::DBuf<int32_t> res_off;
    // lattice fast path (corr.cu): 64-target groups whose blocks read shared
    // 64 x 64 row blocks (the box lattice table, potential.cpp:256-267) run
    // as tensor-core GEMMs; every other target through the CSR kernel
    int64_t nlat = 0, nmat = 0, nother = 0;
    vpg::DBuf<int32_t> lat_group;   // group g -> its first target (64 consecutive targets)
    vpg::DBuf<int32_t> lat_cell;    // [group][matrix] -> f offset of the cell (node_off), -1 none
    vpg::DBuf<double> lat_mats;     // [matrix][64][64] dense shared-row matrices
    vpg::DBuf<int32_t> lat_toff, lat_tmats;  // per CTA tile of groups: the matrices it uses (CSR)
    int lat_tile = 64;              // groups per CTA
    vpg::DBuf<int32_t> other_t;     // targets with residual blocks (CSR kernel)
};

namespace vpg {
void corr_create_impl(int64_t nt, const int32_t* blk_off, int64_t nblocks, const int32_t* blk_cell,
                      const int32_t* blk_pool, int64_t npool, const int64_t* pool_off, const double* pool_vals,
                      bool dev_pool, int64_t ncell, const int32_t* node_off, int device, vpg_corr** corr);
}

struct vpg_charges {
    int device = 0;
    int64_t ncell = 0, ndofs = 0, nsrc = 0;
    int np[2] = {0, 0}, nq[2] = {0, 0};
    vpg::DBuf<int32_t> cell_type, node_off, src_off;
    vpg::DBuf<double> over0, over1, src_wj;
    // per-kind cell lists of the tensor-core kernel (corr.cu charges_mma_kernel)
    int64_t ncells_kind[2] = {0, 0};
    vpg::DBuf<int32_t> cells_kind[2];
    int sm_count = 148;
    bool fallback = false;  // O too large for smem: the per-cell kernel
};

