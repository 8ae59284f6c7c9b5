// maps.cuh -- device-resident correction and charge maps (corr.cu), shared
// with the operator-level apply (api.cu).
#pragma once

#include "plan.cuh"

struct vpg_corr {
    int device = 0;
    int64_t nt = 0, nblocks = 0, npool = 0, ncell = 0, ndofs = 0;
    vpg::DBuf<int32_t> blk_off, blk_cell, blk_pool, node_off;
    vpg::DBuf<int64_t> pool_off;
    vpg::DBuf<double> pool_vals;
    // lattice fast path (corr.cu): 64-target groups whose blocks read shared
    // 64 x 64 row blocks (the box lattice table, potential.cpp:256-267) run
    // as tensor-core GEMMs; every other target through the CSR kernel
    int64_t nlat = 0, nmat = 0, nother = 0;
    vpg::DBuf<int32_t> lat_group;   // group g -> first target 64 g
    vpg::DBuf<int32_t> lat_cell;    // [group][matrix] -> f offset of the cell (node_off), -1 none
    vpg::DBuf<int64_t> lat_moff;    // [matrix] -> offset of its 64 x 64 block in pool_vals
    vpg::DBuf<int32_t> other_t;     // targets of the CSR kernel
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
};

