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
};

struct vpg_charges {
    int device = 0;
    int64_t ncell = 0, ndofs = 0, nsrc = 0;
    int np[2] = {0, 0}, nq[2] = {0, 0};
    vpg::DBuf<int32_t> cell_type, node_off, src_off;
    vpg::DBuf<double> over0, over1, src_wj;
};

