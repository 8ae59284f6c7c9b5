// p2p.cuh -- the Laplace pair interaction shared by the near-field and
// all-pairs kernels.
//
// One pair costs 14 FP64 instructions: dx, dy, r^2 (2), the exponent
// conversion, the table reduction, the degree-5 log1p, and two
// accumulations (sum q*t and sum q*e, so ln2 is applied once per target).
// The r^2 == 0 skip of the reference (summation.cpp:340, 630) is an integer
// test on the bit pattern: the charge is zeroed, no FP64 compare is spent.
// Subnormal r^2 (distances below 1.5e-154) take a rare exact path.
#pragma once

#include "common.cuh"

namespace vpg {

struct LapAcc {
    double a = 0.0;  // sum q * t
    double b = 0.0;  // sum q * e
    double c = 0.0;  // rare-path sum q * log(r2) for subnormal r2
};

__device__ __forceinline__ void lap_pair(double tx, double ty, double sx,
                                         double sy, double q,
                                         const double2* tab, int lane8,
                                         LapAcc& acc) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    const int hi = __double2hiint(r2);
    double qe = q;
    if (hi < 0x00100000) {  // zero or subnormal: never taken on real meshes
        if ((hi | __double2loint(r2)) != 0) acc.c = fma(q, log(r2), acc.c);
        qe = 0.0;
    }
    double ed;
    const double t = fast_log_split(r2, tab, lane8, ed);
    acc.a = fma(qe, t, acc.a);
    acc.b = fma(qe, ed, acc.b);
}

// sum_j q_j log(r2_j) from the split accumulators.
__device__ __forceinline__ double lap_total(const LapAcc& acc) {
    return fma(acc.b, kLn2Hi, fma(acc.b, kLn2Lo, acc.a)) + acc.c;
}

}  // namespace vpg
