// p2p.cuh -- the Laplace pair interaction shared by the near-field and
// all-pairs kernels.
//
// One pair costs 14 FP64 instructions: dx, dy, r^2 (2), the exponent
// conversion, the table reduction, the degree-5 log1p, and two
// accumulations (sum q*t and sum q*e, so ln2 is applied once per target),
// plus ~7 integer/LDS instructions (table address, mantissa, exponent).
#pragma once

#include "common.cuh"

namespace vpg {

struct LapAcc {
    double a = 0.0;  // sum q * t
    double b = 0.0;  // sum q * e
    double c = 0.0;  // rare-path sum q * log(r2) for subnormal r2
};

// Hot-loop pair: no zero test at all.  r^2 == 0 yields t = 0 and
// e = -1023 (the pattern's exponent field is 0), i.e. a spurious -1023 q ln2
// that the caller removes in a fix-up pass (lap_pair_fixup) over the pairs
// that can be coincident -- for the near field, only sources of the
// target's own leaf (equal coordinates fall in the same leaf).
__device__ __forceinline__ void lap_pair_fast(double tx, double ty, double sx,
                                              double sy, double q, uint32_t tab_lane,
                                              LapAcc& acc) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    double ed;
    const double t = fast_log_split(r2, tab_lane, ed);
    acc.a = fma(q, t, acc.a);
    acc.b = fma(q, ed, acc.b);
}

// Undoes lap_pair_fast for r^2 below the normal range and applies the
// reference semantics instead: skip r^2 == 0 (summation.cpp:340), exact
// log for subnormal r^2.
__device__ __forceinline__ void lap_pair_fixup(double tx, double ty, double sx,
                                               double sy, double q, uint32_t tab_lane,
                                               LapAcc& acc) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    if (__double2hiint(r2) >= 0x00100000) return;
    double ed;
    const double t = fast_log_split(r2, tab_lane, ed);
    acc.a = fma(-q, t, acc.a);
    acc.b = fma(-q, ed, acc.b);
    if (r2 != 0.0) acc.c = fma(q, log(r2), acc.c);
}

// Self-contained pair for the all-pairs kernels (coincidences anywhere):
// the charge of an r^2 == 0 pair is zeroed by an integer test.
__device__ __forceinline__ void lap_pair(double tx, double ty, double sx,
                                         double sy, double q, uint32_t tab_lane,
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
    const double t = fast_log_split(r2, tab_lane, ed);
    acc.a = fma(qe, t, acc.a);
    acc.b = fma(qe, ed, acc.b);
}

// sum_j q_j log(r2_j) from the split accumulators.
__device__ __forceinline__ double lap_total(const LapAcc& acc) {
    return fma(acc.b, kLn2Hi, fma(acc.b, kLn2Lo, acc.a)) + acc.c;
}

}  // namespace vpg
