// p2p.cuh -- the Laplace pair interaction shared by the near-field and
// all-pairs kernels.
//
// One pair costs 11 FP64 instructions: dx, dy, r^2 (2), the table
// reduction, the exponent term, the degree-4 log1p (4 with the addend) and
// the accumulation, plus ~9 integer/LDS/conversion instructions (table
// address, mantissa, exponent).
#pragma once

#include "common.cuh"

namespace vpg {

struct LapAcc {
    double a = 0.0;  // sum q * ln(r2)  (VPG_LOG_FOLD=0: sum q * t)
    double b = 0.0;  // VPG_LOG_FOLD=0 only: sum q * e
    double c = 0.0;  // rare-path sum q * log(r2) for subnormal r2
};

// One pair's contribution to the accumulators (the hot-loop form).
__device__ __forceinline__ void lap_acc(double r2, double q, uint32_t tab_lane, LapAcc& acc) {
#if VPG_LOG_FOLD
    acc.a = fma(q, near_log(r2, tab_lane), acc.a);
#else
    double ed;
    const double t = fast_log_split(r2, tab_lane, ed);
    acc.a = fma(q, t, acc.a);
    acc.b = fma(q, ed, acc.b);
#endif
}

// Hot-loop pair: no zero test at all.  r^2 == 0 yields ln = -1023 ln2 +
// (table entry 0) -- a spurious term that the caller removes in a fix-up
// pass (lap_pair_fixup) over the pairs that can be coincident or subnormal
// (the plan's coincidence list).
__device__ __forceinline__ void lap_pair_fast(double tx, double ty, double sx,
                                              double sy, double q, uint32_t tab_lane,
                                              LapAcc& acc) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    lap_acc(r2, q, tab_lane, acc);
}

#if VPG_LOG_FOLD
// The global-table twin (same bits; fast_log(double, const double2*)).
__device__ __forceinline__ void lap_acc(double r2, double q, const double2* gtab, LapAcc& acc) {
    acc.a = fma(q, near_log(r2, gtab), acc.a);
}
#endif

// Undoes lap_pair_fast for r^2 below the normal range and applies the
// reference semantics instead: skip r^2 == 0 (summation.cpp:340), exact
// log for subnormal r^2.  Tab: the lane's smem table address (uint32_t) or
// the global table (const double2*).
template <class Tab>
__device__ __forceinline__ void lap_pair_fixup(double tx, double ty, double sx,
                                               double sy, double q, Tab tab_lane,
                                               LapAcc& acc) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    if (__double2hiint(r2) >= 0x00100000) return;
    lap_acc(r2, -q, tab_lane, acc);
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
#if VPG_LOG_FOLD
    acc.a = fma(qe, fast_log(r2, tab_lane), acc.a);  // round-to-nearest centres: ln 1 = 0 exactly
#else
    lap_acc(r2, qe, tab_lane, acc);
#endif
}

// sum_j q_j log(r2_j) from the accumulators.
__device__ __forceinline__ double lap_total(const LapAcc& acc) {
#if VPG_LOG_FOLD
    return acc.a + acc.c;
#else
    return fma(acc.b, kLn2Hi, fma(acc.b, kLn2Lo, acc.a)) + acc.c;
#endif
}

// ln(r2) of the symmetric kernel: one double feeding both targets.
__device__ __forceinline__ double lap_log(double r2, uint32_t tab_lane) {
#if VPG_LOG_FOLD
    return near_log(r2, tab_lane);
#else
    double ed;
    const double t = fast_log_split(r2, tab_lane, ed);
    return fma(ed, kLn2Lo, fma(ed, kLn2Hi, t));
#endif
}

}  // namespace vpg
