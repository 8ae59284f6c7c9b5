// k0.cuh -- modified Bessel K0 on the device, for the modified-Helmholtz
// kernel G = (1/2pi) K0(lambda r) (kernel.cpp:181-186).
//
// Same split as the reference bessel_k0 (kernel.cpp:167-172):
//   x <= 2: K0 = -(ln(x/2) + gamma) I0(x) + sum_k q^k H_k / (k!)^2,
//           q = x^2/4 (kernel.cpp:17-31).  Here both series are evaluated
//           as fixed degree-16 polynomials in q by Horner (the reference
//           loop stops once a term drops below 1e-19 I0; the omitted tail is
//           below 1e-26 for q <= 1), which keeps the warp converged.
//   x > 2:  K0 = g(x) e^-x / sqrt(x) with g a 25-coefficient Chebyshev fit of
//           K0(x) e^x sqrt(x) on the dyadic intervals [2,4], ..., [512,1024]
//           (kernel.cpp:93-163).  The fit is computed on the host in long
//           double (k0_fit.cu) and lives in global memory.
//   exp(-x) underflow (x > ~745) returns 0 like kernel.cpp:158-161.
#pragma once

#include <cmath>

#include "common.cuh"

namespace vpg {

constexpr int kK0Intervals = 9;
constexpr int kK0Coeffs = 25;

// 1/(k!)^2 and H_k/(k!)^2, k = 0..16, in constant memory: the Horner
// steps take them as c[bank][offset] operands instead of materialising 34
// double immediates per call site.
static __constant__ double c_k0_i0[17] = {
    1.0, 1.0, 0.25, 0.027777777777777776, 0.001736111111111111,
    6.944444444444444e-05, 1.9290123456790124e-06, 3.936759889140842e-08,
    6.151187326782565e-10, 7.594058428126624e-12, 7.594058428126623e-14,
    6.276081345559193e-16, 4.358389823304995e-18, 2.5789288895295828e-20,
    1.3157800456783586e-22, 5.8479113141260385e-25, 2.2843403570804838e-27};
static __constant__ double c_k0_h[17] = {
    0.0, 1.0, 0.375, 0.05092592592592592, 0.003616898148148148,
    0.0001585648148148148, 4.72608024691358e-06, 1.0207455998272325e-07,
    1.6718048413148328e-09, 2.1483350211950277e-11, 2.224275605476294e-13,
    1.895299587006153e-15, 1.3525001839484812e-17, 8.201338813682637e-20,
    4.278340826570208e-22, 1.9404708872364884e-24, 7.722735675585063e-27};

__device__ __forceinline__ double k0_small(double x) {
    const double* c = c_k0_i0;
    const double* d = c_k0_h;
    const double q = 0.25 * x * x;
    double i0 = c[16], s = d[16];
#pragma unroll
    for (int k = 15; k >= 0; --k) {
        i0 = fma(i0, q, c[k]);
        s = fma(s, q, d[k]);
    }
    constexpr double kGamma = 0.57721566490153286061;
    return -(log(0.5 * x) + kGamma) * i0 + s;
}

// The x <= 2 branch from q = x^2 / 4 directly (no square root):
// ln(x/2) = ln(q) / 2.
__device__ __forceinline__ double k0_small_q(double q) {
    const double* c = c_k0_i0;
    const double* d = c_k0_h;
    double i0 = c[16], s = d[16];
#pragma unroll
    for (int k = 15; k >= 0; --k) {
        i0 = fma(i0, q, c[k]);
        s = fma(s, q, d[k]);
    }
    constexpr double kGamma = 0.57721566490153286061;
    return -(0.5 * log(q) + kGamma) * i0 + s;
}

// Degree-D truncations of the two series; D = 9 for q <= 1/4 (the dropped
// tail is below q^10 / (10!)^2 ~ 7e-20 relative), lower when the plan bounds
// q further (k0_series_degree).
template <int D>
__device__ __forceinline__ double k0_i0_d(double q) {
    double v = c_k0_i0[D];
#pragma unroll
    for (int k = D - 1; k >= 0; --k) v = fma(v, q, c_k0_i0[k]);
    return v;
}
template <int D>
__device__ __forceinline__ double k0_h_d(double q) {
    double v = c_k0_h[D];
#pragma unroll
    for (int k = D - 1; k >= 0; --k) v = fma(v, q, c_k0_h[k]);
    return v;
}
__device__ __forceinline__ double k0_i0_9(double q) { return k0_i0_d<9>(q); }
__device__ __forceinline__ double k0_h_9(double q) { return k0_h_d<9>(q); }

// Smallest degree D in [5, 9] whose dropped tail at q <= qmax stays below
// 1e-17 of K0 there (K0 >= K0(1) = 0.42 for q <= 1/4; |ln(x/2) + gamma| <= 2).
inline int k0_series_degree(double qmax) {
    static const double i0[11] = {1.0, 1.0, 0.25, 0.027777777777777776, 0.001736111111111111,
                                  6.944444444444444e-05, 1.9290123456790124e-06, 3.936759889140842e-08,
                                  6.151187326782565e-10, 7.594058428126624e-12, 7.594058428126623e-14};
    static const double h[11] = {0.0, 1.0, 0.375, 0.05092592592592592, 0.003616898148148148,
                                 0.0001585648148148148, 4.72608024691358e-06, 1.0207455998272325e-07,
                                 1.6718048413148328e-09, 2.1483350211950277e-11, 2.224275605476294e-13};
    for (int d = 5; d < 9; ++d)
        if (std::pow(qmax, d + 1) * (2.0 * i0[d + 1] + h[d + 1]) <= 4e-18) return d;
    return 9;
}

__device__ __forceinline__ double k0_large(double x, const double* tab) {
    const double ex = exp(-x);
    if (ex == 0.0) return 0.0;
    // Interval iv covers (2^(iv+1), 2^(iv+2)] like the reference search
    // (kernel.cpp:139-146); x beyond 1024 extrapolates on the last one.
    const int e = ilogb(x);
    int iv = (x == ldexp(1.0, e)) ? e - 2 : e - 1;
    iv = max(0, min(iv, kK0Intervals - 1));
    // u = (2x - (lo+hi)) / (hi-lo) with lo = 2^(iv+1): exact power-of-two
    // scaling, one rounding, same value as the reference expression.
    const double u = fma(x, ldexp(1.0, -iv), -3.0);
    const double* c = tab + iv * kK0Coeffs;
    const double u2 = 2.0 * u;
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int k = kK0Coeffs - 1; k >= 1; --k) {
        const double b0 = fma(u2, b1, c[k] - b2);
        b2 = b1;
        b1 = b0;
    }
    const double g = fma(u, b1, 0.5 * c[0] - b2);
    return g * ex * rsqrt(x);
}

__device__ __forceinline__ double k0_dev(double x, const double* tab) {
    return x <= 2.0 ? k0_small(x) : k0_large(x, tab);
}

// q * K0(lambda r) for one pair, r^2 == 0 skipped (summation.cpp:486, 630).
__device__ __forceinline__ double k0_pair(double tx, double ty, double sx,
                                          double sy, double q, double lambda,
                                          const double* tab) {
    const double dx = tx - sx, dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    if (r2 == 0.0) return 0.0;
    return q * k0_dev(lambda * sqrt(r2), tab);
}

// Host: builds the Chebyshev table (kK0Intervals x kK0Coeffs doubles).
void k0_fit_host(double* out);
void k1_fit_host(double* out);  // the K1 table, same layout

// ---- K1 (kernel.cpp:33-49, 174-179), for the double-layer kernel ----
// x <= 2: K1 = (ln(x/2) + gamma) I1 + 1/x - (x/4) S with I1 = (x/2) sum c_k q^k,
// c_k = 1/(k! (k+1)!), S = sum (H_k + H_{k+1}) c_k q^k, q = x^2/4: fixed
// degree-16 polynomials (tail < 1e-27 for q <= 1, where the reference loop
// stops at a 1e-19 relative term).  x > 2: the K1 Chebyshev fit of
// K1(x) e^x sqrt(x) on the reference's dyadic intervals.
static __constant__ double c_k1_c[17] = {
    1.0, 0.5, 0.08333333333333333, 0.006944444444444444, 0.00034722222222222224,
    1.1574074074074073e-05, 2.755731922398589e-07, 4.920949861426052e-09, 6.834652585313961e-11,
    7.594058428126623e-13, 6.903689480115112e-15, 5.230067787965994e-17, 3.352607556388458e-19,
    1.842092063949702e-21, 8.771866971189057e-24, 3.654944571328774e-26, 1.3437296218120491e-28};
static __constant__ double c_k1_s[17] = {
    1.0, 1.25, 0.2777777777777778, 0.027199074074074073, 0.0015162037037037036,
    5.4783950617283953e-05, 1.3896762408667172e-06, 2.613375872835907e-08, 3.791062453869784e-10,
    4.3726106266713215e-12, 4.106898277957945e-14, 3.202416543243305e-16, 2.1065588026621898e-18,
    1.1847776309828747e-20, 5.762933548568204e-23, 2.448432012616415e-25, 9.16461430197137e-28};

__device__ __forceinline__ double k1_small(double x) {
    const double q = 0.25 * x * x;
    double i1s = c_k1_c[16], s = c_k1_s[16];
#pragma unroll
    for (int k = 15; k >= 0; --k) {
        i1s = fma(i1s, q, c_k1_c[k]);
        s = fma(s, q, c_k1_s[k]);
    }
    constexpr double kGamma = 0.57721566490153286061;
    return (log(0.5 * x) + kGamma) * (0.5 * x * i1s) + 1.0 / x - 0.25 * x * s;
}

__device__ __forceinline__ double k1_dev(double x, const double* tab1) {
    return x <= 2.0 ? k1_small(x) : k0_large(x, tab1);  // same fit layout
}

// ---- fast K0 for the treecode's proxy loop (same accuracy, fewer ops) ----
// x > 2: quarter-octave intervals with 14-term Chebyshev fits (the nearest
// singularity of g at 0 is >= 11 half-widths away: rho^-14 < 1e-18); the
// interval comes from the exponent and two mantissa compares, the map onto
// [-1, 1] is one FMA.  x <= 2: the series truncated at q^12 (tail < 1e-19).
constexpr int kK0FastIntervals = 36;  // [2, 1024]
constexpr int kK0FastCoeffs = 14;
constexpr int kK0FastStride = 16;     // 14 coefficients + (a, b)
void k0_fit_fast_host(double* out);

__device__ __forceinline__ double k0_small12(double x) {
    const double q = 0.25 * x * x;
    double i0 = c_k0_i0[12], s = c_k0_h[12];
#pragma unroll
    for (int k = 11; k >= 0; --k) {
        i0 = fma(i0, q, c_k0_i0[k]);
        s = fma(s, q, c_k0_h[k]);
    }
    constexpr double kGamma = 0.57721566490153286061;
    return -(log(0.5 * x) + kGamma) * i0 + s;
}

// tab: kK0FastIntervals x kK0FastStride doubles (shared memory)
__device__ __forceinline__ double k0_fast(double x, const double* tab) {
    if (x <= 2.0) return k0_small12(x);
    if (x > 745.0) return 0.0;  // exp(-x) underflows (kernel.cpp:158-161)
    const int hi = __double2hiint(x);
    const int e = (hi >> 20) - 1023;                       // x = 2^e m, e >= 1
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(x));
    int iv = 4 * (e - 1) + (m >= 1.189207115002721) + (m >= 1.4142135623730951) + (m >= 1.6817928305074290);
    iv = min(iv, kK0FastIntervals - 1);
    const double* c = tab + iv * kK0FastStride;
    const double u = fma(x, c[kK0FastCoeffs], c[kK0FastCoeffs + 1]);
    const double u2 = 2.0 * u;
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int k = kK0FastCoeffs - 1; k >= 1; --k) {
        const double b0 = fma(u2, b1, c[k] - b2);
        b2 = b1;
        b1 = b0;
    }
    const double g = fma(u, b1, 0.5 * c[0] - b2);
    return g * exp(-x) * rsqrt(x);
}

}  // namespace vpg
