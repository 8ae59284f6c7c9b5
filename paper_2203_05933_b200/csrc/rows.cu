// rows.cu -- correction-row generation on the device: the
// rows of VolumePotentialOperator's correction map (potential.cpp:133-349),
//
//   pool row = (accurate V-hat row - smooth_potential_row) . C
//
// with the accurate row from one of the reference's quadratures
//   SingularTargetRule::row      (singular.cpp:343-415)  "self" rule: a split
//       -t log t / t Gauss rule (20 + 20 points) along every ray from the
//       target to the reference-cell boundary,
//   reduce_to_rays + apply_ray_quadrature (singular.cpp:229-310) "ray" rule:
//       graded ray rules from a boundary star point (the singular rule when
//       the star is the target, per-ray near rules bucketed by decade),
//   box_correction_table         (singular.cpp:486-646)  the shared lattice
//       rows of uniform boxes (Laplace: the h-independent log moments
//       rescaled; modified Helmholtz: per h),
// and the smooth row (singular.cpp:428-456) on the operator's oversampled
// source rule.
//
// Layout of the work: one CTA per row task.  Thread 0 resolves the task
// geometry (Cell::invert, nearest_reference_point, the nearest table star,
// geom.cuh) and the panel endpoints of boundary_discretization; the rays are
// laid out in shared memory (per ray: start, direction, weight factor, inner
// rule); then the CTA walks the flattened (ray, inner node) list in tiles of
// 128 nodes: each thread maps one node (map_deriv, the kernel value, the
// basis at the node into a smem tile), and the tile is folded into the
// row's partial sums by (group, basis) threads.  Sums are fixed-order per
// task, so rows are run-to-run identical.
//
// Host side (this file, restated from quad1d.cpp): Gauss-Legendre by Newton
// in long double, the graded panel rules, the ray rules, and the Gauss rules
// for the weights t and -t log t (Stieltjes on a deep graded rule + Golub-
// Welsch with a tridiagonal QL eigensolver in long double).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "geom.cuh"
#include "k0.cuh"
#include "maps.cuh"
#include "plan.cuh"

namespace vpg {
const double* k0_table_dev();
}

using vpg::geom::V2;

// Triangle rows at p = 8 accumulate in registers (1) or through the smem
// basis tile like every other row (0, A/B)
#ifndef VPG_ROWS_REGACC
#define VPG_ROWS_REGACC 0  // 1: 192 registers cost occupancy, rows 0.61 -> 0.71 s on 1.34M dofs
#endif

namespace vpg {
namespace rows {

constexpr double kInvTwoPi = 0.15915494309189533577;
constexpr double kEulerGamma = 0.57721566490153286061;
constexpr int kMaxP = 12;
constexpr int kMaxNb = kMaxP * kMaxP;
constexpr int kThreads = 128;
constexpr int kTile = 128;
constexpr int kMaxBnodes = geom::kMaxEndpoints * 16;
constexpr int kNearQ0 = -2, kNearQ1 = 9;  // ray_near_rule decade buckets (d in [1e-9, 16])
constexpr int kNumNear = kNearQ1 - kNearQ0 + 1;

// ------------------------------------------------------- host: 1-D rules --
struct Rule1 {
    std::vector<double> x, w;
};

// quad1d.cpp:17-49
Rule1 gauss_legendre(int n) {
    Rule1 r;
    r.x.resize(size_t(n));
    r.w.resize(size_t(n));
    for (int i = 0; i < (n + 1) / 2; ++i) {
        long double x = std::cos(M_PI * (i + 0.75L) / (n + 0.5L));
        long double dp = 0;
        for (int it = 0; it < 100; ++it) {
            long double p0 = 1, p1 = x;
            for (int k = 2; k <= n; ++k) {
                long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1);
            long double dx = p1 / dp;
            x -= dx;
            if (std::abs(dx) < 1e-19L) break;
        }
        long double w = 2.0L / ((1 - x * x) * dp * dp);
        r.x[size_t(i)] = static_cast<double>(-x);
        r.w[size_t(i)] = static_cast<double>(w);
        r.x[size_t(n - 1 - i)] = static_cast<double>(x);
        r.w[size_t(n - 1 - i)] = static_cast<double>(w);
    }
    if (n == 1) {
        r.x[0] = 0;
        r.w[0] = 2;
    }
    return r;
}

void append_panel(Rule1& r, const Rule1& base, double a, double b) {
    const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
    for (size_t i = 0; i < base.x.size(); ++i) {
        r.x.push_back(mid + half * base.x[i]);
        r.w.push_back(half * base.w[i]);
    }
}

// quad1d.cpp:62-82
Rule1 build_graded(double cutoff, double sigma, int points) {
    const Rule1 base = gauss_legendre(points);
    Rule1 r;
    double hi = 1.0;
    while (hi > cutoff) {
        double lo = hi * sigma;
        if (lo <= cutoff) lo = 0;
        if (lo == 0) {
            append_panel(r, base, hi * 0.5, hi);
            append_panel(r, base, 0, hi * 0.5);
        } else {
            append_panel(r, base, lo, hi);
        }
        hi = lo;
    }
    if (r.x.empty()) {
        append_panel(r, base, 0.5, 1.0);
        append_panel(r, base, 0, 0.5);
    }
    return r;
}

// near_rule_impl for the shallow ray rules (quad1d.cpp:87-102): bucket q =
// floor(-log10 d), graded down to max(10^(-q-1), 3e-8).
Rule1 ray_near_rule_bucket(int q) {
    const double lower = std::pow(10.0, -q - 1);
    double cutoff = std::max(lower, 3e-8);
    if (cutoff >= 1.0) cutoff = 0.999;
    return build_graded(cutoff, 0.25, 16);
}

// Symmetric tridiagonal eigenproblem (diagonal d, off-diagonal e[i] between
// i and i+1) by implicit QL with Wilkinson-type shifts, long double; returns
// ascending eigenvalues and the first component of each unit eigenvector
// (all Golub-Welsch needs).
void tridiag_eig(std::vector<long double> d, std::vector<long double> e, std::vector<long double>& lam,
                 std::vector<long double>& v0) {
    const int n = int(d.size());
    e.resize(size_t(n), 0.0L);
    std::vector<long double> z(static_cast<size_t>(n) * static_cast<size_t>(n), 0.0L);  // eigenvectors, columns
    for (int i = 0; i < n; ++i) z[size_t(i) * n + i] = 1.0L;
    for (int l = 0; l < n; ++l) {
        for (int iter = 0; iter < 200; ++iter) {
            int m = l;
            for (; m < n - 1; ++m) {
                const long double dd = std::fabs(d[size_t(m)]) + std::fabs(d[size_t(m + 1)]);
                if (std::fabs(e[size_t(m)]) <= 1e-30L * dd) break;
            }
            if (m == l) break;
            long double g = (d[size_t(l + 1)] - d[size_t(l)]) / (2.0L * e[size_t(l)]);
            long double r = std::hypot(g, 1.0L);
            g = d[size_t(m)] - d[size_t(l)] + e[size_t(l)] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
            long double s = 1, c = 1, p = 0;
            int i = m - 1;
            for (; i >= l; --i) {
                long double f = s * e[size_t(i)], b = c * e[size_t(i)];
                r = std::hypot(f, g);
                e[size_t(i + 1)] = r;
                if (r == 0) {
                    d[size_t(i + 1)] -= p;
                    e[size_t(m)] = 0;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[size_t(i + 1)] - p;
                r = (d[size_t(i)] - g) * s + 2.0L * c * b;
                p = s * r;
                d[size_t(i + 1)] = g + p;
                g = c * r - b;
                for (int k = 0; k < n; ++k) {
                    f = z[size_t(k) * n + i + 1];
                    z[size_t(k) * n + i + 1] = s * z[size_t(k) * n + i] + c * f;
                    z[size_t(k) * n + i] = c * z[size_t(k) * n + i] - s * f;
                }
            }
            if (r == 0 && i >= l) continue;
            d[size_t(l)] -= p;
            e[size_t(l)] = g;
            e[size_t(m)] = 0;
        }
    }
    std::vector<int> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return d[size_t(a)] < d[size_t(b)]; });
    lam.resize(size_t(n));
    v0.resize(size_t(n));
    for (int j = 0; j < n; ++j) {
        lam[size_t(j)] = d[size_t(ord[size_t(j)])];
        long double nrm = 0;
        for (int k = 0; k < n; ++k) nrm += z[size_t(k) * n + ord[size_t(j)]] * z[size_t(k) * n + ord[size_t(j)]];
        v0[size_t(j)] = z[size_t(ord[size_t(j)])] / std::sqrt(nrm);
    }
}

// build_weighted_gauss (quad1d.cpp:153-212): Gauss rule on [0, 1] for the
// weight t (log_weight false) or -t log t (true).
Rule1 weighted_gauss(int n, bool log_weight) {
    const Rule1 aux = build_graded(1e-15, 0.25, 48);
    const int m = int(aux.x.size());
    std::vector<long double> x(static_cast<size_t>(m)), W(static_cast<size_t>(m));
    for (int i = 0; i < m; ++i) {
        const long double xi = aux.x[size_t(i)];
        x[size_t(i)] = xi;
        W[size_t(i)] = aux.w[size_t(i)] * (log_weight ? -xi * std::log(xi) : xi);
    }
    std::vector<long double> alpha(static_cast<size_t>(n)), beta(static_cast<size_t>(n)), pk(static_cast<size_t>(m), 1.0L), pk1(static_cast<size_t>(m), 0.0L);
    long double mu0 = 0;
    for (int i = 0; i < m; ++i) mu0 += W[size_t(i)];
    long double nrm_prev = 0;
    for (int k = 0; k < n; ++k) {
        long double nrm = 0, xav = 0;
        for (int i = 0; i < m; ++i) {
            const long double q = W[size_t(i)] * pk[size_t(i)] * pk[size_t(i)];
            nrm += q;
            xav += q * x[size_t(i)];
        }
        alpha[size_t(k)] = xav / nrm;
        beta[size_t(k)] = k == 0 ? mu0 : nrm / nrm_prev;
        for (int i = 0; i < m; ++i) {
            const long double next =
                (x[size_t(i)] - alpha[size_t(k)]) * pk[size_t(i)] - (k == 0 ? 0.0L : beta[size_t(k)] * pk1[size_t(i)]);
            pk1[size_t(i)] = pk[size_t(i)];
            pk[size_t(i)] = next;
        }
        nrm_prev = nrm;
    }
    // the reference rounds the Jacobi matrix to double before its eigensolve
    std::vector<long double> d(static_cast<size_t>(n)), e(static_cast<size_t>(n), 0.0L);
    for (int k = 0; k < n; ++k) {
        d[size_t(k)] = static_cast<double>(alpha[size_t(k)]);
        if (k + 1 < n) e[size_t(k)] = std::sqrt(static_cast<double>(beta[size_t(k + 1)]));
    }
    std::vector<long double> lam, v0;
    tridiag_eig(d, e, lam, v0);
    Rule1 r;
    r.x.resize(size_t(n));
    r.w.resize(size_t(n));
    for (int i = 0; i < n; ++i) {
        r.x[size_t(i)] = static_cast<double>(lam[size_t(i)]);
        const double v = static_cast<double>(v0[size_t(i)]);
        r.w[size_t(i)] = static_cast<double>(mu0) * v * v;
    }
    return r;
}

// fejer1 (basis.cpp:143-161): Chebyshev roots ascending, Fejer-1 weights
void fejer1(int p, std::vector<double>& z, std::vector<double>& w) {
    z.resize(size_t(p));
    w.resize(size_t(p));
    for (int i = 0; i < p; ++i) {
        const double theta = (2 * i + 1) * M_PI / (2 * p);
        double s = 0;
        for (int k = 1; k <= p / 2; ++k) s += std::cos(2 * k * theta) / (4.0 * k * k - 1.0);
        z[size_t(i)] = -std::cos(theta);
        w[size_t(i)] = (2.0 / p) * (1 - 2 * s);
    }
}

// ----------------------------------------------------------- device data --
// Rule table: one flat (x, w) array; rule r occupies [off[r], off[r+1]).
enum RuleId : int {
    kGL16 = 0,
    kTLog20 = 1,
    kT20 = 2,
    kRaySing = 3,
    kNear0 = 4,                    // kNear0 + (q - kNearQ0)
    kBoxSrc = kNear0 + kNumNear,   // the operator's q x q box source rule (nodes, w)
    kTriSrc,                       // the operator's triangle source rule
    kBox30,                        // the 30 x 30 box rule of the lattice table's outer ring
    kNumRules
};

struct DevCtx {
    const geom::Curve* curves;
    const geom::Cell* cells;
    const double2* rule_xw;   // (x, w) for 1-D rules; for source rules x = node index into src_nodes
    const int* rule_off;
    const double2* src_nodes; // 2-D source nodes of kBoxSrc / kTriSrc / kBox30 (by rule)
    const double* tri_C;      // nb x nb row-major (values -> coefficients)
    const double* box_C;
    const double* tri_nodes;  // reference interpolation nodes (n x 2)
    const double* box_nodes;
    const double* k0tab;
    int family;
    double lambda;
    int p;
    int nb_tri, nb_box;
};

// Row task jobs
enum Job : int32_t {
    kJobSelf = 0,         // SingularTargetRule(kind, p, zeta0).row(cell, kernel, r0)  [aux: zeta0 given]
    kJobRay = 1,          // reduce_to_rays(cell, zeta0, zstar, kernel, r0) + apply  [zeta0, zstar given]
    kJobSmooth = 2,       // smooth_potential_row(cell, p, rule, r0)  [aux_i = rule id]
    kJobTriSelfNode = 3,  // operator row: SingularTargetRule at tri node aux_i, minus smooth, x C
    kJobTriNearSnap = 4,  // operator row: near rule on the nearest table star, minus smooth, x C
    kJobSelfGeneric = 5,  // operator row: self rule at invert(r0), minus smooth, x C
    kJobNearGeneric = 6,  // operator row: ray rule from nearest_reference_point, minus smooth, x C
    kJobLattice = 7,      // operator row: table row (aux_i = offset * 256 + node) minus smooth, x C
    kJobTableLap = 8,     // box_log entry (aux_i = offset * 256 + node) / -1/2pi on the reference box
    kJobTableHelm = 9,    // box_correction_table entry for modified Helmholtz on the origin box
};

struct RowTask {
    int32_t job;
    int32_t cell;
    int32_t aux_i;
    int32_t pad;
    double2 r0;
    double2 zeta0;
    double2 zstar;
    int64_t out;  // first output double
};

__device__ __forceinline__ V2 v2(double2 a) { return V2{a.x, a.y}; }

__device__ double radial_r2(const DevCtx& c, double r2) {
    if (c.family == VPG_LAPLACE) return -0.25 / M_PI * log(r2);
    return 0.5 / M_PI * k0_dev(c.lambda * sqrt(r2), c.k0tab);
}

// i0_and_t (singular.cpp:317-334)
__device__ void i0_and_t(double x, double& i0, double& tser) {
    const double u = 0.25 * x * x;
    double term = 1.0, hk = 0.0;
    i0 = 1.0;
    double hsum = 0.0;
    for (int k = 1; k <= 80; ++k) {
        term *= u / (static_cast<double>(k) * k);
        hk += 1.0 / k;
        i0 += term;
        hsum += hk * term;
        if (term * (hk + 1.0) <= 1e-18 * (i0 + hsum)) break;
    }
    tser = hsum - kEulerGamma * i0;
}

// Division-free recurrence coefficients of the basis (built once per CTA):
// the Jacobi step P_{k+1}^{(0, b)} = (c1 + c2 x) P_k - c3 P_{k-1} with
// c = (a2, a3, a4) / a1 of jacobi_next (basis.cpp:36-43), and the Q_m step
// Q_{m+1} = q1 s Q_m - q2 z2 Q_{m-1}, q1 = (2m+1)/(m+1), q2 = m/(m+1)
// (basis.cpp:24-34).  The reference divides by a1 and (m+1) per call; the
// reciprocal form differs by rounding only.
struct BasisCoef {
    double jc[kMaxP][kMaxP][3];  // [m][k][c1, c2, c3] for P_{k+1} from P_k (k >= 1)
    double qc[kMaxP][2];         // [m][q1, q2]
    double gam[kMaxNb];          // sqrt(2 (2m+1)(n+1)) at n(n+1)/2 + m (basis.cpp:222)
};

__device__ void basis_coef_init(int p, BasisCoef& B) {
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
        const int m = e / p, k = e % p;
        const double beta = 2 * m + 1;
        if (k >= 1) {
            const double a1 = 2 * (k + 1) * (k + beta + 1) * (2 * k + beta);
            const double a2 = (2 * k + beta + 1) * (-beta * beta);
            const double a3 = (2 * k + beta) * (2 * k + beta + 1) * (2 * k + beta + 2);
            const double a4 = 2 * (k + beta) * k * (2 * k + beta + 2);
            B.jc[m][k][0] = a2 / a1;
            B.jc[m][k][1] = a3 / a1;
            B.jc[m][k][2] = a4 / a1;
        }
        if (k == 0) {
            B.qc[m][0] = double(2 * m + 1) / (m + 1);
            B.qc[m][1] = double(m) / (m + 1);
        }
    }
    for (int n = 0; n < p; ++n)
        for (int m = threadIdx.x; m <= n; m += blockDim.x) B.gam[n * (n + 1) / 2 + m] = sqrt(2 * (2 * m + 1) * (n + 1.0));
}

// basis values at a reference point into out[0..nb) (chebyshev2d_eval,
// koornwinder_eval: basis.cpp:24-45, 193-228)
__device__ void eval_basis(bool box, int p, V2 z, const BasisCoef& B, double* out, int stride) {
    if (box) {
        double tx[kMaxP], ty[kMaxP];
        geom::cheb1d(p, z.x, tx);
        geom::cheb1d(p, z.y, ty);
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) out[(a * p + b) * stride] = tx[a] * ty[b];
        return;
    }
    double q[kMaxP];
    const double xi = z.x, eta = z.y;
    const double s = 2 * xi - (1 - eta);
    const double z2 = (1 - eta) * (1 - eta);
    q[0] = 1;
    if (p > 1) q[1] = s;
    for (int m = 1; m + 1 < p; ++m) q[m + 1] = B.qc[m][0] * s * q[m] - B.qc[m][1] * z2 * q[m - 1];
    const double x = 1 - 2 * eta;
    for (int m = 0; m < p; ++m) {
        const double beta = 2 * m + 1;
        double pkm1 = 0, pk = 1;
        for (int n = m; n < p; ++n) {
            const int k = n - m;
            if (k > 0) {
                const double pk1 = k == 1 ? 0.5 * ((beta + 2) * x - beta)
                                          : (B.jc[m][k - 1][0] + B.jc[m][k - 1][1] * x) * pk - B.jc[m][k - 1][2] * pkm1;
                pkm1 = pk;
                pk = pk1;
            }
            const int idx = n * (n + 1) / 2 + m;
            out[idx * stride] = B.gam[idx] * pk * q[m];
        }
    }
}

// p = 8 (the reference operator's default order) fully unrolled: the
// recurrences stay in registers (the runtime-p loops above index local arrays)
template <int P>
__device__ __forceinline__ void eval_basis_p(bool box, V2 z, const BasisCoef& B, double* out, int stride) {
    if (box) {
        double tx[P], ty[P];
        tx[0] = 1;
        ty[0] = 1;
        if (P > 1) {
            tx[1] = z.x;
            ty[1] = z.y;
        }
#pragma unroll
        for (int k = 2; k < P; ++k) {
            tx[k] = 2 * z.x * tx[k - 1] - tx[k - 2];
            ty[k] = 2 * z.y * ty[k - 1] - ty[k - 2];
        }
#pragma unroll
        for (int a = 0; a < P; ++a)
#pragma unroll
            for (int b = 0; b < P; ++b) out[(a * P + b) * stride] = tx[a] * ty[b];
        return;
    }
    double q[P];
    const double xi = z.x, eta = z.y;
    const double s = 2 * xi - (1 - eta);
    const double z2 = (1 - eta) * (1 - eta);
    q[0] = 1;
    if (P > 1) q[1] = s;
#pragma unroll
    for (int m = 1; m + 1 < P; ++m) q[m + 1] = B.qc[m][0] * s * q[m] - B.qc[m][1] * z2 * q[m - 1];
    const double x = 1 - 2 * eta;
#pragma unroll
    for (int m = 0; m < P; ++m) {
        const double beta = 2 * m + 1;
        double pkm1 = 0, pk = 1;
#pragma unroll
        for (int n = m; n < P; ++n) {
            const int k = n - m;
            if (k > 0) {
                const double pk1 = k == 1 ? 0.5 * ((beta + 2) * x - beta)
                                          : (B.jc[m][k - 1][0] + B.jc[m][k - 1][1] * x) * pk - B.jc[m][k - 1][2] * pkm1;
                pkm1 = pk;
                pk = pk1;
            }
            const int idx = n * (n + 1) / 2 + m;
            out[idx * stride] = B.gam[idx] * pk * q[m];
        }
    }
}


struct RowSmem {
    double ep[geom::kMaxEndpoints];
    BasisCoef bc;
    double inv_t[40];  // 1 / t of the split self rule's inner nodes
    double acc[kMaxNb];
    double sm[kMaxNb];
    // the rays of the current layout, reconstructed per node from their panel
    // (A, E, mid, half of the kept panels) instead of stored (smem: 4 CTAs/SM)
    double pan[geom::kMaxEndpoints][6];
    int rstart[kMaxBnodes + 1];        // first flattened node of each ray
    unsigned char rrule[kMaxBnodes];  // inner rule of each ray
    int np;          // panel endpoints
    int nrays;
    int total;       // flattened node count
    int mode;        // 0 self split rule, 1 rays
    int box;
    int cell;
    int err;
    int smooth_rule; // rule for the subtraction, -1 none
    int post;        // 0 raw, 1 x C, 2 / -kInvTwoPi
    long long nodes; // quadrature nodes evaluated (accurate + smooth rules)
    double r0x, r0y, z0x, z0y, zsx, zsy;
};

// Ray b of the layout: its boundary node and per-ray weight factor (the
// expressions of boundary_discretization, singular.cpp:184-190).
__device__ __forceinline__ void ray_at(const RowSmem& S, const double2* gl, V2 star, int b, V2& zeta, double& factor) {
    const double* pn = S.pan[b >> 4];
    const int l = b & 15;
    const V2 A{pn[0], pn[1]}, E{pn[2], pn[3]};
    const double mid = pn[4], half = pn[5];
    const double s = mid + half * gl[l].x;
    zeta = A + s * E;
    factor = geom::cross(zeta - star, E) * (gl[l].y * half);
}

// the ray owning flattened node i (binary search over the ray starts)
__device__ __forceinline__ int ray_of(const RowSmem& S, int i) {
    int lo = 0, hi = S.nrays - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.rstart[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// One node of the current task: reference point, weight, kernel factor.
__device__ bool node_at(const DevCtx& c, const RowSmem& S, const geom::Cell& cell, int i, V2& chi, double& coef) {
    const double2* xw = c.rule_xw;
    const V2 r0{S.r0x, S.r0y};
    if (S.mode == 0) {  // split self rule: 20 -t log t + 20 t nodes per ray
        const int b = i / 40, l = i % 40;
        const V2 z0{S.z0x, S.z0y};
        V2 zeta;
        double factor;
        ray_at(S, xw + c.rule_off[kGL16], z0, b, zeta, factor);
        const V2 dir = zeta - z0;
        const bool log_part = l < 20;
        const double2 tw = log_part ? xw[c.rule_off[kTLog20] + l] : xw[c.rule_off[kT20] + l - 20];
        chi = z0 + tw.x * dir;
        const double w = tw.y * factor;
        V2 x, dxi, deta;
        double jac;
        geom::map_deriv(cell, c.curves, chi, x, dxi, deta, jac);
        const double r = geom::dist(x, r0);
        double k;
        if (c.family == VPG_LAPLACE) {
            k = log_part ? kInvTwoPi : -kInvTwoPi * log(r * S.inv_t[l]);
        } else {
            double i0, tser;
            i0_and_t(c.lambda * r, i0, tser);
            k = log_part ? kInvTwoPi * i0 : kInvTwoPi * (tser - i0 * log(c.lambda * r * (0.5 * S.inv_t[l])));
        }
        coef = w * jac * k;
        return true;
    }
    if (S.mode == 1) {  // rays: binary search the ray owning flattened node i
        const int b = ray_of(S, i);
        const int l = i - S.rstart[b];
        const double2 tw = xw[c.rule_off[S.rrule[b]] + l];
        const V2 zs{S.zsx, S.zsy};
        V2 zeta;
        double factor;
        ray_at(S, xw + c.rule_off[kGL16], zs, b, zeta, factor);
        const V2 dir = zeta - zs;
        chi = V2{zs.x + tw.x * dir.x, zs.y + tw.x * dir.y};
        const double w = tw.x * tw.y * factor;
        V2 x, dxi, deta;
        double jac;
        geom::map_deriv(cell, c.curves, chi, x, dxi, deta, jac);
        coef = w * jac * radial_r2(c, geom::norm2(x - r0));
        return true;
    }
    // smooth rule (mode 2): node i of rule S.smooth_rule
    const double2 zw = xw[c.rule_off[S.smooth_rule] + i];
    const double2 zn = c.src_nodes[int(zw.x)];
    chi = V2{zn.x, zn.y};
    V2 x, dxi, deta;
    double jac;
    geom::map_deriv(cell, c.curves, chi, x, dxi, deta, jac);
    const double r2 = geom::norm2(x - r0);
    if (r2 == 0.0) {  // singular.cpp:441: a source node on the target contributes nothing
        coef = 0.0;
        return false;
    }
    coef = zw.y * jac * radial_r2(c, r2);
    return true;
}

// Walks the flattened node list of the current mode, adding into dst[nb].
// Triangle rows at p = 8: each thread keeps its own 36 row sums in registers
// (coef * basis added node by node, no smem tile) and the CTA adds the
// threads' sums once per task (warp butterflies, then the 4 warps in order).
__device__ void accumulate_tri8(const DevCtx& c, RowSmem& S, const geom::Cell& cell, int total,
                                double* red, double* dst) {
    constexpr int NB = 36;
    double acc[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) acc[k] = 0.0;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        V2 chi;
        double coef = 0.0;
        if (!node_at(c, S, cell, i, chi, coef)) continue;
        // koornwinder_eval (basis.cpp:193-228) with the coefficient tables, fused
        // with the accumulation
        double q[8];
        const double xi = chi.x, eta = chi.y;
        const double sv = 2 * xi - (1 - eta);
        const double z2 = (1 - eta) * (1 - eta);
        q[0] = 1;
        q[1] = sv;
#pragma unroll
        for (int m = 1; m + 1 < 8; ++m) q[m + 1] = S.bc.qc[m][0] * sv * q[m] - S.bc.qc[m][1] * z2 * q[m - 1];
        const double x = 1 - 2 * eta;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const double beta = 2 * m + 1;
            const double cq = coef * q[m];
            double pkm1 = 0, pk = 1;
#pragma unroll
            for (int n = m; n < 8; ++n) {
                const int k = n - m;
                if (k > 0) {
                    const double pk1 = k == 1 ? 0.5 * ((beta + 2) * x - beta)
                                              : (S.bc.jc[m][k - 1][0] + S.bc.jc[m][k - 1][1] * x) * pk -
                                                    S.bc.jc[m][k - 1][2] * pkm1;
                    pkm1 = pk;
                    pk = pk1;
                }
                const int idx = n * (n + 1) / 2 + m;
                acc[idx] = fma(cq, S.bc.gam[idx] * pk, acc[idx]);
            }
        }
    }
    // reduction: butterflies within each warp, then the warps in order
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp * NB + k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NB) {
        double v = 0.0;
        for (int w = 0; w < nw; ++w) v += red[w * NB + threadIdx.x];
        dst[threadIdx.x] += v;
    }
    __syncthreads();
}

__device__ void accumulate(const DevCtx& c, RowSmem& S, const geom::Cell& cell, int total, int nb,
                           double* tile, double* ctile, double* dst) {
    if (threadIdx.x == 0) S.nodes += total;
#if VPG_ROWS_REGACC
    if (!S.box && c.p == 8) {
        accumulate_tri8(c, S, cell, total, tile, dst);
        return;
    }
#endif
    const int groups = max(1, kThreads / nb);
    const int g = threadIdx.x / nb, n = threadIdx.x % nb;
    const bool active = g < groups && threadIdx.x < groups * nb;
    double part[(kMaxNb + kThreads - 1) / kThreads];  // basis entries this thread owns when nb > kThreads
    const int nown = nb > kThreads ? (nb + kThreads - 1) / kThreads : 1;
    for (int k = 0; k < nown; ++k) part[k] = 0.0;
    const int stride = kTile + 1;
    for (int t0 = 0; t0 < total; t0 += kTile) {
        const int i = t0 + threadIdx.x;
        if (threadIdx.x < kTile) {
            double coef = 0.0;
            if (i < total) {
                V2 chi;
                if (node_at(c, S, cell, i, chi, coef))
                {
                    if (c.p == 8)
                        eval_basis_p<8>(S.box, chi, S.bc, tile + threadIdx.x, stride);
                    else
                        eval_basis(S.box, c.p, chi, S.bc, tile + threadIdx.x, stride);
                }
                else
                    for (int k = 0; k < nb; ++k) tile[k * stride + threadIdx.x] = 0.0;
            }
            ctile[threadIdx.x] = i < total ? coef : 0.0;
        }
        __syncthreads();
        const int cnt = min(kTile, total - t0);
        if (nb <= kThreads) {
            if (active) {
                double a = 0.0;
                for (int j = g; j < cnt; j += groups) a = fma(ctile[j], tile[n * stride + j], a);
                part[0] += a;
            }
        } else {
            for (int k = 0; k < nown; ++k) {
                const int nn = threadIdx.x + k * kThreads;
                if (nn < nb) {
                    double a = 0.0;
                    for (int j = 0; j < cnt; ++j) a = fma(ctile[j], tile[nn * stride + j], a);
                    part[k] += a;
                }
            }
        }
        __syncthreads();
    }
    // fold the groups in a fixed order
    if (nb <= kThreads) {
        if (active) ctile[threadIdx.x] = part[0];
        __syncthreads();
        if (threadIdx.x < nb) {
            double s = 0.0;
            for (int gg = 0; gg < groups; ++gg) s += ctile[gg * nb + threadIdx.x];
            dst[threadIdx.x] += s;
        }
        __syncthreads();
    } else {
        for (int k = 0; k < nown; ++k) {
            const int nn = threadIdx.x + k * kThreads;
            if (nn < nb) dst[nn] += part[k];
        }
        __syncthreads();
    }
}

// Lays out the rays of a boundary star (boundary_discretization, assemble
// rays): thread 0 finds the panel endpoints; then every thread fills rays.
// mode 0: split self rule (fixed 40 nodes per ray); mode 1: ray rules.
__device__ void layout_rays(const DevCtx& c, RowSmem& S, const geom::Cell& cell, V2 star, int mode,
                            bool all_singular, double d) {
    if (threadIdx.x == 0) S.np = geom::boundary_endpoints(S.box, star, S.ep);
    __syncthreads();
    // kept panels: serial (<= 67)
    __shared__ int kept[geom::kMaxEndpoints];
    __shared__ int nkept;
    if (threadIdx.x == 0) {
        int m = 0;
        for (int k = 0; k < S.np; ++k) {
            V2 A, E;
            double sa, sb;
            if (geom::boundary_panel(S.box, star, S.ep, S.np, k, A, E, sa, sb)) kept[m++] = k;
        }
        nkept = m;
        S.nrays = m * 16;
    }
    __syncthreads();
    const double2* gl = c.rule_xw + c.rule_off[kGL16];
    for (int m = threadIdx.x; m < nkept; m += blockDim.x) {
        V2 A, E;
        double sa, sb;
        geom::boundary_panel(S.box, star, S.ep, S.np, kept[m], A, E, sa, sb);
        double* pn = S.pan[m];
        pn[0] = A.x;
        pn[1] = A.y;
        pn[2] = E.x;
        pn[3] = E.y;
        pn[4] = 0.5 * (sa + sb);
        pn[5] = 0.5 * (sb - sa);
    }
    __syncthreads();
    V2 rstar{0, 0};
    if (mode == 1 && !all_singular) rstar = geom::cell_map(cell, c.curves, star);
    for (int b = threadIdx.x; b < S.nrays; b += blockDim.x) {
        int rule = 0;
        if (mode == 1) {
            if (all_singular) {
                rule = kRaySing;
            } else {
                V2 zeta;
                double factor;
                ray_at(S, gl, star, b, zeta, factor);
                const double len = geom::dist(geom::cell_map(cell, c.curves, zeta), rstar);
                const double deff = fmin(fmax(d / fmax(len, 1e-300), 1e-9), 16.0);
                const int q = int(floor(-log10(deff)));
                rule = kNear0 + min(max(q, kNearQ0), kNearQ1) - kNearQ0;
            }
        }
        S.rrule[b] = (unsigned char)rule;
        S.rstart[b + 1] = mode == 0 ? 40 : c.rule_off[rule + 1] - c.rule_off[rule];
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // ray sizes -> starts
        S.rstart[0] = 0;
        for (int b = 0; b < S.nrays; ++b) S.rstart[b + 1] += S.rstart[b];
        S.total = S.rstart[S.nrays];
    }
    __syncthreads();
}

__device__ bool is_self_target(V2 zeta0, V2 zstar) {
    return geom::dist(zstar, zeta0) <= 1e-12 * (1.0 + geom::norm(zeta0));
}

#if VPG_ROWS_REGACC
__global__ void __maxnreg__(192)
#else
__global__ void __launch_bounds__(kThreads)
#endif
rows_kernel(DevCtx c, const RowTask* tasks, const double* table, double* out, int* err,
            unsigned long long* nodes_done) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ RowSmem S;
    const RowTask T = tasks[blockIdx.x];
    const int p = c.p;
    for (int i = threadIdx.x; i < kMaxNb; i += blockDim.x) {
        S.acc[i] = 0.0;
        S.sm[i] = 0.0;
    }
    // Koornwinder normalisations sqrt(2 (2m+1)(n+1)) (basis.cpp:222)
    basis_coef_init(p, S.bc);
    for (int l = threadIdx.x; l < 40; l += blockDim.x)
        S.inv_t[l] = 1.0 / c.rule_xw[l < 20 ? c.rule_off[kTLog20] + l : c.rule_off[kT20] + l - 20].x;
    // the task's cell: a mesh cell, or the reference box / the origin box for the tables
    geom::Cell cell = c.cells[T.cell];
    if (threadIdx.x == 0) {
        S.err = 0;
        S.nodes = 0;
        S.cell = T.cell;
        S.box = cell.type == geom::kBox;
        S.smooth_rule = -1;
        S.post = 0;
        S.r0x = T.r0.x;
        S.r0y = T.r0.y;
        S.z0x = T.zeta0.x;
        S.z0y = T.zeta0.y;
        S.zsx = T.zstar.x;
        S.zsy = T.zstar.y;
        S.mode = -1;
        const V2 r0 = v2(T.r0);
        const bool helm = c.family != VPG_LAPLACE;
        switch (T.job) {
            case kJobSelf: S.mode = 0; break;
            case kJobRay: S.mode = 1; break;
            case kJobSmooth: S.mode = 2; S.smooth_rule = T.aux_i; break;
            case kJobTriSelfNode: {  // potential.cpp:300-315
                S.mode = 0;
                S.z0x = c.tri_nodes[2 * T.aux_i];
                S.z0y = c.tri_nodes[2 * T.aux_i + 1];
                S.post = 1;
                break;
            }
            case kJobTriNearSnap: {  // potential.cpp:322-334, singular.cpp:566-583
                const V2 z0 = geom::invert(cell, c.curves, r0);
                const V2 zs = geom::nearest_reference_point(cell, c.curves, r0, nullptr);
                const double tpar = geom::nearest_boundary_param(0, zs);
                const double u = geom::wrap_param(tpar, 3);
                const long k = lround(u * 64);
                const double tstar = double(k % 192) / 64;
                const V2 star = geom::ref_boundary_point(0, tstar);
                S.z0x = z0.x;
                S.z0y = z0.y;
                S.zsx = star.x;
                S.zsy = star.y;
                S.mode = 1;
                S.post = 1;
                break;
            }
            case kJobSelfGeneric:
            case kJobNearGeneric: {  // potential.cpp:351-358, singular.cpp:458-470
                const V2 z0 = geom::invert(cell, c.curves, r0);
                const V2 zs = T.job == kJobSelfGeneric ? z0 : geom::nearest_reference_point(cell, c.curves, r0, nullptr);
                S.z0x = z0.x;
                S.z0y = z0.y;
                S.zsx = zs.x;
                S.zsy = zs.y;
                S.mode = T.job == kJobSelfGeneric ? 0 : 1;
                S.post = 1;
                break;
            }
            case kJobLattice: S.mode = 3; S.post = 1; break;
            case kJobTableLap:
            case kJobTableHelm: {  // singular.cpp:486-516, 615-643
                const int o = T.aux_i / 256, j = T.aux_i % 256;
                const int ox = o % 5 - 2, oy = o / 5 - 2;
                const int ring = max(abs(ox), abs(oy));
                const V2 z0{c.box_nodes[2 * j] + 2.0 * ox, c.box_nodes[2 * j + 1] + 2.0 * oy};
                const double half = 0.5 * cell.h;
                const V2 rr = T.job == kJobTableLap ? z0 : V2{half * z0.x, half * z0.y};
                S.r0x = rr.x;
                S.r0y = rr.y;
                S.z0x = z0.x;
                S.z0y = z0.y;
                if (ring == 0) {
                    S.mode = 0;
                } else if (ring == 1) {
                    const V2 zs = geom::nearest_reference_point(cell, c.curves, rr, nullptr);
                    S.zsx = zs.x;
                    S.zsy = zs.y;
                    S.mode = 1;
                } else {
                    S.mode = 2;
                    S.smooth_rule = kBox30;
                }
                S.post = T.job == kJobTableLap ? 2 : 0;
                break;
            }
        }
        // SingularTargetRule::row: modified Helmholtz on a large cell takes the
        // graded composite rule from the target itself (singular.cpp:386-391)
        if (S.mode == 0 && helm && c.lambda * geom::cell_diameter(cell, c.curves) > 8.0) {
            S.mode = 1;
            S.zsx = S.z0x;
            S.zsy = S.z0y;
        }
        if (S.post == 1) S.smooth_rule = S.box ? kBoxSrc : kTriSrc;
    }
    __syncthreads();
    const int nb = S.box ? p * p : p * (p + 1) / 2;
    double* tile = dyn;                      // [nb][kTile + 1]
    double* ctile = dyn + nb * (kTile + 1);  // [max(kTile, kThreads)]
    const V2 r0{S.r0x, S.r0y}, z0{S.z0x, S.z0y}, zs{S.zsx, S.zsy};

    if (S.mode == 0) {
        layout_rays(c, S, cell, z0, 0, true, 0.0);
        accumulate(c, S, cell, S.total, nb, tile, ctile, S.acc);
    } else if (S.mode == 1) {
        // assemble_rays (singular.cpp:229-272)
        bool all_singular = is_self_target(z0, zs);
        double d = 0.0;
        if (!all_singular) {
            V2 lo, hi;
            geom::bounding_box(cell, c.curves, lo, hi);
            d = geom::dist(r0, geom::cell_map(cell, c.curves, zs));
            all_singular = d <= 1e-14 * geom::norm(hi - lo);
        }
        layout_rays(c, S, cell, zs, 1, all_singular, d);
        // node checks of assemble_rays: inside the closed cell, never on the target
        for (int i = threadIdx.x; i < S.total; i += blockDim.x) {
            const int b = ray_of(S, i);
            const double t = c.rule_xw[c.rule_off[S.rrule[b]] + i - S.rstart[b]].x;
            V2 zeta;
            double factor;
            ray_at(S, c.rule_xw + c.rule_off[kGL16], zs, b, zeta, factor);
            const V2 chi{zs.x + t * (zeta.x - zs.x), zs.y + t * (zeta.y - zs.y)};
            const double pad = 1e-12;
            const bool inside = S.box ? fabs(chi.x) <= 1 + pad && fabs(chi.y) <= 1 + pad
                                      : chi.x >= -pad && chi.y >= -pad && chi.x + chi.y <= 1 + pad;
            if (!inside) atomicOr(&S.err, 1);
            if (chi.x == z0.x && chi.y == z0.y) atomicOr(&S.err, 2);
        }
        accumulate(c, S, cell, S.total, nb, tile, ctile, S.acc);
    } else if (S.mode == 2) {
        // raw smooth row (lattice-table outer ring / testing)
        const int tot = c.rule_off[S.smooth_rule + 1] - c.rule_off[S.smooth_rule];
        accumulate(c, S, cell, tot, nb, tile, ctile, S.acc);
        S.smooth_rule = -1;
    } else if (S.mode == 3) {
        // the lattice table row (potential.cpp:284): table[o](j, :)
        for (int n = threadIdx.x; n < nb; n += blockDim.x) S.acc[n] = table[int64_t(T.aux_i / 256) * 256 * nb +
                                                                           int64_t(T.aux_i % 256) * nb + n];
        __syncthreads();
    }
    if (S.smooth_rule >= 0) {
        const int m0 = S.mode;
        if (threadIdx.x == 0) S.mode = 2;
        __syncthreads();
        const int tot = c.rule_off[S.smooth_rule + 1] - c.rule_off[S.smooth_rule];
        accumulate(c, S, cell, tot, nb, tile, ctile, S.sm);
        if (threadIdx.x == 0) S.mode = m0;
        __syncthreads();
    }
    // post: (acc - sm) . C  |  acc / -kInvTwoPi  |  acc
    double* o = out + T.out;
    if (S.post == 1) {
        const double* C = S.box ? c.box_C : c.tri_C;
        for (int n = threadIdx.x; n < nb; n += blockDim.x) S.acc[n] -= S.sm[n];
        __syncthreads();
        for (int j = threadIdx.x; j < nb; j += blockDim.x) {
            double s = 0.0;
            for (int n = 0; n < nb; ++n) s = fma(S.acc[n], C[n * nb + j], s);
            o[j] = s;
        }
    } else if (S.post == 2) {
        for (int n = threadIdx.x; n < nb; n += blockDim.x) o[n] = S.acc[n] / -kInvTwoPi;
    } else {
        for (int n = threadIdx.x; n < nb; n += blockDim.x) o[n] = S.acc[n];
    }
    if (threadIdx.x == 0 && S.err) atomicOr(err, S.err);
    if (threadIdx.x == 0) atomicAdd(nodes_done + (S.box ? 1 : 0), (unsigned long long)S.nodes);
}

// Laplace lattice table from the log moments (singular.cpp:596-613):
// out[o](i, n) = -1/2pi * area * (L[o](i, n) + shift * beta_n)
__global__ void lap_table_kernel(const double* L, int p, double h, double* out) {
    const int nb = p * p;
    const int64_t tot = 25LL * nb * nb;  // entries (o, j, n), stored at (o * 256 + j) * nb + n
    const double area = 0.25 * h * h;
    const double shift = log(0.5 * h);
    for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < tot; f += int64_t(gridDim.x) * blockDim.x) {
        const int n = int(f % nb);
        const int64_t oj = f / nb;
        const int64_t e = ((oj / nb) * 256 + oj % nb) * nb + n;
        const int a = n / p, b = n % p;
        const double ma = a % 2 ? 0.0 : 2.0 / (1.0 - double(a) * a);
        const double mb = b % 2 ? 0.0 : 2.0 / (1.0 - double(b) * b);
        out[e] = -kInvTwoPi * area * (L[e] + shift * (ma * mb));
    }
}

}  // namespace rows
}  // namespace vpg

using namespace vpg;
using namespace vpg::rows;

// --------------------------------------------------------------- context --
struct vpg_rows {
    int device = 0;
    int family = 0;
    double lambda = 0;
    int p = 0, q = 0;
    int ncell = 0;      // mesh cells; two synthetic boxes follow
    int nb_tri = 0, nb_box = 0;
    std::vector<geom::Cell> cells_h;
    std::vector<geom::Curve> curves_h;
    std::vector<double> tri_nodes_h, box_nodes_h;
    std::vector<int> rule_off_h;
    std::vector<double2> rule_xw_h;
    DBuf<geom::Curve> curves;
    DBuf<geom::Cell> cells;
    DBuf<double2> rule_xw, src_nodes;
    DBuf<int> rule_off;
    DBuf<double> tri_C, box_C, tri_nodes, box_nodes;
    DBuf<double> lap_log;   // 25 x 256 x nb box_log moments (Laplace, h-independent)
    std::mutex mu;
    DevCtx ctx() const {
        DevCtx c;
        c.curves = curves.p;
        c.cells = cells.p;
        c.rule_xw = rule_xw.p;
        c.rule_off = rule_off.p;
        c.src_nodes = src_nodes.p;
        c.tri_C = tri_C.p;
        c.box_C = box_C.p;
        c.tri_nodes = tri_nodes.p;
        c.box_nodes = box_nodes.p;
        c.k0tab = k0_table_dev();
        c.family = family;
        c.lambda = lambda;
        c.p = p;
        c.nb_tri = nb_tri;
        c.nb_box = nb_box;
        return c;
    }
    int ref_box() const { return ncell; }      // [-1,1]^2, h = 2
    int origin_box(double h);                  // centre 0, size h (appended on demand)
};

namespace {

template <typename F>
int guarded_r(F&& f) {
    try {
        f();
        return VPG_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return VPG_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        set_error(e.what());
        return VPG_ERR_CUDA;
    }
}

template <typename T>
void upload(DBuf<T>& b, const T* h, size_t n) {
    b.alloc(n);
    if (n) VPG_CUDA(cudaMemcpy(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
}

size_t row_smem_bytes(int nb) { return sizeof(double) * (size_t(nb) * (kTile + 1) + std::max(kTile, kThreads)); }

// returns the quadrature nodes evaluated on triangle / box cells (nodes[2])
void run_tasks(vpg_rows& R, const std::vector<RowTask>& tasks, const double* table, double* out_dev,
               cudaStream_t s, int64_t* nodes_out = nullptr) {
    if (tasks.empty()) return;
    DBuf<int> err;
    err.alloc(1);
    DBuf<unsigned long long> cnt;
    cnt.alloc(2);
    VPG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
    VPG_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), s));
    // triangle rows (p(p+1)/2 basis) and box rows (p^2) launch separately: the
    // smem tile is sized by the basis, so triangle rows fit more CTAs per SM
    std::vector<RowTask> part[2];
    for (const RowTask& t : tasks) part[R.cells_h[size_t(t.cell)].type == geom::kBox ? 1 : 0].push_back(t);
    const DevCtx c = R.ctx();
    DBuf<RowTask> tdk[2];
    for (int kind = 0; kind < 2; ++kind) {
        if (part[kind].empty()) continue;
        upload(tdk[kind], part[kind].data(), part[kind].size());
        const size_t smem = row_smem_bytes(kind ? R.nb_box : R.nb_tri);
        smem_optin(reinterpret_cast<const void*>(&rows_kernel), int(row_smem_bytes(std::max(R.nb_tri, R.nb_box))));
        for (size_t t0 = 0; t0 < part[kind].size(); t0 += 1u << 30) {
            const unsigned n = unsigned(std::min<size_t>(part[kind].size() - t0, 1u << 30));
            rows_kernel<<<n, kThreads, smem, s>>>(c, tdk[kind].p + t0, table, out_dev, err.p, cnt.p);
            VPG_LAUNCH_CHECK();
        }
    }
    int herr = 0;
    unsigned long long nodes[2] = {0, 0};
    VPG_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaMemcpyAsync(nodes, cnt.p, sizeof(nodes), cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
    if (herr & 1) throw Error{VPG_ERR_INVALID_ARGUMENT, "ray node left the reference cell"};
    if (herr & 2) throw Error{VPG_ERR_INVALID_ARGUMENT, "ray node coincides with the target"};
    if (nodes_out) {
        nodes_out[0] = int64_t(nodes[0]);
        nodes_out[1] = int64_t(nodes[1]);
    }
}

}  // namespace

int vpg_rows::origin_box(double h) {
    for (size_t k = size_t(ncell) + 1; k < cells_h.size(); ++k)
        if (cells_h[k].h == h) return int(k);
    geom::Cell b{};
    b.type = geom::kBox;
    b.curve = -1;
    b.center = V2{0, 0};
    b.h = h;
    cells_h.push_back(b);
    upload(cells, cells_h.data(), cells_h.size());
    return int(cells_h.size() - 1);
}

// Builds the table of shared lattice rows for mesh size h on the device:
// 25 offsets x nb_box nodes x nb_box basis (box_correction_table).
static void lattice_table(vpg_rows& R, double h, DBuf<double>& table, cudaStream_t s) {
    const int nb = R.nb_box;
    table.alloc(size_t(25) * 256 * nb);
    if (R.family == VPG_LAPLACE) {
        if (!R.lap_log.p) {
            std::vector<RowTask> tk;
            R.lap_log.alloc(size_t(25) * 256 * nb);
            for (int o = 0; o < 25; ++o)
                for (int j = 0; j < nb; ++j) {
                    RowTask t{};
                    t.job = kJobTableLap;
                    t.cell = R.ref_box();
                    t.aux_i = o * 256 + j;
                    t.out = (int64_t(o) * 256 + j) * nb;
                    tk.push_back(t);
                }
            run_tasks(R, tk, nullptr, R.lap_log.p, s);
        }
        lap_table_kernel<<<148, 256, 0, s>>>(R.lap_log.p, R.p, h, table.p);
        VPG_LAUNCH_CHECK();
        return;
    }
    const int ob = R.origin_box(h);
    std::vector<RowTask> tk;
    for (int o = 0; o < 25; ++o)
        for (int j = 0; j < nb; ++j) {
            RowTask t{};
            t.job = kJobTableHelm;
            t.cell = ob;
            t.aux_i = o * 256 + j;
            t.out = (int64_t(o) * 256 + j) * nb;
            tk.push_back(t);
        }
    run_tasks(R, tk, nullptr, table.p, s);
}

extern "C" {

int vpg_rows_create(int family, double lambda, int p, int q, int64_t ncurve, const int32_t* curve_kind,
                    const double* curve_par, int64_t ncell, const int32_t* cell_type, const int32_t* cell_curve,
                    const double* cell_v, const double* cell_t, const double* cell_ch, const double* tri_nodes,
                    const double* tri_C, const double* box_C, int64_t ntri_src, const double* tri_src_xy,
                    const double* tri_src_w, int device, vpg_rows** out) {
    return guarded_r([&] {
        if (!out) throw Error{VPG_ERR_INVALID_ARGUMENT, "out is NULL"};
        *out = nullptr;
        if (family != VPG_LAPLACE && family != VPG_MODIFIED_HELMHOLTZ)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown kernel family"};
        if (family == VPG_MODIFIED_HELMHOLTZ && !(lambda > 0.0))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "make_kernel: modified Helmholtz needs lambda > 0"};
        if (p < 1 || p > kMaxP) throw Error{VPG_ERR_INVALID_ARGUMENT, "order p out of range [1, 12]"};
        if (q < 1 || q > 40) throw Error{VPG_ERR_INVALID_ARGUMENT, "source order q out of range [1, 40]"};
        if (ncell < 0 || ncurve < 0 || (ncell && (!cell_type || !cell_v || !cell_t || !cell_ch || !cell_curve)) ||
            (ncurve && (!curve_kind || !curve_par)) || !tri_nodes || !tri_C || !box_C || ntri_src < 1 ||
            !tri_src_xy || !tri_src_w)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad rows arrays"};
        use_device(device);
        auto R = std::make_unique<vpg_rows>();
        R->device = device;
        R->family = family;
        R->lambda = lambda;
        R->p = p;
        R->q = q;
        R->ncell = int(ncell);
        R->nb_tri = p * (p + 1) / 2;
        R->nb_box = p * p;
        for (int64_t k = 0; k < ncurve; ++k) {
            geom::Curve cu{};
            const double* a = curve_par + 6 * k;
            cu.kind = curve_kind[k];
            cu.cx = a[0];
            cu.cy = a[1];
            if (cu.kind == geom::kCircle) {
                cu.a = a[2];
            } else if (cu.kind == geom::kEllipse) {
                cu.a = a[2];
                cu.b = a[3];
                cu.cs = std::cos(a[4]);
                cu.sn = std::sin(a[4]);
            } else if (cu.kind == geom::kStar) {
                cu.a = a[2];
                cu.b = a[3];
                cu.arms = int(a[4]);
                cu.phase = a[5];
            } else {
                throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown curve kind"};
            }
            R->curves_h.push_back(cu);
        }
        for (int64_t k = 0; k < ncell; ++k) {
            geom::Cell c{};
            c.type = cell_type[k];
            if (c.type < 0 || c.type > 2) throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown cell type"};
            c.curve = cell_curve[k];
            if (c.type == geom::kCurvedTri && (c.curve < 0 || c.curve >= ncurve))
                throw Error{VPG_ERR_INVALID_ARGUMENT, "curved cell without a curve"};
            for (int v = 0; v < 3; ++v) c.v[v] = V2{cell_v[6 * k + 2 * v], cell_v[6 * k + 2 * v + 1]};
            c.ta = cell_t[2 * k];
            c.tb = cell_t[2 * k + 1];
            c.center = V2{cell_ch[3 * k], cell_ch[3 * k + 1]};
            c.h = cell_ch[3 * k + 2];
            R->cells_h.push_back(c);
        }
        geom::Cell rb{};
        rb.type = geom::kBox;
        rb.curve = -1;
        rb.center = V2{0, 0};
        rb.h = 2.0;  // the reference box [-1, 1]^2 (singular.cpp:37-50)
        R->cells_h.push_back(rb);
        // rules
        std::vector<Rule1> rules(kNumRules);
        rules[kGL16] = gauss_legendre(16);
        rules[kTLog20] = weighted_gauss(20, true);
        rules[kT20] = weighted_gauss(20, false);
        rules[kRaySing] = build_graded(3e-8, 0.25, 16);
        for (int qq = kNearQ0; qq <= kNearQ1; ++qq) rules[kNear0 + qq - kNearQ0] = ray_near_rule_bucket(qq);
        std::vector<double2> src;
        auto add_src = [&](int id, const std::vector<double2>& nodes, const std::vector<double>& w) {
            Rule1 r;
            for (size_t i = 0; i < nodes.size(); ++i) {
                r.x.push_back(double(src.size()));
                r.w.push_back(w[i]);
                src.push_back(nodes[i]);
            }
            rules[size_t(id)] = r;
        };
        auto box_rule = [&](int n, std::vector<double2>& nodes, std::vector<double>& w) {
            std::vector<double> z, wz;
            fejer1(n, z, wz);
            for (int ix = 0; ix < n; ++ix)
                for (int iy = 0; iy < n; ++iy) {  // basis.cpp:290-297
                    nodes.push_back(make_double2(z[size_t(ix)], z[size_t(iy)]));
                    w.push_back(wz[size_t(ix)] * wz[size_t(iy)]);
                }
        };
        {
            std::vector<double2> nd;
            std::vector<double> w;
            box_rule(q, nd, w);
            add_src(kBoxSrc, nd, w);
        }
        {
            std::vector<double2> nd;
            std::vector<double> w(tri_src_w, tri_src_w + ntri_src);
            for (int64_t i = 0; i < ntri_src; ++i) nd.push_back(make_double2(tri_src_xy[2 * i], tri_src_xy[2 * i + 1]));
            add_src(kTriSrc, nd, w);
        }
        {
            std::vector<double2> nd;
            std::vector<double> w;
            box_rule(30, nd, w);
            add_src(kBox30, nd, w);
        }
        R->rule_off_h.assign(1, 0);
        for (int r = 0; r < kNumRules; ++r) {
            for (size_t i = 0; i < rules[size_t(r)].x.size(); ++i)
                R->rule_xw_h.push_back(make_double2(rules[size_t(r)].x[i], rules[size_t(r)].w[i]));
            R->rule_off_h.push_back(int(R->rule_xw_h.size()));
        }
        // box interpolation nodes (basis.cpp:163-170): tensor Fejer nodes
        {
            std::vector<double> z, wz;
            fejer1(p, z, wz);
            for (int ix = 0; ix < p; ++ix)
                for (int iy = 0; iy < p; ++iy) {
                    R->box_nodes_h.push_back(z[size_t(ix)]);
                    R->box_nodes_h.push_back(z[size_t(iy)]);
                }
        }
        R->tri_nodes_h.assign(tri_nodes, tri_nodes + 2 * R->nb_tri);
        upload(R->curves, R->curves_h.data(), R->curves_h.size());
        upload(R->cells, R->cells_h.data(), R->cells_h.size());
        upload(R->rule_xw, R->rule_xw_h.data(), R->rule_xw_h.size());
        upload(R->rule_off, R->rule_off_h.data(), R->rule_off_h.size());
        upload(R->src_nodes, src.data(), src.size());
        upload(R->tri_C, tri_C, size_t(R->nb_tri) * R->nb_tri);
        upload(R->box_C, box_C, size_t(R->nb_box) * R->nb_box);
        upload(R->tri_nodes, R->tri_nodes_h.data(), R->tri_nodes_h.size());
        upload(R->box_nodes, R->box_nodes_h.data(), R->box_nodes_h.size());
        *out = R.release();
    });
}

int vpg_rows_destroy(vpg_rows* r) {
    return guarded_r([&] {
        if (!r) return;
        cudaSetDevice(r->device);
        delete r;
    });
}

// Host copy of one of the context's 1-D rules (tests): which = RuleId.
int vpg_rows_rule(const vpg_rows* r, int which, double* x, double* w, int64_t* n) {
    return guarded_r([&] {
        if (!r || !n || which < 0 || which >= kNumRules) throw Error{VPG_ERR_INVALID_ARGUMENT, "bad rule query"};
        const int a = r->rule_off_h[size_t(which)], b = r->rule_off_h[size_t(which) + 1];
        *n = b - a;
        for (int i = a; i < b; ++i) {
            if (x) x[i - a] = r->rule_xw_h[size_t(i)].x;
            if (w) w[i - a] = r->rule_xw_h[size_t(i)].y;
        }
    });
}

// Evaluates row tasks (host arrays): job, cell, aux_i, r0 (2), zeta0 (2),
// zstar (2) per task; rows written back to back (nb of the cell's kind).
int vpg_rows_eval(vpg_rows* r, int64_t ntask, const int32_t* job, const int32_t* cell, const int32_t* aux,
                  const double* r0, const double* zeta0, const double* zstar, double lattice_h, double* out,
                  int64_t* out_len) {
    return guarded_r([&] {
        if (!r || ntask < 0 || (ntask && (!job || !cell))) throw Error{VPG_ERR_INVALID_ARGUMENT, "bad tasks"};
        std::lock_guard<std::mutex> lk(r->mu);
        VPG_CUDA(cudaSetDevice(r->device));
        std::vector<RowTask> tk(static_cast<size_t>(ntask));
        int64_t at = 0;
        bool need_table = false;
        for (int64_t i = 0; i < ntask; ++i) {
            RowTask& t = tk[size_t(i)];
            t.job = job[i];
            t.cell = cell[i] < 0 ? r->ref_box() : cell[i];
            if (t.cell < 0 || t.cell >= int(r->cells_h.size())) throw Error{VPG_ERR_INVALID_ARGUMENT, "cell out of range"};
            t.aux_i = aux ? aux[i] : 0;
            if (t.job == kJobSmooth) t.aux_i = t.aux_i == 30 ? kBox30 : (r->cells_h[size_t(t.cell)].type == geom::kBox ? kBoxSrc : kTriSrc);
            t.r0 = r0 ? make_double2(r0[2 * i], r0[2 * i + 1]) : make_double2(0, 0);
            t.zeta0 = zeta0 ? make_double2(zeta0[2 * i], zeta0[2 * i + 1]) : make_double2(0, 0);
            t.zstar = zstar ? make_double2(zstar[2 * i], zstar[2 * i + 1]) : make_double2(0, 0);
            if (t.job == kJobTableHelm) t.cell = r->origin_box(lattice_h);
            if (t.job == kJobLattice) {
                need_table = true;
                t.cell = r->origin_box(lattice_h);
            }
            t.out = at;
            at += r->cells_h[size_t(t.cell)].type == geom::kBox ? r->nb_box : r->nb_tri;
        }
        if (out_len) *out_len = at;
        if (!out) return;
        cudaStream_t s = nullptr;
        VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamDefault));
        struct SD {
            cudaStream_t s;
            ~SD() { cudaStreamDestroy(s); }
        } sd{s};
        DBuf<double> table, od;
        if (need_table) lattice_table(*r, lattice_h, table, s);
        od.alloc(size_t(std::max<int64_t>(at, 1)));
        run_tasks(*r, tk, table.p, od.p, s);
        VPG_CUDA(cudaMemcpy(out, od.p, size_t(at) * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"

// ------------------------------------------------------------------------
// The whole correction map on the device side: classify_target for every
// target (mesh.cpp:410-448, one thread per target over the cell locator of
// mesh.cpp:171-199), the task list and pool slots of build_corrections
// (potential.cpp:153-240, host: a hash lookup of node-coincident targets and
// the lattice-slot assignment), then the rows above.
// ------------------------------------------------------------------------
namespace vpg {
namespace rows {

constexpr int kMaxNear = 30;

// out: self cell, near count (or -1: no self cell, -2: > 30 near cells) and
// the near cells in locator (ascending cell) order
__global__ void classify_kernel(const geom::Cell* cells, const geom::Curve* curves, const double4* bbox,
                                const int* loc_off, const int* loc_cells, double lox, double loy, double bucket,
                                int nx, int ny, double reach, double inside_tol, const double2* tgt, int64_t nt,
                                int* self_out, int* nnear_out, int* near_out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const V2 r0{tgt[t].x, tgt[t].y};
    const int ix = int(floor((r0.x - lox) / bucket));
    const int iy = int(floor((r0.y - loy) / bucket));
    int self = -1, nn = 0;
    if (ix < 0 || iy < 0 || ix >= nx || iy >= ny) {
        self_out[t] = -3;  // outside the mesh
        nnear_out[t] = 0;
        return;
    }
    const int b = ix + nx * iy;
    const double slack = reach + inside_tol;
    for (int e = loc_off[b]; e < loc_off[b + 1]; ++e) {
        const int k = loc_cells[e];
        const double4 bb = bbox[k];
        if (r0.x < bb.x - slack || r0.x > bb.z + slack || r0.y < bb.y - slack || r0.y > bb.w + slack) continue;
        double d = 0;
        geom::nearest_reference_point(cells[k], curves, r0, &d);
        if (self < 0 && d <= inside_tol) {
            self = k;
            continue;
        }
        if (d < reach) {
            if (nn < kMaxNear) near_out[t * kMaxNear + nn] = k;
            ++nn;
        }
    }
    self_out[t] = self;
    nnear_out[t] = nn;
}

}  // namespace rows
}  // namespace vpg

extern "C" int vpg_corr_build(vpg_rows* r, int64_t ndofs, const double* nodes_xy, const int32_t* node_off,
                              int64_t nt, const double* tgt_xy, double D, vpg_corr** out, double* stats) {
    return guarded_r([&] {
        if (!r || !out || ndofs < 0 || nt < 0 || (ndofs && !nodes_xy) || !node_off || (nt && !tgt_xy))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad correction-build arguments"};
        if (!(D > 0)) throw Error{VPG_ERR_INVALID_ARGUMENT, "classify_target: D must be positive"};
        *out = nullptr;
        std::lock_guard<std::mutex> lk(r->mu);
        VPG_CUDA(cudaSetDevice(r->device));
        const int ncell = r->ncell;
        const auto& cells = r->cells_h;
        const auto* curves = r->curves_h.data();
        if (ncell == 0) throw Error{VPG_ERR_INVALID_ARGUMENT, "classify_target: mesh is empty"};
        if (node_off[ncell] != ndofs) throw Error{VPG_ERR_INVALID_ARGUMENT, "node_off does not end at ndofs"};
        double h = cells[0].h;  // HybridMesh::h: every cell carries the mesh size (mesh.cpp:387-401)
        for (int k = 0; k < ncell; ++k)
            if (cells[size_t(k)].type == geom::kBox) {
                h = cells[size_t(k)].h;
                break;
            }
        const auto t_begin = std::chrono::steady_clock::now();
        cudaStream_t s = nullptr;
        VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamDefault));
        struct SD {
            cudaStream_t s;
            ~SD() { cudaStreamDestroy(s); }
        } sd{s};
        // locator (mesh.cpp:171-199): bucket = h, pad = h/2
        std::vector<double4> bb(static_cast<size_t>(ncell));
        V2 lo{HUGE_VAL, HUGE_VAL}, hi{-HUGE_VAL, -HUGE_VAL};
        for (int k = 0; k < ncell; ++k) {
            V2 a, b;
            geom::bounding_box(cells[size_t(k)], curves, a, b);
            bb[size_t(k)] = make_double4(a.x, a.y, b.x, b.y);
            lo.x = std::min(lo.x, a.x);
            lo.y = std::min(lo.y, a.y);
            hi.x = std::max(hi.x, b.x);
            hi.y = std::max(hi.y, b.y);
        }
        const double bucket = h, pad = 0.5 * h;
        const V2 llo{lo.x - pad, lo.y - pad};
        const int nx = int(std::ceil((hi.x + pad - llo.x) / bucket)) + 1;
        const int ny = int(std::ceil((hi.y + pad - llo.y) / bucket)) + 1;
        const double reach = D * h;
        if (!(reach <= pad)) throw Error{VPG_ERR_INVALID_ARGUMENT, "classify_target: D * h exceeds the locator pad"};
        std::vector<std::vector<int>> lists(static_cast<size_t>(nx) * static_cast<size_t>(ny));
        for (int k = 0; k < ncell; ++k) {
            const double4 q = bb[size_t(k)];
            auto cl = [](int v, int n) { return std::min(std::max(v, 0), n - 1); };
            const int x0 = cl(int(std::floor((q.x - pad - llo.x) / bucket)), nx);
            const int x1 = cl(int(std::floor((q.z + pad - llo.x) / bucket)), nx);
            const int y0 = cl(int(std::floor((q.y - pad - llo.y) / bucket)), ny);
            const int y1 = cl(int(std::floor((q.w + pad - llo.y) / bucket)), ny);
            for (int iy = y0; iy <= y1; ++iy)
                for (int ix = x0; ix <= x1; ++ix) lists[size_t(ix) + size_t(nx) * iy].push_back(k);
        }
        std::vector<int> loc_off(1, 0), loc_cells;
        for (const auto& l : lists) {
            loc_cells.insert(loc_cells.end(), l.begin(), l.end());
            loc_off.push_back(int(loc_cells.size()));
        }
        DBuf<double4> bbd;
        DBuf<int> lo_d, lc_d, self_d, nn_d, near_d;
        DBuf<double2> tg_d;
        upload(bbd, bb.data(), bb.size());
        upload(lo_d, loc_off.data(), loc_off.size());
        upload(lc_d, loc_cells.data(), loc_cells.size());
        upload(tg_d, reinterpret_cast<const double2*>(tgt_xy), size_t(nt));
        self_d.alloc(size_t(std::max<int64_t>(nt, 1)));
        nn_d.alloc(size_t(std::max<int64_t>(nt, 1)));
        near_d.alloc(size_t(std::max<int64_t>(nt, 1)) * kMaxNear);
        if (nt)
            classify_kernel<<<unsigned((nt + 127) / 128), 128, 0, s>>>(
                r->cells.p, r->curves.p, bbd.p, lo_d.p, lc_d.p, llo.x, llo.y, bucket, nx, ny, reach, 1e-9 * h, tg_d.p,
                nt, self_d.p, nn_d.p, near_d.p);
        VPG_LAUNCH_CHECK();
        std::vector<int> self(static_cast<size_t>(nt)), nnear(static_cast<size_t>(nt)), nearc(static_cast<size_t>(nt) * kMaxNear);
        if (nt) {
            VPG_CUDA(cudaMemcpyAsync(self.data(), self_d.p, size_t(nt) * 4, cudaMemcpyDeviceToHost, s));
            VPG_CUDA(cudaMemcpyAsync(nnear.data(), nn_d.p, size_t(nt) * 4, cudaMemcpyDeviceToHost, s));
            VPG_CUDA(cudaMemcpyAsync(nearc.data(), near_d.p, size_t(nt) * kMaxNear * 4, cudaMemcpyDeviceToHost, s));
            VPG_CUDA(cudaStreamSynchronize(s));
        }
        const auto t_cls = std::chrono::steady_clock::now();
        for (int64_t t = 0; t < nt; ++t) {
            auto where = [&] {
                char buf[160];
                std::snprintf(buf, sizeof buf, "target %lld at (%f, %f): ", (long long)t, tgt_xy[2 * t],
                              tgt_xy[2 * t + 1]);
                return std::string(buf);
            };
            if (self[size_t(t)] == -3)
                throw Error{VPG_ERR_INVALID_ARGUMENT, where() + "classify_target: point is outside the mesh"};
            if (self[size_t(t)] < 0)
                throw Error{VPG_ERR_INVALID_ARGUMENT, where() + "classify_target: point is not inside any cell"};
            if (nnear[size_t(t)] > kMaxNear)
                throw Error{VPG_ERR_INVALID_ARGUMENT, where() + "classify_target: near set exceeds 30 cells"};
        }
        // node lookup by exact bits (potential.cpp:140-152)
        struct KeyHash {
            size_t operator()(const std::pair<uint64_t, uint64_t>& k) const {
                uint64_t hh = k.first + 0x9e3779b97f4a7c15ull;
                hh = (hh ^ (hh >> 30)) * 0xbf58476d1ce4e5b9ull;
                hh ^= k.second + 0x9e3779b97f4a7c15ull;
                hh = (hh ^ (hh >> 27)) * 0x94d049bb133111ebull;
                return size_t(hh ^ (hh >> 31));
            }
        };
        auto bits = [](double v) {
            uint64_t u;
            std::memcpy(&u, &v, 8);
            return u;
        };
        std::unordered_map<std::pair<uint64_t, uint64_t>, int, KeyHash> node_of;
        node_of.reserve(size_t(ndofs) * 2);
        for (int64_t i = 0; i < ndofs; ++i)
            node_of.emplace(std::make_pair(bits(nodes_xy[2 * i]), bits(nodes_xy[2 * i + 1])), int(i));
        std::vector<int> node_cell(static_cast<size_t>(ndofs));
        for (int c = 0; c < ncell; ++c)
            for (int i = node_off[c]; i < node_off[c + 1]; ++i) node_cell[size_t(i)] = c;
        auto lattice_offset = [&](const geom::Cell& tc, const geom::Cell& sc) -> int {  // potential.cpp:196-205
            if (tc.h != h || sc.h != h) return -1;
            const double fx = (tc.center.x - sc.center.x) / h;
            const double fy = (tc.center.y - sc.center.y) / h;
            const double rx = std::round(fx), ry = std::round(fy);
            if (std::abs(fx - rx) > 1e-9 || std::abs(fy - ry) > 1e-9) return -1;
            if (std::abs(rx) > 2 || std::abs(ry) > 2) return -1;
            return (int(ry) + 2) * 5 + (int(rx) + 2);
        };
        // tasks (potential.cpp:207-240)
        struct HT {
            int job, cell, local, off;
        };
        std::vector<HT> tasks;
        tasks.reserve(size_t(nt) * 4);
        std::vector<int32_t> blk_off(static_cast<size_t>(nt) + 1, 0);
        int64_t njob[10] = {0};
        for (int64_t t = 0; t < nt; ++t) {
            auto it = node_of.find(std::make_pair(bits(tgt_xy[2 * t]), bits(tgt_xy[2 * t + 1])));
            const int nid = it == node_of.end() ? -1 : it->second;
            const int hc = nid >= 0 ? node_cell[size_t(nid)] : -1;
            const geom::Cell* home = nid >= 0 ? &cells[size_t(hc)] : nullptr;
            const int local = nid >= 0 ? nid - node_off[hc] : -1;
            auto add = [&](int cid, bool is_self) {
                const geom::Cell& cell = cells[size_t(cid)];
                HT task{0, cid, -1, -1};
                if (cell.type == geom::kBox) {
                    const int off = home && home->type == geom::kBox && hc == (is_self ? cid : hc)
                                        ? lattice_offset(*home, cell) : -1;
                    if (off >= 0) {
                        task.job = kJobLattice;
                        task.local = local;
                        task.off = off;
                    } else {
                        task.job = is_self ? kJobSelfGeneric : kJobNearGeneric;
                    }
                } else if (is_self) {
                    if (nid >= 0 && hc == cid) {
                        task.job = kJobTriSelfNode;
                        task.local = local;
                    } else {
                        task.job = kJobSelfGeneric;
                    }
                } else {
                    task.job = kJobTriNearSnap;
                }
                ++njob[task.job];
                tasks.push_back(task);
            };
            add(self[size_t(t)], true);
            for (int k = 0; k < nnear[size_t(t)]; ++k) add(nearc[size_t(t) * kMaxNear + k], false);
            blk_off[size_t(t) + 1] = int32_t(tasks.size());
        }
        // pool slots (potential.cpp:242-254) and the device row tasks
        std::unordered_map<int, int> lattice_slot;
        std::vector<int32_t> blk_cell(tasks.size()), blk_pool(tasks.size());
        std::vector<int64_t> pool_off(1, 0);
        std::vector<RowTask> rt;
        rt.reserve(tasks.size());
        for (size_t i = 0; i < tasks.size(); ++i) {
            const HT& task = tasks[i];
            blk_cell[i] = task.cell;
            const int nbk = cells[size_t(task.cell)].type == geom::kBox ? r->nb_box : r->nb_tri;
            int slot;
            bool fresh = true;
            if (task.job == kJobLattice) {
                auto ins = lattice_slot.emplace(task.off * 256 + task.local, int(pool_off.size() - 1));
                slot = ins.first->second;
                fresh = ins.second;
            } else {
                slot = int(pool_off.size() - 1);
            }
            blk_pool[i] = slot;
            if (!fresh) continue;
            pool_off.push_back(pool_off.back() + nbk);
            RowTask t{};
            t.job = task.job;
            t.cell = task.cell;
            t.out = pool_off[size_t(slot)];
            if (task.job == kJobLattice) {
                const int ox = task.off % 5 - 2, oy = task.off / 5 - 2, j = task.local;
                t.cell = r->origin_box(h);
                t.aux_i = task.off * 256 + j;
                t.r0 = make_double2(ox * h + 0.5 * h * r->box_nodes_h[size_t(2 * j)],
                                    oy * h + 0.5 * h * r->box_nodes_h[size_t(2 * j + 1)]);
            } else {
                const int64_t tg = std::upper_bound(blk_off.begin(), blk_off.end(), int32_t(i)) - blk_off.begin() - 1;
                t.aux_i = task.local;
                t.r0 = make_double2(tgt_xy[2 * tg], tgt_xy[2 * tg + 1]);
            }
            rt.push_back(t);
        }
        const int64_t npool = int64_t(pool_off.size()) - 1;
        DBuf<double> table, pool;
        if (!lattice_slot.empty()) lattice_table(*r, h, table, s);
        pool.alloc(size_t(std::max<int64_t>(pool_off.back(), 1)));
        const auto t_tasks = std::chrono::steady_clock::now();
        // heavy rows first (self / near ray rules), cheap lattice rows last
        std::stable_sort(rt.begin(), rt.end(), [](const RowTask& a, const RowTask& b) {
            return (a.job == kJobLattice) < (b.job == kJobLattice);
        });
        int64_t nodes[2] = {0, 0};
        run_tasks(*r, rt, table.p, pool.p, s, nodes);
        const auto t_rows = std::chrono::steady_clock::now();
        vpg::corr_create_impl(nt, blk_off.data(), int64_t(tasks.size()), blk_cell.data(), blk_pool.data(), npool,
                              pool_off.data(), pool.p, true, ncell, node_off, r->device, out);
        if (stats) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            stats[0] = ms(t_begin, t_cls);     // locator + classification (device) + download
            stats[1] = ms(t_cls, t_tasks);     // tasks, pool slots (host), lattice table (device)
            stats[2] = ms(t_tasks, t_rows);    // row kernels
            stats[3] = double(tasks.size());   // blocks
            stats[4] = double(npool);          // pool rows
            stats[5] = double(pool_off.back());
            for (int j = 3; j <= 7; ++j) stats[3 + j] = double(njob[j]);  // stats[6..10]: job counts 3..7
            stats[11] = double(nodes[0]);       // quadrature nodes evaluated on triangle cells
            stats[12] = double(nodes[1]);       // ... on box cells
        }
    });
}

// mesh_nodes (potential.cpp:63-74, which = 0: the order-p interpolation nodes
// of every cell, xy only) and build_sources (potential.cpp:133-151, which = 1:
// the order-q source rule mapped, xy and w * jacobian) on the host, from the
// context's cells and tables; *n = point count (xy / wj may be NULL to size).
extern "C" int vpg_rows_map(const vpg_rows* r, int which, double* xy, double* wj, int64_t* n) {
    return guarded_r([&] {
        if (!r || !n || (which != 0 && which != 1)) throw Error{VPG_ERR_INVALID_ARGUMENT, "bad map query"};
        const int box_rule = which == 0 ? -1 : kBoxSrc, tri_rule = which == 0 ? -1 : kTriSrc;
        std::vector<double2> src_nodes;  // host copy of the source nodes (rule x = node index)
        int64_t cnt = 0;
        for (int c = 0; c < r->ncell; ++c) {
            const bool box = r->cells_h[size_t(c)].type == geom::kBox;
            if (which == 0)
                cnt += box ? r->nb_box : r->nb_tri;
            else
                cnt += r->rule_off_h[size_t(box ? box_rule : tri_rule) + 1] - r->rule_off_h[size_t(box ? box_rule : tri_rule)];
        }
        *n = cnt;
        if (!xy && !wj) return;
        std::vector<double2> sn;
        if (which == 1) {
            sn.resize(r->src_nodes.n);
            VPG_CUDA(cudaMemcpy(sn.data(), r->src_nodes.p, r->src_nodes.bytes(), cudaMemcpyDeviceToHost));
        }
        int64_t at = 0;
        for (int c = 0; c < r->ncell; ++c) {
            const geom::Cell& cell = r->cells_h[size_t(c)];
            const bool box = cell.type == geom::kBox;
            if (which == 0) {
                const int nb = box ? r->nb_box : r->nb_tri;
                const double* nd = box ? r->box_nodes_h.data() : r->tri_nodes_h.data();
                for (int i = 0; i < nb; ++i, ++at) {
                    const V2 x = geom::cell_map(cell, r->curves_h.data(), V2{nd[2 * i], nd[2 * i + 1]});
                    if (xy) {
                        xy[2 * at] = x.x;
                        xy[2 * at + 1] = x.y;
                    }
                }
            } else {
                const int rid = box ? box_rule : tri_rule;
                for (int e = r->rule_off_h[size_t(rid)]; e < r->rule_off_h[size_t(rid) + 1]; ++e, ++at) {
                    const double2 zw = r->rule_xw_h[size_t(e)];
                    const double2 z = sn[size_t(zw.x)];
                    V2 x, a, b;
                    double jac;
                    geom::map_deriv(cell, r->curves_h.data(), V2{z.x, z.y}, x, a, b, jac);
                    if (xy) {
                        xy[2 * at] = x.x;
                        xy[2 * at + 1] = x.y;
                    }
                    if (wj) wj[at] = zw.y * jac;
                }
            }
        }
    });
}
