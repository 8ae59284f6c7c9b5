// geom.cuh -- host/device restatement of the reference cell geometry and the
// reference-cell boundary layouts the correction rows integrate over:
//   curves (geometry.cpp:63-132: Circle, Ellipse, StarCurve),
//   Cell::map_deriv / invert / bounding_box (geometry.cpp:160-303),
//   nearest_reference_point (geometry.cpp:305-380),
//   ref_cell_corner / ref_boundary_point / nearest_boundary_param /
//   boundary_discretization (singular.cpp:57-190),
//   chebyshev2d_eval / koornwinder_eval (basis.cpp:24-45, 131-140, 193-228).
// Everything is __host__ __device__ so the plan-time host code (target
// classification, task building) and the row kernels share one statement.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace vpg {
namespace geom {

#define VPG_HD __host__ __device__ __forceinline__

struct V2 {
    double x, y;
};
VPG_HD V2 mk(double x, double y) { return V2{x, y}; }
VPG_HD V2 operator+(V2 a, V2 b) { return V2{a.x + b.x, a.y + b.y}; }
VPG_HD V2 operator-(V2 a, V2 b) { return V2{a.x - b.x, a.y - b.y}; }
VPG_HD V2 operator*(double s, V2 v) { return V2{v.x * s, v.y * s}; }  // Vec2 operator*(s, v) = v * s
VPG_HD double dot(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }
VPG_HD double cross(V2 a, V2 b) { return a.x * b.y - a.y * b.x; }
VPG_HD double norm2(V2 a) { return a.x * a.x + a.y * a.y; }
VPG_HD double norm(V2 a) { return sqrt(norm2(a)); }
VPG_HD double dist(V2 a, V2 b) { return norm(a - b); }

// ------------------------------------------------------------------ curves --
enum CurveKind : int32_t { kCircle = 0, kEllipse = 1, kStar = 2 };
struct Curve {
    int32_t kind;
    int32_t arms;      // star
    double cx, cy;
    double a, b;       // circle: a = radius; ellipse: semiaxes; star: a = r0, b = amp
    double cs, sn;     // ellipse rotation (cos, sin of the angle)
    double phase;      // star
};

// order 0: pos, 1: deriv, 2: deriv2, 3: deriv3
VPG_HD V2 curve_eval(const Curve& c, double t, int order) {
    const double ct = cos(t), st = sin(t);
    if (c.kind == kCircle) {
        const double r = c.a;
        switch (order) {
            case 0: return V2{c.cx, c.cy} + r * V2{ct, st};
            case 1: return r * V2{-st, ct};
            case 2: return r * V2{-ct, -st};
            default: return r * V2{st, -ct};
        }
    }
    if (c.kind == kEllipse) {
        double u, v;
        switch (order) {
            case 0: u = c.a * ct; v = c.b * st; break;
            case 1: u = -c.a * st; v = c.b * ct; break;
            case 2: u = -c.a * ct; v = -c.b * st; break;
            default: u = c.a * st; v = -c.b * ct; break;
        }
        const V2 w{c.cs * u - c.sn * v, c.sn * u + c.cs * v};
        return order == 0 ? V2{c.cx, c.cy} + w : w;
    }
    // StarCurve (geometry.cpp:106-132)
    const double k = c.arms;
    const double r0 = c.a, amp = c.b;
    const double ck = cos(k * t + c.phase), sk = sin(k * t + c.phase);
    const double rho = r0 * (1 + amp * ck);
    const V2 u{ct, st}, up{-st, ct};
    if (order == 0) return V2{c.cx, c.cy} + rho * u;
    const double drho = -r0 * amp * k * sk;
    if (order == 1) return drho * u + rho * up;
    const double d2rho = -r0 * amp * k * k * ck;
    if (order == 2) return (d2rho - rho) * u + (2 * drho) * up;
    const double d3rho = r0 * amp * k * k * k * sk;
    return (d3rho - 3 * drho) * u + (3 * d2rho - rho) * up;
}

// pos and deriv at one t together (one sincos per angle; blend_terms needs both)
VPG_HD void curve_pos_deriv(const Curve& c, double t, V2& pos, V2& der) {
    double st, ct;
    sincos(t, &st, &ct);
    if (c.kind == kCircle) {
        pos = V2{c.cx, c.cy} + c.a * V2{ct, st};
        der = c.a * V2{-st, ct};
        return;
    }
    if (c.kind == kEllipse) {
        const double u0 = c.a * ct, v0 = c.b * st, u1 = -c.a * st, v1 = c.b * ct;
        pos = V2{c.cx, c.cy} + V2{c.cs * u0 - c.sn * v0, c.sn * u0 + c.cs * v0};
        der = V2{c.cs * u1 - c.sn * v1, c.sn * u1 + c.cs * v1};
        return;
    }
    const double k = c.arms;
    const double r0 = c.a, amp = c.b;
    double sk, ck;
    sincos(k * t + c.phase, &sk, &ck);
    const double rho = r0 * (1 + amp * ck);
    const V2 u{ct, st}, up{-st, ct};
    pos = V2{c.cx, c.cy} + rho * u;
    const double drho = -r0 * amp * k * sk;
    der = drho * u + rho * up;
}

// ------------------------------------------------------------------- cells --
enum CellType : int32_t { kStraightTri = 0, kCurvedTri = 1, kBox = 2 };
struct Cell {
    int32_t type;
    int32_t curve;  // index into the curve table (curved triangles), else -1
    V2 v[3];
    double ta, tb;
    V2 center;
    double h;
};

// geometry.cpp:166-185 (kBlendTaylorCut = 1e-5)
VPG_HD void blend_terms(const Cell& c, const Curve* curves, double xi, V2& phi, V2& dphi) {
    const Curve& cu = curves[c.curve];
    const double dt = c.tb - c.ta;
    const double s = 1 - xi;
    const V2 base = c.v[1] - c.v[0];
    if (s >= 1e-5) {
        const double t = c.ta + xi * dt;
        V2 lam, der;
        curve_pos_deriv(cu, t, lam, der);
        const V2 dlam = dt * der;
        const V2 num = lam - (1 - xi) * c.v[0] - xi * c.v[1];
        phi = (1.0 / s) * num;
        dphi = (1.0 / s) * (dlam - base + phi);
    } else {
        const V2 d1 = dt * curve_eval(cu, c.tb, 1);
        const V2 d2 = (dt * dt) * curve_eval(cu, c.tb, 2);
        const V2 d3 = (dt * dt * dt) * curve_eval(cu, c.tb, 3);
        phi = -1.0 * (d1 - base) + (s / 2) * d2 - (s * s / 6) * d3;
        dphi = -0.5 * d2 + (s / 3) * d3;
    }
}

// Cell::map_deriv (geometry.cpp:198-223)
VPG_HD void map_deriv(const Cell& c, const Curve* curves, V2 z, V2& x, V2& dxi, V2& deta, double& jac) {
    if (c.type == kBox) {
        x = c.center + (c.h / 2) * z;
        dxi = V2{c.h / 2, 0};
        deta = V2{0, c.h / 2};
        jac = c.h * c.h / 4;
        return;
    }
    if (c.type == kStraightTri) {
        dxi = c.v[1] - c.v[0];
        deta = c.v[2] - c.v[0];
        x = c.v[0] + z.x * dxi + z.y * deta;
        jac = cross(dxi, deta);
        return;
    }
    V2 phi, dphi;
    blend_terms(c, curves, z.x, phi, dphi);
    const double blend = 1 - z.x - z.y;
    dxi = (c.v[1] - c.v[0]) - phi + blend * dphi;
    deta = (c.v[2] - c.v[0]) - phi;
    x = c.v[0] + z.x * (c.v[1] - c.v[0]) + z.y * (c.v[2] - c.v[0]) + blend * phi;
    jac = cross(dxi, deta);
}

VPG_HD V2 cell_map(const Cell& c, const Curve* curves, V2 z) {
    V2 x, a, b;
    double j;
    map_deriv(c, curves, z, x, a, b, j);
    return x;
}

// Cell::invert (geometry.cpp:232-256)
VPG_HD V2 invert(const Cell& c, const Curve* curves, V2 x) {
    if (c.type == kBox) return (2 / c.h) * (x - c.center);
    const V2 e1 = c.v[1] - c.v[0], e2 = c.v[2] - c.v[0];
    const double det = cross(e1, e2);
    const V2 r0 = x - c.v[0];
    V2 zeta{(r0.x * e2.y - r0.y * e2.x) / det, (e1.x * r0.y - e1.y * r0.x) / det};
    if (c.type == kStraightTri) return zeta;
    const double scale = norm(e1) + norm(e2);
    for (int it = 0; it < 40; ++it) {
        V2 X, dxi, deta;
        double jac;
        map_deriv(c, curves, zeta, X, dxi, deta, jac);
        const V2 r = x - X;
        if (norm(r) <= 1e-15 * scale) break;
        const V2 step{(r.x * deta.y - r.y * deta.x) / jac, (dxi.x * r.y - dxi.y * r.x) / jac};
        zeta = zeta + step;
        if (fabs(zeta.x) > 20 || fabs(zeta.y) > 20) break;
    }
    return zeta;
}

VPG_HD bool ref_contains(const Cell& c, V2 z, double pad) {
    if (c.type == kBox) return fabs(z.x) <= 1 + pad && fabs(z.y) <= 1 + pad;
    return z.x >= -pad && z.y >= -pad && z.x + z.y <= 1 + pad;
}

VPG_HD int num_corners(const Cell& c) { return c.type == kBox ? 4 : 3; }

VPG_HD V2 cell_ref_corner(const Cell& c, int i) {
    if (c.type == kBox) {
        const int k = i & 3;
        return V2{(k == 1 || k == 2) ? 1.0 : -1.0, k >= 2 ? 1.0 : -1.0};
    }
    const int k = i % 3;
    return V2{k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
}

// Cell::bounding_box over Cell::outline (geometry.cpp:283-318)
VPG_HD void bounding_box(const Cell& c, const Curve* curves, V2& lo, V2& hi) {
    lo = V2{1e300, 1e300};
    hi = V2{-1e300, -1e300};
    const int per_edge = c.type == kCurvedTri ? 32 : 2;
    const int nc = num_corners(c);
    for (int e = 0; e < nc; ++e) {
        const V2 a = cell_ref_corner(c, e), b = cell_ref_corner(c, (e + 1) % nc);
        for (int j = 0; j < per_edge; ++j) {
            const double s = static_cast<double>(j) / per_edge;
            const V2 p = cell_map(c, curves, a + s * (b - a));
            lo.x = fmin(lo.x, p.x);
            lo.y = fmin(lo.y, p.y);
            hi.x = fmax(hi.x, p.x);
            hi.y = fmax(hi.y, p.y);
        }
    }
}

VPG_HD double cell_diameter(const Cell& c, const Curve* curves) {
    V2 lo, hi;
    bounding_box(c, curves, lo, hi);
    return norm(hi - lo);
}

VPG_HD double edge_dist2(const Cell& c, const Curve* curves, V2 a, V2 b, double s, V2 x) {
    return norm2(cell_map(c, curves, a + s * (b - a)) - x);
}

// nearest_reference_point (geometry.cpp:326-380)
VPG_HD V2 nearest_reference_point(const Cell& c, const Curve* curves, V2 x, double* distance) {
    V2 zeta = invert(c, curves, x);
    if (ref_contains(c, zeta, 1e-10)) {
        const V2 p = cell_map(c, curves, zeta);
        if (distance) *distance = dist(p, x);
        if (dist(p, x) < 1e-9 * (1 + fabs(x.x) + fabs(x.y))) return zeta;
    }
    const int nc = num_corners(c);
    double best = 1e300;
    V2 best_zeta{0, 0};
    const double gr = (sqrt(5.0) - 1) / 2;
    for (int e = 0; e < nc; ++e) {
        const V2 a = cell_ref_corner(c, e), b = cell_ref_corner(c, (e + 1) % nc);
        const int ns = 32;
        int imin = 0;
        double dmin = 1e300;
        for (int i = 0; i <= ns; ++i) {
            const double d2 = edge_dist2(c, curves, a, b, static_cast<double>(i) / ns, x);
            if (d2 < dmin) {
                dmin = d2;
                imin = i;
            }
        }
        double lo = fmax(0.0, (imin - 1.0) / ns);
        double hi = fmin(1.0, (imin + 1.0) / ns);
        double c1 = hi - gr * (hi - lo), c2 = lo + gr * (hi - lo);
        double f1 = edge_dist2(c, curves, a, b, c1, x), f2 = edge_dist2(c, curves, a, b, c2, x);
        for (int it = 0; it < 80 && hi - lo > 1e-13; ++it) {
            if (f1 < f2) {
                hi = c2;
                c2 = c1;
                f2 = f1;
                c1 = hi - gr * (hi - lo);
                f1 = edge_dist2(c, curves, a, b, c1, x);
            } else {
                lo = c1;
                c1 = c2;
                f1 = f2;
                c2 = lo + gr * (hi - lo);
                f2 = edge_dist2(c, curves, a, b, c2, x);
            }
        }
        const double s = 0.5 * (lo + hi);
        const double d2 = edge_dist2(c, curves, a, b, s, x);
        if (d2 < best) {
            best = d2;
            best_zeta = a + s * (b - a);
        }
    }
    if (distance) *distance = sqrt(best);
    return best_zeta;
}

// ------------------------------------------------- reference-cell boundary --
// kind: 0 simplex (3 edges), 1 box [-1,1]^2 (4 edges)  (singular.cpp:57-75)
VPG_HD int ref_edges(int box) { return box ? 4 : 3; }
VPG_HD V2 ref_corner(int box, int i) {
    if (!box) {
        const int k = ((i % 3) + 3) % 3;
        return V2{k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    }
    const int k = ((i % 4) + 4) % 4;
    return V2{(k == 1 || k == 2) ? 1.0 : -1.0, k >= 2 ? 1.0 : -1.0};
}

// singular.cpp:22-33
VPG_HD double wrap_param(double t, int nc) {
    double r = fmod(t, static_cast<double>(nc));
    if (r < 0) r += nc;
    if (r >= nc) r = 0;
    return r;
}
VPG_HD double cyclic_dist(double a, double b, int nc) {
    const double d = fabs(a - b);
    return fmin(d, nc - d);
}

// singular.cpp:77-85
VPG_HD V2 ref_boundary_point(int box, double t) {
    const int nc = ref_edges(box);
    t = wrap_param(t, nc);
    const int e = min(nc - 1, static_cast<int>(floor(t)));
    const double s = t - e;
    const V2 a = ref_corner(box, e), b = ref_corner(box, e + 1);
    return a + s * (b - a);
}

// singular.cpp:87-104
VPG_HD double nearest_boundary_param(int box, V2 z) {
    const int nc = ref_edges(box);
    double best_t = 0, best_d = HUGE_VAL;
    for (int e = 0; e < nc; ++e) {
        const V2 a = ref_corner(box, e);
        const V2 ab = ref_corner(box, e + 1) - a;
        const double s = fmin(fmax(dot(z - a, ab) / norm2(ab), 0.0), 1.0);
        const double d = norm(z - (a + s * ab));
        if (d < best_d) {
            best_d = d;
            best_t = e + s;
        }
    }
    return wrap_param(best_t, nc);
}

// Panel endpoints of boundary_discretization (singular.cpp:106-161): returns
// the count (<= kMaxEndpoints) written to ep[], ascending on [0, nc).
constexpr int kMaxEndpoints = 4 * 4 + 1 + 10 + 4 * 10;
VPG_HD int boundary_endpoints(int box, V2 zs, double* ep) {
    const int nc = ref_edges(box);
    const double tol = 1e-9;
    const double t1 = nearest_boundary_param(box, zs);
    double pts[kMaxEndpoints];
    int n = 0;
    for (int e = 0; e < nc; ++e)
        for (int j = 0; j < 4; ++j) pts[n++] = e + 0.25 * j;
    const double grid = round(t1 * 4.0) * 0.25;
    const bool on_grid = cyclic_dist(t1, wrap_param(grid, nc), nc) <= tol;
    if (!on_grid) pts[n++] = t1;
    double step = on_grid ? 0.5 : 0.25;
    for (int j = 1; j <= 5; ++j) {
        step *= 0.25;
        pts[n++] = wrap_param(t1 + step, nc);
        pts[n++] = wrap_param(t1 - step, nc);
    }
    const double reach = box ? 1.0 : 0.5;
    for (int c = 0; c < nc; ++c) {
        const double dc = norm(zs - ref_corner(box, c));
        if (dc > reach) continue;
        double cstep = 0.25;
        for (int j = 1; j <= 5; ++j) {
            cstep *= 0.25;
            pts[n++] = wrap_param(c + cstep, nc);
            pts[n++] = wrap_param(c - cstep, nc);
        }
    }
    for (int i = 0; i < n; ++i) {
        const double q = round(pts[i] * 4.0) * 0.25;
        if (fabs(pts[i] - q) <= tol) pts[i] = wrap_param(q, nc);
    }
    // insertion sort (n <= 67)
    for (int i = 1; i < n; ++i) {
        const double v = pts[i];
        int j = i - 1;
        while (j >= 0 && pts[j] > v) {
            pts[j + 1] = pts[j];
            --j;
        }
        pts[j + 1] = v;
    }
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (m == 0 || pts[i] - ep[m - 1] > tol) ep[m++] = pts[i];
    if (m > 1 && ep[0] + nc - ep[m - 1] <= tol) --m;
    return m;
}

// One panel k of the layout: its edge, corner A, edge vector E, local
// parameters [sa, sb]; false when the panel is collinear with the star
// (dropped, singular.cpp:176-182).
VPG_HD bool boundary_panel(int box, V2 zs, const double* ep, int np, int k, V2& A, V2& E, double& sa,
                           double& sb) {
    const int nc = ref_edges(box);
    const double tol = 1e-9;
    const double a = ep[k];
    const double b = (k + 1 < np) ? ep[k + 1] : ep[0] + nc;
    int e = static_cast<int>(floor(a + tol));
    if (e >= nc) e -= nc;
    A = ref_corner(box, e);
    E = ref_corner(box, e + 1) - A;
    sa = a - e;
    sb = b - e;
    const double elen = norm(E);
    return !(fabs(cross(A + sa * E - zs, E)) <= 1e-11 * elen && fabs(cross(A + sb * E - zs, E)) <= 1e-11 * elen);
}

// ------------------------------------------------------------------- basis --
// chebyshev2d_eval (basis.cpp:131-137, 193-199): out[a p + b] = T_a(x) T_b(y)
VPG_HD void cheb1d(int p, double z, double* t) {
    t[0] = 1;
    if (p > 1) t[1] = z;
    for (int k = 2; k < p; ++k) t[k] = 2 * z * t[k - 1] - t[k - 2];
}

// Jacobi P^{(0,beta)} recurrence (basis.cpp:36-43)
VPG_HD double jacobi_next(int k, double beta, double x, double pk, double pkm1) {
    const double a1 = 2 * (k + 1) * (k + beta + 1) * (2 * k + beta);
    const double a2 = (2 * k + beta + 1) * (-beta * beta);
    const double a3 = (2 * k + beta) * (2 * k + beta + 1) * (2 * k + beta + 2);
    const double a4 = 2 * (k + beta) * k * (2 * k + beta + 2);
    return ((a2 + a3 * x) * pk - a4 * pkm1) / a1;
}

#undef VPG_HD

}  // namespace geom
}  // namespace vpg
