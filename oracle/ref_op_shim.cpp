// TEST INFRASTRUCTURE ONLY.  extern "C" adapter around the UNMODIFIED reference
// operator sources (proj/src/{potential,singular,basis,quad1d,geometry,mesh,
// delaunay,bie,triangle_node_data,kernel,common,summation}.cpp), compiled in
// place from /root/reference by oracle/Makefile against the Eigen restatement
// (oracle/eigen_restated/Eigen/Dense) into oracle/_ref/libvolpot_ref_op.so.
//
// potential.cpp is #included into this translation unit (not copied) so the
// adapter can read the operator's private correction map
// (VolumePotentialOperator::Impl, potential.cpp:81-131) for the parity pins.
//
// Wrapped reference entry points:
//   build_mesh + StarCurve                   (mesh.hpp:38, geometry.hpp:60-72)
//   VolumePotentialOperator ctor / apply     (potential.hpp:36-52)
//   Impl::build_charges                      (potential.cpp:397-412)
//   smooth_potential_row                     (singular.cpp:428-456)
//   SingularTargetRule::row                  (singular.cpp:383-415)
//   reduce_to_rays + apply_ray_quadrature    (singular.cpp:274-310)
//   box_correction_table                     (singular.cpp:586-646)
//   basis tables / source rules / oversample (basis.cpp:48-324)
//   classify_target                          (mesh.cpp:410-448)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iomanip>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <ostream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <Eigen/Dense>

#include "volpot/basis.hpp"
#include "volpot/common.hpp"
#include "volpot/geometry.hpp"
#include "volpot/kernel.hpp"
#include "volpot/mesh.hpp"
#include "volpot/quad1d.hpp"
#include "volpot/singular.hpp"
#include "volpot/summation.hpp"

#define private public
#include "volpot/potential.hpp"
#undef private
#include "../src/potential.cpp"  // NOLINT: compiled in place for Impl access
#include "volpot/bie.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct MeshBox {
    volpot::Domain dom;
    volpot::HybridMesh mesh;
};

struct OpBox {
    std::unique_ptr<volpot::VolumePotentialOperator> op;
};

volpot::Kernel kern(int family, double lambda) {
    return volpot::make_kernel(family == 0 ? volpot::KernelFamily::Laplace
                                           : volpot::KernelFamily::ModifiedHelmholtz,
                               lambda);
}

void put(double* out, const Eigen::Dense& v) {
    for (Eigen::Index i = 0; i < v.size(); ++i) out[i] = v(i);
}
}  // namespace

extern "C" {

const char* refop_last_error() { return g_err.c_str(); }
void refop_set_threads(int n) { volpot::set_thread_count(n); }

// ---- mesh ----
int refop_mesh_star_holes(double cx, double cy, double r0, double amp, int arms, double phase, double h,
                          double delta, int nholes, const double* holes /*cx, cy, r per circle*/, void** out) {
    return guarded([&] {
        auto mb = std::make_unique<MeshBox>();
        mb->dom.outer = std::make_shared<volpot::StarCurve>(volpot::Vec2{cx, cy}, r0, amp, arms, phase);
        for (int k = 0; k < nholes; ++k)
            mb->dom.holes.push_back(std::make_shared<volpot::Circle>(volpot::Vec2{holes[3 * k], holes[3 * k + 1]},
                                                                     holes[3 * k + 2]));
        mb->mesh = volpot::build_mesh(mb->dom, h, delta);
        mb->mesh.domain = &mb->dom;
        *out = mb.release();
    });
}

int refop_mesh_star(double cx, double cy, double r0, double amp, int arms, double phase, double h,
                    double delta, void** out) {
    return guarded([&] {
        auto mb = std::make_unique<MeshBox>();
        mb->dom.outer = std::make_shared<volpot::StarCurve>(volpot::Vec2{cx, cy}, r0, amp, arms, phase);
        mb->mesh = volpot::build_mesh(mb->dom, h, delta);
        mb->mesh.domain = &mb->dom;
        *out = mb.release();
    });
}

void refop_mesh_free(void* m) { delete static_cast<MeshBox*>(m); }

int refop_mesh_info(void* m, int* ncell, int* ntri, int* nbox, double* h) {
    const auto& me = static_cast<MeshBox*>(m)->mesh;
    *ncell = me.num_cells();
    *ntri = me.n_tri;
    *nbox = me.n_box;
    *h = me.h;
    return 0;
}

// type: 0 StraightTri, 1 CurvedTri, 2 Box; v: 6 per cell; tt: (ta, tb);
// ch: (center.x, center.y, h); curve: index into the domain's curves or -1
int refop_mesh_cells(void* m, int* type, double* v, double* tt, double* ch, int* curve) {
    const auto& mb = *static_cast<MeshBox*>(m);
    const auto& cells = mb.mesh.cells;
    for (size_t c = 0; c < cells.size(); ++c) {
        const auto& cl = cells[c];
        type[c] = cl.type == volpot::CellType::StraightTri ? 0 : cl.type == volpot::CellType::CurvedTri ? 1 : 2;
        for (int k = 0; k < 3; ++k) {
            v[6 * c + 2 * k] = cl.v[k].x;
            v[6 * c + 2 * k + 1] = cl.v[k].y;
        }
        tt[2 * c] = cl.ta;
        tt[2 * c + 1] = cl.tb;
        ch[3 * c] = cl.center.x;
        ch[3 * c + 1] = cl.center.y;
        ch[3 * c + 2] = cl.h;
        curve[c] = -1;
        if (cl.curve == mb.dom.outer.get()) curve[c] = 0;
        for (size_t k = 0; k < mb.dom.holes.size(); ++k)
            if (cl.curve == mb.dom.holes[k].get()) curve[c] = int(k) + 1;
    }
    return 0;
}

int refop_mesh_nodes(void* m, int p, double* xy) {
    return guarded([&] {
        const auto nodes = volpot::mesh_nodes(static_cast<MeshBox*>(m)->mesh, p);
        for (size_t i = 0; i < nodes.size(); ++i) {
            xy[2 * i] = nodes[i].x;
            xy[2 * i + 1] = nodes[i].y;
        }
    });
}

int refop_classify(void* m, double x, double y, double D, int* self, int* near, int* nnear) {
    return guarded([&] {
        const auto tc = volpot::classify_target(static_cast<MeshBox*>(m)->mesh, {x, y}, D);
        *self = tc.self;
        *nnear = static_cast<int>(tc.near_cells.size());
        for (size_t k = 0; k < tc.near_cells.size(); ++k) near[k] = tc.near_cells[k];
    });
}

// ---- operator ----
int refop_op_create(void* m, int family, double lambda, int p, int q, const double* tgt, int64_t nt,
                    double eps, void** out) {
    return guarded([&] {
        std::vector<volpot::Vec2> t(static_cast<size_t>(nt));
        for (int64_t i = 0; i < nt; ++i) t[size_t(i)] = {tgt[2 * i], tgt[2 * i + 1]};
        auto ob = std::make_unique<OpBox>();
        ob->op = std::make_unique<volpot::VolumePotentialOperator>(
            static_cast<MeshBox*>(m)->mesh, kern(family, lambda), p, q, std::move(t), eps);
        *out = ob.release();
    });
}

void refop_op_free(void* o) { delete static_cast<OpBox*>(o); }

// sizes: ndofs, nsrcs, nt, ncell, nblocks, npool, pool_len, build_ms
int refop_op_sizes(void* o, double* s) {
    const auto& im = *static_cast<OpBox*>(o)->op->impl_;
    int64_t len = 0;
    for (const auto& r : im.pool) len += r.size();
    s[0] = im.stats.ndofs;
    s[1] = im.stats.nsrcs;
    s[2] = static_cast<double>(im.targets.size());
    s[3] = static_cast<double>(im.mesh->cells.size());
    s[4] = static_cast<double>(im.blocks.size());
    s[5] = static_cast<double>(im.pool.size());
    s[6] = static_cast<double>(len);
    s[7] = im.stats.build_seconds * 1e3;
    return 0;
}

// The operator's data in its own layouts.  Any pointer may be null.
int refop_op_export(void* o, double* node_xy, int* node_off, int* src_off, double* src_xy, double* src_wj,
                    int* blk_off, int* blk_cell, int* blk_pool, int64_t* pool_off, double* pool_vals) {
    const auto& im = *static_cast<OpBox*>(o)->op->impl_;
    if (node_xy)
        for (size_t i = 0; i < im.nodes.size(); ++i) {
            node_xy[2 * i] = im.nodes[i].x;
            node_xy[2 * i + 1] = im.nodes[i].y;
        }
    if (node_off) std::copy(im.node_off.begin(), im.node_off.end(), node_off);
    if (src_off) std::copy(im.src_off.begin(), im.src_off.end(), src_off);
    if (src_xy)
        for (size_t i = 0; i < im.src_pts.size(); ++i) {
            src_xy[2 * i] = im.src_pts[i].x;
            src_xy[2 * i + 1] = im.src_pts[i].y;
        }
    if (src_wj) std::copy(im.src_wj.begin(), im.src_wj.end(), src_wj);
    if (blk_off) std::copy(im.blk_off.begin(), im.blk_off.end(), blk_off);
    for (size_t k = 0; k < im.blocks.size(); ++k) {
        if (blk_cell) blk_cell[k] = im.blocks[k].cell;
        if (blk_pool) blk_pool[k] = im.blocks[k].pool;
    }
    int64_t at = 0;
    for (size_t r = 0; r < im.pool.size(); ++r) {
        if (pool_off) pool_off[r] = at;
        if (pool_vals)
            for (Eigen::Index j = 0; j < im.pool[r].size(); ++j) pool_vals[at + j] = im.pool[r](j);
        at += im.pool[r].size();
    }
    if (pool_off) pool_off[im.pool.size()] = at;
    return 0;
}

int refop_op_apply(void* o, const double* f, int64_t n, double* out, double* times) {
    return guarded([&] {
        const auto& op = *static_cast<OpBox*>(o)->op;
        volpot::ApplyTimings tm;
        const auto r = op.apply(std::vector<double>(f, f + n), &tm);
        std::copy(r.begin(), r.end(), out);
        if (times) {
            times[0] = tm.smooth_seconds;
            times[1] = tm.correction_seconds;
        }
    });
}

int refop_op_build_charges(void* o, const double* f, int64_t n, double* charges) {
    return guarded([&] {
        const auto& im = *static_cast<OpBox*>(o)->op->impl_;
        std::vector<double> ch;
        im.build_charges(std::vector<double>(f, f + n), ch);
        std::copy(ch.begin(), ch.end(), charges);
    });
}

int refop_op_correction_row_generic(void* o, int cell, double x, double y, int is_self, double* out) {
    return guarded([&] {
        const auto& im = *static_cast<OpBox*>(o)->op->impl_;
        put(out, im.correction_row_generic(im.mesh->cells[size_t(cell)], {x, y}, is_self != 0));
    });
}

// ---- rows on one cell ----
int refop_smooth_row(void* m, int cell, int p, int q, double x, double y, int family, double lambda,
                     double* out) {
    return guarded([&] {
        const auto& c = static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)];
        put(out, volpot::smooth_potential_row(c, p, q, {x, y}, kern(family, lambda)));
    });
}

int refop_self_row(void* m, int cell, int p, double zx, double zy, double x, double y, int family,
                   double lambda, double* out) {
    return guarded([&] {
        const auto& c = static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)];
        volpot::SingularTargetRule rule(volpot::ref_cell_of(c.type), p, {zx, zy});
        put(out, rule.row(c, kern(family, lambda), {x, y}));
    });
}

int refop_self_rule_nodes(int kind, int p, double zx, double zy, int* n) {
    return guarded([&] {
        volpot::SingularTargetRule rule(kind == 2 ? volpot::RefCell::Box : volpot::RefCell::Simplex, p,
                                        {zx, zy});
        *n = rule.num_nodes();
    });
}

int refop_ray_row(void* m, int cell, int p, double zx, double zy, double sx, double sy, double x, double y,
                  int family, double lambda, double* out) {
    return guarded([&] {
        const auto& c = static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)];
        const auto k = kern(family, lambda);
        const auto rq = volpot::reduce_to_rays(c, {zx, zy}, {sx, sy}, k, {x, y});
        put(out, volpot::apply_ray_quadrature(rq, c, p, k, {x, y}));
    });
}

int refop_nearest_reference_point(void* m, int cell, double x, double y, double* z, double* d) {
    return guarded([&] {
        const auto& c = static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)];
        const auto zz = volpot::nearest_reference_point(c, {x, y}, d);
        z[0] = zz.x;
        z[1] = zz.y;
    });
}

int refop_cell_invert(void* m, int cell, double x, double y, double* z) {
    return guarded([&] {
        const auto zz = static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)].invert({x, y});
        z[0] = zz.x;
        z[1] = zz.y;
    });
}

int refop_cell_map_deriv(void* m, int cell, double zx, double zy, double* o7) {
    return guarded([&] {
        volpot::Vec2 x, a, b;
        double j;
        static_cast<MeshBox*>(m)->mesh.cells[size_t(cell)].map_deriv({zx, zy}, x, a, b, j);
        const double v[7] = {x.x, x.y, a.x, a.y, b.x, b.y, j};
        std::copy(v, v + 7, o7);
    });
}

// box_correction_table(p, kernel, h): 25 blocks of p^2 x p^2, row-major per block
int refop_box_table(int p, int family, double lambda, double h, double* out) {
    return guarded([&] {
        const auto t = volpot::box_correction_table(p, kern(family, lambda), h);
        const int nb = p * p;
        for (int o = 0; o < 25; ++o)
            for (int i = 0; i < nb; ++i)
                for (int j = 0; j < nb; ++j) out[(size_t(o) * nb + i) * nb + j] = t[size_t(o)](i, j);
    });
}

// reference box_log moments (h- and kernel-independent), same layout
int refop_box_log(int p, double* out) {
    return guarded([&] {
        const auto& tb = volpot::reference_tables(p);
        const int nb = p * p;
        for (int o = 0; o < 25; ++o)
            for (int i = 0; i < nb; ++i)
                for (int j = 0; j < nb; ++j) out[(size_t(o) * nb + i) * nb + j] = tb.box_log[size_t(o)](i, j);
    });
}

// Basis data.  which: 0 tri nodes (n x 2), 1 tri C (n x n), 2 box nodes, 3 box C,
// 4 tri source nodes (q), 5 tri source w, 6 box source nodes, 7 box source w,
// 8 triangle_oversample(p, q) (nq x n), 9 box_oversample(p, q).  Row-major.
// Returns the element count in *n (call with out = null to size).
int refop_basis(int which, int p, int q, double* out, int64_t* n) {
    return guarded([&] {
        Eigen::MatrixXd m;
        switch (which) {
            case 0: m = volpot::triangle_table(p).nodes; break;
            case 1: m = volpot::triangle_table(p).C; break;
            case 2: m = volpot::box_table(p).nodes; break;
            case 3: m = volpot::box_table(p).C; break;
            case 4: m = volpot::triangle_source_rule(q).nodes; break;
            case 5: m = volpot::triangle_source_rule(q).w; break;
            case 6: m = volpot::box_source_rule(q).nodes; break;
            case 7: m = volpot::box_source_rule(q).w; break;
            case 8: m = volpot::triangle_oversample(p, q); break;
            case 9: m = volpot::box_oversample(p, q); break;
            default: throw std::invalid_argument("refop_basis: which");
        }
        *n = m.size();
        if (out)
            for (Eigen::Index i = 0; i < m.rows(); ++i)
                for (Eigen::Index j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j);
    });
}

// 1-D rules: which 0 gauss_legendre(n), 1 gauss_weight_t(n), 2 gauss_weight_tlog(n),
// 3 ray_singular_rule(), 4 ray_near_rule(d).  x then w.
int refop_rule1d(int which, int n, double d, double* x, double* w, int* size) {
    return guarded([&] {
        const volpot::QuadRule1D* r = nullptr;
        switch (which) {
            case 0: r = &volpot::gauss_legendre(n); break;
            case 1: r = &volpot::gauss_weight_t(n); break;
            case 2: r = &volpot::gauss_weight_tlog(n); break;
            case 3: r = &volpot::ray_singular_rule(); break;
            case 4: r = &volpot::ray_near_rule(d); break;
            default: throw std::invalid_argument("refop_rule1d: which");
        }
        *size = r->size();
        if (x) std::copy(r->x.begin(), r->x.end(), x);
        if (w) std::copy(r->w.begin(), r->w.end(), w);
    });
}

// boundary_discretization(kind, star): node zeta (2), t, factor per node
int refop_boundary(int kind, double sx, double sy, double* zeta, double* t, double* factor, int* n) {
    return guarded([&] {
        const auto bd = volpot::boundary_discretization(
            kind == 2 ? volpot::RefCell::Box : volpot::RefCell::Simplex, {sx, sy});
        *n = static_cast<int>(bd.nodes.size());
        if (zeta)
            for (size_t i = 0; i < bd.nodes.size(); ++i) {
                zeta[2 * i] = bd.nodes[i].zeta.x;
                zeta[2 * i + 1] = bd.nodes[i].zeta.y;
                t[i] = bd.nodes[i].t;
                factor[i] = bd.nodes[i].factor;
            }
    });
}

}  // extern "C"

// ---- boundary integral layer (bie.hpp:29-90) ----
namespace {
struct LayerBox {
    volpot::Domain dom;
    volpot::BoundarySystem sys;
};
}  // namespace

extern "C" {

int refop_layer_create(int family, double lambda, const double* star /*cx,cy,r0,amp,arms,phase*/, int nholes,
                       const double* holes /*cx,cy,r per hole*/, const int* n_per_curve, int ncount, void** out) {
    return guarded([&] {
        auto lb = std::make_unique<LayerBox>();
        lb->dom.outer = std::make_shared<volpot::StarCurve>(volpot::Vec2{star[0], star[1]}, star[2], star[3],
                                                            static_cast<int>(star[4]), star[5]);
        for (int k = 0; k < nholes; ++k)
            lb->dom.holes.push_back(std::make_shared<volpot::Circle>(
                volpot::Vec2{holes[3 * k], holes[3 * k + 1]}, holes[3 * k + 2]));
        lb->sys = volpot::assemble_nystrom(lb->dom, kern(family, lambda),
                                           std::vector<int>(n_per_curve, n_per_curve + ncount));
        *out = lb.release();
    });
}

void refop_layer_free(void* s) { delete static_cast<LayerBox*>(s); }

int refop_layer_info(void* s, int* ncurves, int* n_density, int* n_aux) {
    const auto& sys = static_cast<LayerBox*>(s)->sys;
    *ncurves = static_cast<int>(sys.curves.size());
    *n_density = sys.n_density;
    *n_aux = sys.n_aux;
    return 0;
}

// geometry of curve block c; scal = (n, offset, length, diam, log_center.x, log_center.y)
int refop_layer_curve(void* s, int c, double* scal, double* x, double* normal, double* speed, double* fx,
                      double* fnormal, double* fspeed) {
    const auto& b = static_cast<LayerBox*>(s)->sys.curves[size_t(c)];
    scal[0] = b.n;
    scal[1] = b.offset;
    scal[2] = b.length;
    scal[3] = b.diam;
    scal[4] = b.log_center.x;
    scal[5] = b.log_center.y;
    auto v2 = [](const std::vector<volpot::Vec2>& v, double* o) {
        if (!o) return;
        for (size_t i = 0; i < v.size(); ++i) {
            o[2 * i] = v[i].x;
            o[2 * i + 1] = v[i].y;
        }
    };
    v2(b.x, x);
    v2(b.normal, normal);
    v2(b.fine_x, fx);
    v2(b.fine_normal, fnormal);
    if (speed) std::copy(b.speed.begin(), b.speed.end(), speed);
    if (fspeed) std::copy(b.fine_speed.begin(), b.fine_speed.end(), fspeed);
    return 0;
}

int refop_layer_solve(void* s, const double* rhs, double* out) {
    return guarded([&] {
        const auto& sys = static_cast<LayerBox*>(s)->sys;
        const auto r = volpot::solve_density(sys, std::vector<double>(rhs, rhs + sys.size()));
        std::copy(r.begin(), r.end(), out);
    });
}

int refop_layer_eval(void* s, const double* coeffs, int64_t nc, const double* tgt, int64_t nt, int allow_close,
                     double* out) {
    return guarded([&] {
        const auto& sys = static_cast<LayerBox*>(s)->sys;
        std::vector<volpot::Vec2> t(static_cast<size_t>(nt));
        for (int64_t i = 0; i < nt; ++i) t[size_t(i)] = {tgt[2 * i], tgt[2 * i + 1]};
        const auto r = volpot::eval_layer_potential(sys, std::vector<double>(coeffs, coeffs + nc), t,
                                                    allow_close != 0);
        std::copy(r.begin(), r.end(), out);
    });
}

}  // extern "C"
