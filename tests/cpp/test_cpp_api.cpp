// C++ mirror smoke/parity program (include/volpot_b200/summation.hpp).
// Reads: n_src n_tgt, then src xy, q, tgt xy (float64) from argv[1];
// writes: fmm potentials, direct potentials (skip semantics checked via
// error path) to argv[2].  Exit 0 on success.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <stdexcept>

#include <cmath>

#include "volpot_b200/bie.hpp"
#include "volpot_b200/summation.hpp"

using namespace volpot_b200;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::ifstream in(argv[1], std::ios::binary);
    int64_t ns = 0, nt = 0;
    in.read(reinterpret_cast<char*>(&ns), 8);
    in.read(reinterpret_cast<char*>(&nt), 8);
    std::vector<Vec2> src(static_cast<size_t>(ns)), tgt(static_cast<size_t>(nt));
    std::vector<double> q(static_cast<size_t>(ns));
    in.read(reinterpret_cast<char*>(src.data()), 16 * ns);
    in.read(reinterpret_cast<char*>(q.data()), 8 * ns);
    in.read(reinterpret_cast<char*>(tgt.data()), 16 * nt);
    const Kernel k = make_kernel(KernelFamily::Laplace);
    SummationPlan plan(k, src, tgt, 1e-12);
    std::vector<double> a = plan.apply(q);
    std::vector<double> b = accelerated_sum(k, SourceSet{src, q}, tgt);
    // reference error semantics
    int errors = 0;
    try {
        plan.apply(std::vector<double>(3, 1.0));
    } catch (const std::invalid_argument& e) {
        errors += std::string(e.what()).find("does not match source count") != std::string::npos;
    }
    try {
        make_kernel(KernelFamily::ModifiedHelmholtz, 0.0);
    } catch (const std::invalid_argument&) {
        ++errors;
    }
    try {
        direct_sum(k, SourceSet{{Vec2{0, 0}}, {1.0}}, {Vec2{0, 0}});
    } catch (const std::invalid_argument& e) {
        errors += std::string(e.what()).find("coincides") != std::string::npos;
    }
    try {
        bessel_k0(-1.0);
    } catch (const std::domain_error&) {
        ++errors;
    }
    SummationPlan moved = std::move(plan);
    std::vector<double> c = moved.apply(q);
    // operator-level apply with an empty correction map and charges = samples:
    // identical to the plan's apply
    if (ns == nt) {
        std::vector<int32_t> blk_off(static_cast<size_t>(nt) + 1, 0), node_off{0, int32_t(ns)};
        CorrectionMap corr(blk_off, {}, {}, {0, 1}, {0.0}, node_off);
        VolumePotentialOperator op(moved, corr);
        ApplyTimings tm;
        const std::vector<double> d = op.apply(q, &tm);
        errors += (d == c) && tm.smooth_seconds > 0.0 ? 0 : 100;
    }
    // layer potential (bie.hpp mirror): phi = 1 on a circle is -1 inside and
    // 0 outside (Gauss's lemma), and a short density throws the reference text
    {
        BoundarySystem sys;
        sys.kernel = k;
        CurveBlock c;
        c.n = 64;
        c.length = M_PI;  // radius 0.5
        c.diam = 1.0;
        for (int j = 0; j < 8 * c.n; ++j) {
            const double t = 2.0 * M_PI * j / (8 * c.n);
            const Vec2 nv{std::cos(t), std::sin(t)};
            c.fine_x.push_back(Vec2{0.5 * nv.x, 0.5 * nv.y});
            c.fine_normal.push_back(nv);
            c.fine_speed.push_back(0.5);
            if (j % 8 == 0) {
                c.x.push_back(c.fine_x.back());
                c.normal.push_back(nv);
                c.speed.push_back(0.5);
            }
        }
        sys.curves.push_back(c);
        sys.n_density = 64;
        const std::vector<double> u =
            eval_layer_potential(sys, std::vector<double>(64, 1.0), {Vec2{0.1, 0.2}, Vec2{2.0, 0.0}});
        errors += (std::fabs(u[0] + 1.0) < 1e-12 && std::fabs(u[1]) < 1e-12) ? 1 : 0;
        try {
            eval_layer_potential(sys, std::vector<double>(63, 1.0), {Vec2{0.1, 0.2}});
        } catch (const std::invalid_argument& e) {
            errors += std::string(e.what()).find("coefficient length mismatch") != std::string::npos;
        }
    }
    std::ofstream out(argv[2], std::ios::binary);
    out.write(reinterpret_cast<const char*>(a.data()), 8 * nt);
    out.write(reinterpret_cast<const char*>(b.data()), 8 * nt);
    out.write(reinterpret_cast<const char*>(c.data()), 8 * nt);
    std::printf("{\"levels\": %d, \"order\": %d, \"errors_ok\": %d}\n", moved.levels(),
                moved.expansion_order(), errors);
    return errors == 6 ? 0 : 1;
}
