// volpot_b200/bie.hpp -- header-only C++ mirror of the reference
// layer-potential evaluation (proj/include/volpot/bie.hpp) on top of the C
// ABI in volpot_b200.h:
//
//   reference (file:line)                           here
//   BoundarySystem::CurveBlock  (bie.hpp:30-47)     CurveBlock (the fields the
//                                                   evaluation reads, same names)
//   BoundarySystem              (bie.hpp:29-59)     BoundarySystem (geometry; no
//                                                   system matrix)
//   eval_layer_potential        (bie.hpp:87-90)     eval_layer_potential
//
// A reference BoundarySystem converts field by field (to_curve_blocks in
// INTEGRATION.md).  The device copy of the geometry is made once per
// LayerEvaluator; eval_layer_potential(sys, ...) builds one per call like the
// reference signature implies.  Exceptions: std::invalid_argument with the
// reference messages (bie.cpp:388, 452, 455-457); std::runtime_error for CUDA
// failures.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "volpot_b200.h"
#include "volpot_b200/summation.hpp"

namespace volpot_b200 {

struct CurveBlock {
    int n = 0;
    int offset = 0;
    double length = 0;
    double diam = 0;
    std::vector<Vec2> x;
    std::vector<Vec2> normal;
    std::vector<double> speed;
    std::vector<Vec2> fine_x;  // 8n refined geometry (bie.cpp:206-215)
    std::vector<Vec2> fine_normal;
    std::vector<double> fine_speed;
    Vec2 log_center;
};

struct BoundarySystem {
    Kernel kernel;
    std::vector<CurveBlock> curves;
    int n_density = 0;
    int n_aux = 0;
    int size() const { return n_density + n_aux; }
};

class LayerEvaluator {
public:
    explicit LayerEvaluator(const BoundarySystem& sys, int device = 0) {
        std::vector<vpg_curve_block> cb;
        for (const CurveBlock& c : sys.curves) {
            if (c.x.size() != size_t(c.n) || c.fine_x.size() != size_t(8 * c.n))
                throw std::invalid_argument("CurveBlock: node arrays do not match n");
            vpg_curve_block b{};
            b.n = c.n;
            b.offset = c.offset;
            b.length = c.length;
            b.diam = c.diam;
            b.x = &c.x[0].x;
            b.normal = &c.normal[0].x;
            b.speed = c.speed.data();
            b.fine_x = &c.fine_x[0].x;
            b.fine_normal = &c.fine_normal[0].x;
            b.fine_speed = c.fine_speed.data();
            b.log_center[0] = c.log_center.x;
            b.log_center[1] = c.log_center.y;
            cb.push_back(b);
        }
        vpg_layer* h = nullptr;
        detail::check(vpg_layer_create(int(sys.kernel.family), sys.kernel.lambda, cb.data(), int(cb.size()),
                                       sys.n_density, sys.n_aux, device, &h));
        h_.reset(h);
    }

    std::vector<double> eval(const std::vector<double>& coeffs, const std::vector<Vec2>& targets,
                             bool allow_close = false) const {
        std::vector<double> out(targets.size(), 0.0);
        detail::check(vpg_layer_eval(h_.get(), coeffs.data(), int64_t(coeffs.size()),
                                     targets.empty() ? nullptr : &targets[0].x, int64_t(targets.size()),
                                     allow_close ? 1 : 0, out.data(), 0u, nullptr));
        return out;
    }

    // device pointers, stream-ordered (VPG_DEVICE_POINTERS)
    void eval_device(const double* coeffs, int64_t ncoeffs, const double* tgt_xy, int64_t nt, double* out,
                     bool allow_close, void* stream) const {
        detail::check(vpg_layer_eval(h_.get(), coeffs, ncoeffs, tgt_xy, nt, allow_close ? 1 : 0, out,
                                     VPG_DEVICE_POINTERS, stream));
    }

private:
    struct Del {
        void operator()(vpg_layer* p) const { vpg_layer_destroy(p); }
    };
    std::unique_ptr<vpg_layer, Del> h_;
};

inline std::vector<double> eval_layer_potential(const BoundarySystem& sys, const std::vector<double>& coeffs,
                                                const std::vector<Vec2>& targets, bool allow_close = false) {
    return LayerEvaluator(sys).eval(coeffs, targets, allow_close);
}

}  // namespace volpot_b200
