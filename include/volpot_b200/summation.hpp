// volpot_b200/summation.hpp -- header-only C++ mirror of the reference
// summation API (proj/include/volpot/summation.hpp, kernel.hpp) on top of the
// C ABI in volpot_b200.h.  Same names, argument meaning and exceptions:
//
//   reference (file:line)                      here
//   volpot::Vec2            (common.hpp:13-32)  volpot_b200::Vec2 (same 16-byte POD)
//   volpot::KernelFamily/Kernel/make_kernel
//                           (kernel.hpp:77-96)  same names
//   volpot::bessel_k0       (kernel.hpp:74)     bessel_k0 (evaluated on the GPU)
//   volpot::SourceSet       (summation.hpp:14)  SourceSet
//   volpot::direct_sum      (summation.hpp:22)  direct_sum
//   volpot::SummationPlan   (summation.hpp:34)  SummationPlan (+ apply_device)
//   volpot::accelerated_sum (summation.hpp:58)  accelerated_sum
//
// Exceptions: std::invalid_argument for size mismatches, coincident points
// in direct_sum and bad kernels; std::domain_error for bessel_k0(x <= 0);
// std::runtime_error for CUDA failures (the reference has no such case).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "volpot_b200.h"

namespace volpot_b200 {

struct Vec2 {
    double x = 0.0, y = 0.0;
};
static_assert(sizeof(Vec2) == 16, "Vec2 must stay a 16-byte xy POD");

namespace detail {
inline void check(int status) {
    if (status == VPG_OK) return;
    const std::string msg = vpg_last_error();
    switch (status) {
        case VPG_ERR_INVALID_ARGUMENT:
        case VPG_ERR_COINCIDENT:
            throw std::invalid_argument(msg);
        case VPG_ERR_DOMAIN:
            throw std::domain_error(msg);
        default:
            throw std::runtime_error(msg);
    }
}
}  // namespace detail

enum class KernelFamily { Laplace = VPG_LAPLACE, ModifiedHelmholtz = VPG_MODIFIED_HELMHOLTZ };

struct Kernel {
    KernelFamily family = KernelFamily::Laplace;
    double lambda = 0.0;
};

inline Kernel make_kernel(KernelFamily family, double lambda = 0.0) {
    if (family == KernelFamily::ModifiedHelmholtz && !(lambda > 0.0))
        throw std::invalid_argument("make_kernel: modified Helmholtz needs lambda > 0");
    return Kernel{family, lambda};
}

inline double bessel_k0(double x, int device = 0) {
    double out = 0.0;
    detail::check(vpg_bessel_k0(&x, 1, &out, device));
    return out;
}

struct SourceSet {
    std::vector<Vec2> points;
    std::vector<double> charges;
};

inline std::vector<double> direct_sum(const Kernel& kernel, const SourceSet& sources,
                                      const std::vector<Vec2>& targets, int device = 0) {
    if (sources.charges.size() != sources.points.size())
        throw std::invalid_argument("direct_sum: points/charges size mismatch");
    std::vector<double> out(targets.size(), 0.0);
    int64_t ci = -1, cj = -1;
    detail::check(vpg_direct_sum(static_cast<int>(kernel.family), kernel.lambda,
                                 reinterpret_cast<const double*>(sources.points.data()),
                                 sources.charges.data(), int64_t(sources.points.size()),
                                 reinterpret_cast<const double*>(targets.data()),
                                 int64_t(targets.size()), out.data(), 0, &ci, &cj, device, 0u,
                                 nullptr));
    return out;
}

class SummationPlan {
  public:
    SummationPlan(const Kernel& kernel, std::vector<Vec2> sources, std::vector<Vec2> targets,
                  double epsilon = 1e-12, int mode = VPG_MODE_REFERENCE, int device = 0) {
        detail::check(vpg_plan_create(static_cast<int>(kernel.family), kernel.lambda,
                                      reinterpret_cast<const double*>(sources.data()),
                                      int64_t(sources.size()),
                                      reinterpret_cast<const double*>(targets.data()),
                                      int64_t(targets.size()), epsilon, mode, device, &plan_));
        detail::check(vpg_plan_info(plan_, &info_));
    }
    ~SummationPlan() {
        if (plan_) vpg_plan_destroy(plan_);
    }
    SummationPlan(SummationPlan&& o) noexcept : plan_(o.plan_), info_(o.info_) { o.plan_ = nullptr; }
    SummationPlan& operator=(SummationPlan&& o) noexcept {
        std::swap(plan_, o.plan_);
        std::swap(info_, o.info_);
        return *this;
    }
    SummationPlan(const SummationPlan&) = delete;
    SummationPlan& operator=(const SummationPlan&) = delete;

    // summation.cpp:610-643: potentials in target order; const and safe to
    // call concurrently with distinct charge vectors.
    std::vector<double> apply(const std::vector<double>& charges) const {
        std::vector<double> out(static_cast<std::size_t>(info_.num_targets));
        detail::check(vpg_plan_apply(plan_, charges.data(), int64_t(charges.size()), out.data(), 0u,
                                     nullptr));
        return out;
    }
    // Device-resident charges/potentials on a caller stream (no copies).
    void apply_device(const double* q_dev, double* out_dev, void* stream = nullptr) const {
        detail::check(vpg_plan_apply(plan_, q_dev, info_.num_sources, out_dev,
                                     VPG_DEVICE_POINTERS | VPG_NO_SYNC, stream));
    }

    std::size_t num_sources() const { return std::size_t(info_.num_sources); }
    std::size_t num_targets() const { return std::size_t(info_.num_targets); }
    int levels() const { return info_.levels; }
    int expansion_order() const { return info_.expansion_order; }
    const vpg_plan_info_t& info() const { return info_; }
    vpg_plan* handle() const { return plan_; }

  private:
    vpg_plan* plan_ = nullptr;
    vpg_plan_info_t info_{};
};

// Correction map (potential.cpp:92-110, 446-462) on the device: out += C f.
class CorrectionMap {
  public:
    CorrectionMap(const std::vector<int32_t>& blk_off, const std::vector<int32_t>& blk_cell,
                  const std::vector<int32_t>& blk_pool, const std::vector<int64_t>& pool_off,
                  const std::vector<double>& pool_vals, const std::vector<int32_t>& node_off, int device = 0)
        : nt_(int64_t(blk_off.size()) - 1), ndofs_(node_off.empty() ? 0 : node_off.back()) {
        detail::check(vpg_corr_create(nt_, blk_off.data(), int64_t(blk_cell.size()), blk_cell.data(),
                                      blk_pool.data(), int64_t(pool_off.size()) - 1, pool_off.data(),
                                      pool_vals.data(), int64_t(node_off.size()) - 1, node_off.data(), device,
                                      &h_));
    }
    ~CorrectionMap() {
        if (h_) vpg_corr_destroy(h_);
    }
    CorrectionMap(const CorrectionMap&) = delete;
    CorrectionMap& operator=(const CorrectionMap&) = delete;
    void apply(const std::vector<double>& f, std::vector<double>& out) const {
        detail::check(vpg_corr_apply(h_, f.data(), int64_t(f.size()), out.data(), 0u, nullptr));
    }
    vpg_corr* handle() const { return h_; }
    int64_t num_targets() const { return nt_; }

  private:
    vpg_corr* h_ = nullptr;
    int64_t nt_ = 0, ndofs_ = 0;
};

// build_charges (potential.cpp:397-412): charges = src_wj * (O_type f) per cell.
class ChargeMap {
  public:
    ChargeMap(const std::vector<int32_t>& cell_type, const std::vector<int32_t>& node_off,
              const std::vector<int32_t>& src_off, const std::vector<double>& over0, int np0, int nq0,
              const std::vector<double>& over1, int np1, int nq1, const std::vector<double>& src_wj,
              int device = 0) {
        detail::check(vpg_charges_create(int64_t(cell_type.size()), cell_type.data(), node_off.data(),
                                         src_off.data(), over0.data(), np0, nq0, over1.data(), np1, nq1,
                                         src_wj.data(), device, &h_));
    }
    ~ChargeMap() {
        if (h_) vpg_charges_destroy(h_);
    }
    ChargeMap(const ChargeMap&) = delete;
    ChargeMap& operator=(const ChargeMap&) = delete;
    vpg_charges* handle() const { return h_; }

  private:
    vpg_charges* h_ = nullptr;
};

// VolumePotentialOperator::apply (potential.cpp:431-470), device-resident:
// out = plan.apply(build_charges(f)) + C f.  Borrows the plan and the maps.
struct ApplyTimings {
    double smooth_seconds = 0.0;
    double correction_seconds = 0.0;
};

class VolumePotentialOperator {
  public:
    VolumePotentialOperator(const SummationPlan& plan, const CorrectionMap& corr,
                            const ChargeMap* charges = nullptr)
        : nt_(int64_t(plan.num_targets())) {
        detail::check(vpg_operator_create(plan.handle(), charges ? charges->handle() : nullptr, corr.handle(),
                                          &h_));
    }
    ~VolumePotentialOperator() {
        if (h_) vpg_operator_destroy(h_);
    }
    VolumePotentialOperator(const VolumePotentialOperator&) = delete;
    VolumePotentialOperator& operator=(const VolumePotentialOperator&) = delete;
    std::vector<double> apply(const std::vector<double>& f_samples, ApplyTimings* timings = nullptr) const {
        std::vector<double> out(static_cast<std::size_t>(nt_));
        float t[2] = {0.f, 0.f};
        detail::check(vpg_operator_apply(h_, f_samples.data(), int64_t(f_samples.size()), out.data(), 0u, nullptr,
                                         timings ? t : nullptr));
        if (timings) {
            timings->smooth_seconds = t[0] * 1e-3;
            timings->correction_seconds = t[1] * 1e-3;
        }
        return out;
    }

  private:
    vpg_operator* h_ = nullptr;
    int64_t nt_ = 0;
};

inline std::vector<double> accelerated_sum(const Kernel& kernel, const SourceSet& sources,
                                           const std::vector<Vec2>& targets,
                                           double epsilon = 1e-12) {
    SummationPlan plan(kernel, sources.points, targets, epsilon);
    return plan.apply(sources.charges);
}

}  // namespace volpot_b200
