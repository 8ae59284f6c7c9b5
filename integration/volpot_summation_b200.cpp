// volpot_summation_b200.cpp -- drop-in replacement for the reference
// translation unit proj/src/summation.cpp.
//
// Compile this file INSTEAD of proj/src/summation.cpp, against the
// reference's own header proj/include/volpot/summation.hpp, and link
// libvolpot_b200.so: every caller of volpot::SummationPlan /
// volpot::direct_sum / volpot::accelerated_sum (potential.cpp:390, 443;
// summation.cpp:645-651 callers; bie.cpp:507-510) then runs the B200
// kernels with no source change.  The reference header declares
// SummationPlan::Impl as an incomplete pimpl type (summation.hpp:52-54), so
// the device plan lives behind it without touching the public API.
//
// Semantics kept: epsilon clamp, pairwise threshold, tree depth and P
// (VPG_MODE_REFERENCE), apply() const + concurrent, std::invalid_argument
// messages of summation.cpp:504-538 and 613-617.
#include <stdexcept>
#include <string>
#include <vector>

#include "volpot/summation.hpp"
#include "volpot_b200.h"

namespace volpot {

namespace {
void check(int status) {
    if (status == VPG_OK) return;
    const std::string msg = vpg_last_error();
    if (status == VPG_ERR_INVALID_ARGUMENT || status == VPG_ERR_COINCIDENT)
        throw std::invalid_argument(msg);
    if (status == VPG_ERR_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}
int family_of(const Kernel& k) {
    return k.family == KernelFamily::Laplace ? VPG_LAPLACE : VPG_MODIFIED_HELMHOLTZ;
}
}  // namespace

std::vector<double> direct_sum(const Kernel& kernel, const SourceSet& sources,
                               const std::vector<Vec2>& targets) {
    if (sources.charges.size() != sources.points.size())
        throw std::invalid_argument("direct_sum: points/charges size mismatch");
    std::vector<double> out(targets.size(), 0.0);
    check(vpg_direct_sum(family_of(kernel), kernel.lambda,
                         reinterpret_cast<const double*>(sources.points.data()),
                         sources.charges.data(), static_cast<int64_t>(sources.points.size()),
                         reinterpret_cast<const double*>(targets.data()),
                         static_cast<int64_t>(targets.size()), out.data(), 0, nullptr, nullptr, 0,
                         0u, nullptr));
    return out;
}

struct SummationPlan::Impl {
    vpg_plan* plan = nullptr;
    vpg_plan_info_t info{};
    ~Impl() {
        if (plan) vpg_plan_destroy(plan);
    }
};

SummationPlan::SummationPlan(const Kernel& kernel, std::vector<Vec2> sources,
                             std::vector<Vec2> targets, double epsilon)
    : impl_(new Impl) {
    check(vpg_plan_create(family_of(kernel), kernel.lambda,
                          reinterpret_cast<const double*>(sources.data()),
                          static_cast<int64_t>(sources.size()),
                          reinterpret_cast<const double*>(targets.data()),
                          static_cast<int64_t>(targets.size()), epsilon, VPG_MODE_REFERENCE, 0,
                          &impl_->plan));
    check(vpg_plan_info(impl_->plan, &impl_->info));
}

SummationPlan::~SummationPlan() = default;
SummationPlan::SummationPlan(SummationPlan&&) noexcept = default;
SummationPlan& SummationPlan::operator=(SummationPlan&&) noexcept = default;

std::vector<double> SummationPlan::apply(const std::vector<double>& charges) const {
    std::vector<double> out(static_cast<std::size_t>(impl_->info.num_targets), 0.0);
    check(vpg_plan_apply(impl_->plan, charges.data(), static_cast<int64_t>(charges.size()),
                         out.data(), 0u, nullptr));
    return out;
}

std::size_t SummationPlan::num_sources() const { return std::size_t(impl_->info.num_sources); }
std::size_t SummationPlan::num_targets() const { return std::size_t(impl_->info.num_targets); }
int SummationPlan::levels() const { return impl_->info.levels; }
int SummationPlan::expansion_order() const { return impl_->info.expansion_order; }

std::vector<double> accelerated_sum(const Kernel& kernel, const SourceSet& sources,
                                    const std::vector<Vec2>& targets, double epsilon) {
    SummationPlan plan(kernel, sources.points, targets, epsilon);
    return plan.apply(sources.charges);
}

}  // namespace volpot
