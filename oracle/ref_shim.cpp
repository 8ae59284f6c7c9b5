// TEST INFRASTRUCTURE ONLY.  extern "C" adapter around the UNMODIFIED
// reference summation code (proj/src/summation.cpp, kernel.cpp, common.cpp),
// compiled in place from /root/reference by oracle/Makefile into
// oracle/_ref/libvolpot_ref.so.  Used by tests/ (parity pins, golden-vector
// generation) and by bench.py's cpu_baseline / --impl reference arm.
//
// Wrapped reference entry points:
//   volpot::SummationPlan ctor/apply/levels/expansion_order  (summation.hpp:34-55)
//   volpot::direct_sum                                       (summation.hpp:22-23)
//   volpot::bessel_k0                                        (kernel.hpp:11)
//   volpot::bessel_k1                                        (kernel.hpp:12)
//   volpot::set_thread_count                                 (common.hpp:44)
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "volpot/common.hpp"
#include "volpot/kernel.hpp"
#include "volpot/summation.hpp"

namespace {
thread_local std::string g_err;

std::vector<volpot::Vec2> to_vec2(const double* xy, int64_t n) {
    std::vector<volpot::Vec2> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[size_t(i)] = {xy[2 * i], xy[2 * i + 1]};
    return v;
}

// 0 ok, 1 invalid_argument, 3 domain_error, 9 other
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
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { volpot::set_thread_count(n); }
int ref_thread_count() { return volpot::thread_count(); }

int ref_plan_create(int family, double lambda, const double* src_xy, int64_t ns,
                    const double* tgt_xy, int64_t nt, double eps, void** out) {
    return guarded([&] {
        volpot::Kernel k = volpot::make_kernel(
            family == 0 ? volpot::KernelFamily::Laplace
                        : volpot::KernelFamily::ModifiedHelmholtz,
            lambda);
        *out = new volpot::SummationPlan(k, to_vec2(src_xy, ns),
                                         to_vec2(tgt_xy, nt), eps);
    });
}

int ref_plan_apply(void* plan, const double* q, int64_t nq, double* out) {
    return guarded([&] {
        auto* p = static_cast<volpot::SummationPlan*>(plan);
        std::vector<double> qv(q, q + nq);
        std::vector<double> r = p->apply(qv);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

int ref_plan_levels(void* plan) {
    return static_cast<volpot::SummationPlan*>(plan)->levels();
}
int ref_plan_order(void* plan) {
    return static_cast<volpot::SummationPlan*>(plan)->expansion_order();
}
void ref_plan_destroy(void* plan) {
    delete static_cast<volpot::SummationPlan*>(plan);
}

int ref_direct_sum(int family, double lambda, const double* src_xy,
                   const double* q, int64_t ns, const double* tgt_xy,
                   int64_t nt, double* out) {
    return guarded([&] {
        volpot::Kernel k = volpot::make_kernel(
            family == 0 ? volpot::KernelFamily::Laplace
                        : volpot::KernelFamily::ModifiedHelmholtz,
            lambda);
        volpot::SourceSet s{to_vec2(src_xy, ns), std::vector<double>(q, q + ns)};
        std::vector<double> r = volpot::direct_sum(k, s, to_vec2(tgt_xy, nt));
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

int ref_bessel_k0(const double* x, int64_t n, double* out) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i) out[i] = volpot::bessel_k0(x[i]);
    });
}

int ref_bessel_k1(const double* x, int64_t n, double* out) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i) out[i] = volpot::bessel_k1(x[i]);
    });
}

}  // extern "C"
