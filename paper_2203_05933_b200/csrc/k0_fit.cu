// k0_fit.cu -- host construction of the K0 Chebyshev table used by
// k0_large() (k0.cuh).  The reference fits g(x) = K0(x) e^x sqrt(x) by
// 25-point Chebyshev interpolation on the dyadic intervals [2,4] .. [512,1024]
// from long-double quadrature of the integral representation
// K0(x) = int_0^inf exp(-x cosh t) dt (kernel.cpp:51-163).  This is an
// independent implementation of the same construction: Gauss-Legendre
// nodes by Newton iteration, composite panels doubled to convergence.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>
#include <vector>

#include "k0.cuh"

namespace vpg {
namespace {

struct GL {
    std::vector<long double> x, w;
    explicit GL(int n) : x(size_t(n)), w(size_t(n)) {
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int i = 0; i < n; ++i) {
            long double z = std::cos(pi * (i + 0.75L) / (n + 0.5L));
            long double dp = 0;
            for (int it = 0; it < 100; ++it) {
                long double p0 = 1, p1 = z;
                for (int k = 2; k <= n; ++k) {
                    const long double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (z * p1 - p0) / (z * z - 1);
                const long double dz = p1 / dp;
                z -= dz;
                if (std::fabs(dz) < 1e-21L) break;
            }
            x[size_t(i)] = z;
            w[size_t(i)] = 2 / ((1 - z * z) * dp * dp);
        }
    }
};

// e^x K0(x) for x >= 2 (e^x K1(x) with order1: integrand times cosh t,
// kernel.cpp:57-91).
long double scaled_k0(long double x, const GL& g, bool order1 = false) {
    const long double T = std::acosh(1.0L + 64.0L / x);  // integrand ~ e^-64
    long double prev = 0;
    for (int panels = 4; panels <= 4096; panels *= 2) {
        const long double h = T / panels;
        long double sum = 0;
        for (int p = 0; p < panels; ++p)
            for (size_t i = 0; i < g.x.size(); ++i) {
                const long double t = h * (p + 0.5L * (g.x[i] + 1));
                const long double ch = std::cosh(t);
                sum += g.w[i] * std::exp(-x * (ch - 1)) * (order1 ? ch : 1.0L);
            }
        sum *= 0.5L * h;
        if (panels > 4 && std::fabs(sum - prev) <= 1e-20L * sum) return sum;
        prev = sum;
    }
    return prev;
}

// The fits' node values g(x_j) are independent: evaluate them on the host's
// cores (each value is the same long-double computation, so the tables do not
// depend on the thread count).
template <typename F>
void parallel_nodes(int n, F&& f) {
    const int nt = std::max(1, std::min(n, int(std::thread::hardware_concurrency())));
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (int i = next++; i < n; i = next++) f(i);
        });
    for (auto& x : th) x.join();
}

}  // namespace

void k0_fit_host(double* out) {
    const GL g(20);
    const long double pi = 3.141592653589793238462643383279502884L;
    const int N = kK0Coeffs;
    std::vector<long double> fv(size_t(kK0Intervals) * N);
    parallel_nodes(kK0Intervals * N, [&](int e) {
        const int iv = e / N, j = e % N;
        const long double lo = std::ldexp(1.0L, iv + 1), hi = 2 * lo;
        const long double th = pi * (j + 0.5L) / N;
        const long double xj = 0.5L * (lo + hi) + 0.5L * (hi - lo) * std::cos(th);
        fv[size_t(e)] = scaled_k0(xj, g) * std::sqrt(xj);
    });
    for (int iv = 0; iv < kK0Intervals; ++iv) {
        const long double* f = fv.data() + size_t(iv) * N;
        for (int k = 0; k < N; ++k) {
            long double s = 0;
            for (int j = 0; j < N; ++j) s += f[j] * std::cos(k * pi * (j + 0.5L) / N);
            out[iv * N + k] = double(2 * s / N);
        }
    }
}

// The K1 fit of the reference (kernel.cpp:93-149 with order1).
void k1_fit_host(double* out) {
    const GL g(20);
    const long double pi = 3.141592653589793238462643383279502884L;
    const int N = kK0Coeffs;
    std::vector<long double> fv(size_t(kK0Intervals) * N);
    parallel_nodes(kK0Intervals * N, [&](int e) {
        const int iv = e / N, j = e % N;
        const long double lo = std::ldexp(1.0L, iv + 1), hi = 2 * lo;
        const long double th = pi * (j + 0.5L) / N;
        const long double xj = 0.5L * (lo + hi) + 0.5L * (hi - lo) * std::cos(th);
        fv[size_t(e)] = scaled_k0(xj, g, true) * std::sqrt(xj);
    });
    for (int iv = 0; iv < kK0Intervals; ++iv) {
        const long double* f = fv.data() + size_t(iv) * N;
        for (int k = 0; k < N; ++k) {
            long double s = 0;
            for (int j = 0; j < N; ++j) s += f[j] * std::cos(k * pi * (j + 0.5L) / N);
            out[iv * N + k] = double(2 * s / N);
        }
    }
}

// Quarter-octave fit for the treecode's hot loop (k0_fast, k0.cuh):
// intervals [2 * 2^(i/4), 2 * 2^((i+1)/4)], i = 0..kK0FastIntervals-1, each
// with kK0FastCoeffs Chebyshev coefficients of g(x) = K0(x) e^x sqrt(x)
// plus the map u = x * a + b onto [-1, 1]; record stride kK0FastStride.
void k0_fit_fast_host(double* out) {
    const GL g(20);
    const long double pi = 3.141592653589793238462643383279502884L;
    const int N = kK0FastCoeffs;
    std::vector<long double> fv(size_t(kK0FastIntervals) * N);
    parallel_nodes(kK0FastIntervals * N, [&](int e) {
        const int iv = e / N, j = e % N;
        const long double lo = 2.0L * std::pow(2.0L, iv / 4.0L), hi = 2.0L * std::pow(2.0L, (iv + 1) / 4.0L);
        const long double th = pi * (j + 0.5L) / N;
        const long double xj = 0.5L * (lo + hi) + 0.5L * (hi - lo) * std::cos(th);
        fv[size_t(e)] = scaled_k0(xj, g) * std::sqrt(xj);
    });
    for (int iv = 0; iv < kK0FastIntervals; ++iv) {
        const long double lo = 2.0L * std::pow(2.0L, iv / 4.0L), hi = 2.0L * std::pow(2.0L, (iv + 1) / 4.0L);
        const long double* f = fv.data() + size_t(iv) * N;
        double* rec = out + iv * kK0FastStride;
        for (int k = 0; k < N; ++k) {
            long double s = 0;
            for (int j = 0; j < N; ++j) s += f[j] * std::cos(k * pi * (j + 0.5L) / N);
            rec[k] = double(2 * s / N);
        }
        rec[N] = double(2.0L / (hi - lo));
        rec[N + 1] = double(-(hi + lo) / (hi - lo));
    }
}

}  // namespace vpg
