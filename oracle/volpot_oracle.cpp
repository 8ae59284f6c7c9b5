// volpot_oracle.cpp -- CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see volpot_oracle.h).  This is the checker the
// CUDA product path is compared against; it is never the thing measured or
// shipped.  Arithmetic mirrors the reference expression by expression (same
// operand order, same loop order) so that the FMM restatement reproduces
// oracle/_ref outputs; tests/test_oracle_pins.py states how closely.
#include "volpot_oracle.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numbers>
#include <vector>

#include <thread>

namespace {

// Worker pool for the checker: an atomic index counter over [0, n); each
// index writes only its own outputs, so results do not depend on threading
// (the reference promise, summation.hpp:32-33).
int g_threads = 0;
int nthreads_now() {
    if (g_threads > 0) return g_threads;
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? int(hc) : 1;
}
template <typename F>
void pfor(int64_t n, F&& fn) {
    const int nt = int(std::min<int64_t>(nthreads_now(), n));
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<int64_t> next(0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (;;) {
                const int64_t i0 = next.fetch_add(16);
                if (i0 >= n) break;
                for (int64_t i = i0; i < std::min(n, i0 + 16); ++i) fn(i);
            }
        });
    for (auto& th : pool) th.join();
}

constexpr double kOneOverTwoPi = 0.15915494309189533577;  // summation.cpp:15

struct C2 {
    double re = 0.0, im = 0.0;
};
// summation.cpp:24-41 (plain complex forms, no NaN recovery)
inline C2 cadd(C2 a, C2 b) { return {a.re + b.re, a.im + b.im}; }
inline C2 cmul(C2 a, C2 b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
inline C2 cscale(double s, C2 a) { return {s * a.re, s * a.im}; }
inline C2 cinv(C2 a) {
    const double d = a.re * a.re + a.im * a.im;
    return {a.re / d, -a.im / d};
}
inline C2 clog(C2 a) {
    return {0.5 * std::log(a.re * a.re + a.im * a.im), std::atan2(a.im, a.re)};
}

// summation.cpp:45-62
inline uint32_t interleave(uint32_t v) {
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
inline uint32_t morton(uint32_t ix, uint32_t iy) {
    return interleave(ix) | (interleave(iy) << 1);
}
inline uint32_t deinterleave(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0F0F0F0Fu;
    v = (v | (v >> 4)) & 0x00FF00FFu;
    v = (v | (v >> 8)) & 0x0000FFFFu;
    return v;
}

inline int64_t level_base(int l) { return ((int64_t(1) << (2 * l)) - 1) / 3; }

struct OTree {
    int L = 0;
    double x0 = 0, y0 = 0, side = 1;
    std::vector<int32_t> soff, sids, toff, tids;
    std::vector<int32_t> scnt, tcnt;  // concatenated levels
    double bside(int l) const { return side / static_cast<double>(1 << l); }
    // summation.cpp:74-78
    void center(int l, uint32_t id, double& cx, double& cy) const {
        const double s = bside(l);
        cx = x0 + (deinterleave(id) + 0.5) * s;
        cy = y0 + (deinterleave(id >> 1) + 0.5) * s;
    }
    int32_t sc(int l, int64_t b) const { return scnt[size_t(level_base(l) + b)]; }
    int32_t tc(int l, int64_t b) const { return tcnt[size_t(level_base(l) + b)]; }
};

// kernel.cpp:12-49 restated
constexpr double kGamma = 0.57721566490153286061;
double series_k0(double x) {
    const double t = 0.25 * x * x;
    double term = 1.0, i0 = 1.0, acc = 0.0, harm = 0.0;
    for (int k = 1; k < 40; ++k) {
        term *= t / (static_cast<double>(k) * k);
        harm += 1.0 / k;
        i0 += term;
        acc += term * harm;
        if (term < 1e-19 * i0) break;
    }
    return -(std::log(0.5 * x) + kGamma) * i0 + acc;
}

// kernel.cpp:33-49 restated: K1 = (ln(x/2) + gamma) I1 + 1/x - (x/4) sum,
// I1 = (x/2) sum_k c_k, c_k = q^k / (k! (k+1)!), the sum weighted by
// H_k + H_{k+1}.
double series_k1(double x) {
    const double t = 0.25 * x * x;
    double c = 1.0, i1s = 1.0, acc = 1.0, h0 = 0.0, h1 = 1.0;
    for (int k = 1; k < 40; ++k) {
        c *= t / (static_cast<double>(k) * (k + 1));
        h0 += 1.0 / k;
        h1 += 1.0 / (k + 1);
        i1s += c;
        acc += (h0 + h1) * c;
        if (c < 1e-19 * i1s) break;
    }
    const double i1 = 0.5 * x * i1s;
    return (std::log(0.5 * x) + kGamma) * i1 + 1.0 / x - 0.25 * x * acc;
}

// kernel.cpp:57-91: e^x K0(x) (e^x K1(x) with order1) by composite 10-point Gauss-Legendre on the
// truncated integral representation, doubling panels until converged.
long double scaled_k0_integral(long double x, bool order1 = false) {
    static const long double nodes[10] = {
        -0.9739065285171717L, -0.8650633666889845L, -0.6794095682990244L,
        -0.4333953941292472L, -0.1488743389816312L, 0.1488743389816312L,
        0.4333953941292472L,  0.6794095682990244L,  0.8650633666889845L,
        0.9739065285171717L};
    static const long double wts[10] = {
        0.0666713443086881L, 0.1494513491505806L, 0.2190863625159820L,
        0.2692667193099963L, 0.2955242247147529L, 0.2955242247147529L,
        0.2692667193099963L, 0.2190863625159820L, 0.1494513491505806L,
        0.0666713443086881L};
    const long double arg = (x + 62.0L) / x;
    const long double tmax = std::log(arg + std::sqrt(arg * arg - 1.0L));
    long double last = 0.0L;
    for (int panels = 8; panels <= 1024; panels *= 2) {
        long double s = 0.0L;
        const long double hp = tmax / panels;
        for (int p = 0; p < panels; ++p) {
            const long double a = p * hp;
            for (int i = 0; i < 10; ++i) {
                const long double t = a + 0.5L * hp * (nodes[i] + 1.0L);
                const long double ch = std::cosh(t);
                long double v = std::exp(-x * (ch - 1.0L));
                if (order1) v *= ch;
                s += wts[i] * v;
            }
        }
        s *= 0.5L * hp;
        if (panels > 8 && std::fabs(s - last) <= 1e-20L * std::fabs(s)) return s;
        last = s;
    }
    return last;
}

// kernel.cpp:93-149: 9 dyadic intervals [2,4]..[512,1024], 25 coefficients
// (order1: the K1 fit, kernel.cpp:123-124)
struct K0Fit {
    static constexpr int NI = 9, NC = 25;
    double c[NI][NC];
    explicit K0Fit(bool order1 = false) {
        for (int iv = 0; iv < NI; ++iv) {
            const long double a = std::pow(2.0L, iv + 1), b = 2.0L * a;
            long double fv[NC];
            for (int j = 0; j < NC; ++j) {
                const long double th = std::numbers::pi_v<long double> * (j + 0.5L) / NC;
                const long double xj = 0.5L * (a + b) + 0.5L * (b - a) * std::cos(th);
                fv[j] = scaled_k0_integral(xj, order1) * std::sqrt(xj);
            }
            for (int k = 0; k < NC; ++k) {
                long double s = 0.0L;
                for (int j = 0; j < NC; ++j) {
                    const long double th = std::numbers::pi_v<long double> * (j + 0.5L) / NC;
                    s += fv[j] * std::cos(k * th);
                }
                c[iv][k] = static_cast<double>(2.0L * s / NC);
            }
        }
    }
    double eval(double x) const {
        int iv = 0;
        double lo = 2.0;
        while (iv + 1 < NI && x > 2.0 * lo) {
            lo *= 2.0;
            ++iv;
        }
        const double hi = 2.0 * lo;
        const double u = (2.0 * x - (lo + hi)) / (hi - lo);
        double b1 = 0.0, b2 = 0.0;
        for (int k = NC - 1; k >= 1; --k) {
            const double b0 = 2.0 * u * b1 - b2 + c[iv][k];
            b2 = b1;
            b1 = b0;
        }
        return u * b1 - b2 + 0.5 * c[iv][0];
    }
};
const K0Fit& k0fit() {
    static const K0Fit f;
    return f;
}

double k0(double x) {
    if (!(x > 0.0)) return std::nan("");
    if (x <= 2.0) return series_k0(x);
    const double ex = std::exp(-x);
    if (ex == 0.0) return 0.0;
    return k0fit().eval(x) * ex / std::sqrt(x);
}

// kernel.cpp:174-179
double k1(double x) {
    if (!(x > 0.0)) return std::nan("");
    if (x <= 2.0) return series_k1(x);
    const double ex = std::exp(-x);
    if (ex == 0.0) return 0.0;
    static const K0Fit fit1(true);
    return fit1.eval(x) * ex / std::sqrt(x);
}

// kernel.cpp:181-186
inline double green_r2(int family, double lambda, double r2) {
    if (family == 0) return -0.25 / std::numbers::pi * std::log(r2);
    return 0.5 / std::numbers::pi * k0(lambda * std::sqrt(r2));
}

void bin(const double* pts, int64_t n, int L, double x0, double y0,
         double side, int32_t* off, int32_t* ids) {
    const int nb = 1 << L;
    const size_t nbox = size_t(nb) * nb;
    auto leaf = [&](int64_t j) {
        int ix = static_cast<int>((pts[2 * j] - x0) / side * nb);
        int iy = static_cast<int>((pts[2 * j + 1] - y0) / side * nb);
        ix = std::clamp(ix, 0, nb - 1);
        iy = std::clamp(iy, 0, nb - 1);
        return morton(uint32_t(ix), uint32_t(iy));
    };
    std::fill(off, off + nbox + 1, 0);
    for (int64_t j = 0; j < n; ++j) ++off[leaf(j) + 1];
    for (size_t b = 0; b < nbox; ++b) off[b + 1] += off[b];
    std::vector<int32_t> cur(off, off + nbox);
    for (int64_t j = 0; j < n; ++j) ids[cur[leaf(j)]++] = static_cast<int32_t>(j);
}

void levels_count(int L, const int32_t* off, int32_t* cnt) {
    const int64_t nl = int64_t(1) << (2 * L);
    int32_t* leaf = cnt + level_base(L);
    for (int64_t b = 0; b < nl; ++b) leaf[b] = off[b + 1] - off[b];
    for (int l = L - 1; l >= 0; --l) {
        int32_t* c = cnt + level_base(l);
        const int32_t* f = cnt + level_base(l + 1);
        for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
            c[b] = 0;
            for (int k = 0; k < 4; ++k) c[b] += f[(b << 2) | k];
        }
    }
}

OTree make_tree(const double* src, int64_t ns, const double* tgt, int64_t nt,
                const vo_params& pr) {
    OTree t;
    t.L = pr.levels;
    t.x0 = pr.x0;
    t.y0 = pr.y0;
    t.side = pr.side;
    const size_t nbox = size_t(1) << (2 * t.L);
    t.soff.resize(nbox + 1);
    t.toff.resize(nbox + 1);
    t.sids.resize(size_t(ns));
    t.tids.resize(size_t(nt));
    bin(src, ns, t.L, t.x0, t.y0, t.side, t.soff.data(), t.sids.data());
    bin(tgt, nt, t.L, t.x0, t.y0, t.side, t.toff.data(), t.tids.data());
    t.scnt.resize(size_t(level_base(t.L + 1)));
    t.tcnt.resize(size_t(level_base(t.L + 1)));
    levels_count(t.L, t.soff.data(), t.scnt.data());
    levels_count(t.L, t.toff.data(), t.tcnt.data());
    return t;
}

// summation.cpp:135-222 restated
struct LapOps {
    int P = 0;
    std::array<std::vector<C2>, 4> up, down;
    std::array<std::vector<C2>, 49> xl;
};

int order_for(double eps) {
    return std::clamp(
        static_cast<int>(std::ceil(std::log(1.0 / eps) / std::log(1.83))) + 4,
        10, 60);
}

LapOps lap_ops(double eps) {
    LapOps o;
    o.P = order_for(eps);
    const int P = o.P, n = P + 1, nb = 2 * P + 1;
    std::vector<double> bn(size_t(nb) * nb, 0.0);
    auto B = [&](int i, int j) -> double& { return bn[size_t(i) * nb + j]; };
    for (int i = 0; i <= 2 * P; ++i) {
        B(i, 0) = 1.0;
        for (int j = 1; j <= i; ++j) B(i, j) = B(i - 1, j - 1) + (j <= i - 1 ? B(i - 1, j) : 0.0);
    }
    for (int c = 0; c < 4; ++c) {
        const C2 t{(c & 1) ? 0.25 : -0.25, (c & 2) ? 0.25 : -0.25};
        std::vector<C2> tp(size_t(2 * P + 1));
        tp[0] = {1.0, 0.0};
        for (int j = 1; j <= 2 * P; ++j) tp[size_t(j)] = cmul(tp[size_t(j - 1)], t);
        auto& U = o.up[size_t(c)];
        U.assign(size_t(n) * n, C2{});
        U[0] = {1.0, 0.0};
        std::vector<double> sig(static_cast<size_t>(n));
        double s = 1.0;
        for (int k = 0; k <= P; ++k, s *= 0.5) sig[size_t(k)] = s;
        for (int l = 1; l <= P; ++l) {
            U[size_t(l) * n] = cscale(-1.0 / l, tp[size_t(l)]);
            for (int k = 1; k <= l; ++k)
                U[size_t(l) * n + k] = cscale(sig[size_t(k)] * B(l - 1, k - 1), tp[size_t(l - k)]);
        }
        auto& D = o.down[size_t(c)];
        D.assign(size_t(n) * n, C2{});
        double h = 1.0;
        for (int m = 0; m <= P; ++m, h *= 0.5)
            for (int l = m; l <= P; ++l)
                D[size_t(m) * n + l] = cscale(h * B(l, m), tp[size_t(l - m)]);
    }
    for (int dy = -3; dy <= 3; ++dy)
        for (int dx = -3; dx <= 3; ++dx) {
            if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
            auto& M = o.xl[size_t((dx + 3) + 7 * (dy + 3))];
            M.assign(size_t(n) * n, C2{});
            const C2 d{double(dx), double(dy)};
            const C2 di = cinv(d);
            std::vector<C2> dp(size_t(2 * P + 1));
            dp[0] = {1.0, 0.0};
            for (int j = 1; j <= 2 * P; ++j) dp[size_t(j)] = cmul(dp[size_t(j - 1)], di);
            M[0] = clog(C2{-d.re, -d.im});
            for (int k = 1; k <= P; ++k) M[size_t(k)] = cscale(k % 2 ? -1.0 : 1.0, dp[size_t(k)]);
            for (int l = 1; l <= P; ++l) {
                M[size_t(l) * n] = cscale(-1.0 / l, dp[size_t(l)]);
                for (int k = 1; k <= P; ++k)
                    M[size_t(l) * n + k] =
                        cscale((k % 2 ? -1.0 : 1.0) * B(l + k - 1, k - 1), dp[size_t(l + k)]);
            }
        }
    return o;
}

// summation.cpp:141-148
inline void mv_acc(const std::vector<C2>& M, const C2* x, C2* y, int n) {
    for (int r = 0; r < n; ++r) {
        const C2* row = M.data() + size_t(r) * n;
        C2 acc;
        for (int c = 0; c < n; ++c) acc = cadd(acc, cmul(row[c], x[c]));
        y[r] = cadd(y[r], acc);
    }
}

// summation.cpp:224-348 restated
void lap_apply(const OTree& tr, const LapOps& o, const double* sp,
               const double* q, const double* tp, double* out) {
    const int L = tr.L, P = o.P, n = P + 1;
    std::vector<double> invk(size_t(n), 0.0);
    for (int k = 1; k <= P; ++k) invk[size_t(k)] = 1.0 / k;
    std::vector<std::vector<C2>> mult(size_t(L + 1)), loc(size_t(L + 1));
    for (int l = 2; l <= L; ++l) {
        mult[size_t(l)].assign((size_t(1) << (2 * l)) * n, C2{});
        loc[size_t(l)].assign((size_t(1) << (2 * l)) * n, C2{});
    }
    const int64_t nleaf = int64_t(1) << (2 * L);
    pfor(nleaf, [&](int64_t b) {
        if (tr.sc(L, b) == 0) return;
        double cx, cy;
        tr.center(L, uint32_t(b), cx, cy);
        const double inv_s = 1.0 / tr.bside(L);
        C2* mb = mult[size_t(L)].data() + size_t(b) * n;
        for (int e = tr.soff[size_t(b)]; e < tr.soff[size_t(b) + 1]; ++e) {
            const int j = tr.sids[size_t(e)];
            const C2 w{(sp[2 * j] - cx) * inv_s, (sp[2 * j + 1] - cy) * inv_s};
            const double qj = q[j];
            mb[0].re += qj;
            C2 pw{qj, 0.0};
            for (int k = 1; k <= P; ++k) {
                pw = cmul(pw, w);
                mb[k] = cadd(mb[k], cscale(-invk[size_t(k)], pw));
            }
        }
    });
    for (int l = L - 1; l >= 2; --l) {
        pfor((int64_t(1) << (2 * l)), [&](int64_t b) {
            if (tr.sc(l, b) == 0) return;
            C2* mb = mult[size_t(l)].data() + size_t(b) * n;
            for (int c = 0; c < 4; ++c) {
                const size_t cid = (size_t(b) << 2) | size_t(c);
                if (tr.sc(l + 1, int64_t(cid)) == 0) continue;
                mv_acc(o.up[size_t(c)], mult[size_t(l + 1)].data() + cid * n, mb, n);
            }
        });
    }
    for (int l = 2; l <= L; ++l) {
        const int nb = 1 << l;
        const double logs = std::log(tr.bside(l));
        pfor((int64_t(1) << (2 * l)), [&](int64_t b) {
            if (tr.tc(l, b) == 0) return;
            const int ix = int(deinterleave(uint32_t(b)));
            const int iy = int(deinterleave(uint32_t(b) >> 1));
            C2* ab = loc[size_t(l)].data() + size_t(b) * n;
            double qsum = 0.0;
            const int px = ix >> 1, py = iy >> 1;
            for (int qy = py - 1; qy <= py + 1; ++qy) {
                if (qy < 0 || qy > (nb >> 1) - 1) continue;
                for (int qx = px - 1; qx <= px + 1; ++qx) {
                    if (qx < 0 || qx > (nb >> 1) - 1) continue;
                    for (int c = 0; c < 4; ++c) {
                        const int jx = 2 * qx + (c & 1), jy = 2 * qy + ((c & 2) >> 1);
                        const int dx = jx - ix, dy = jy - iy;
                        if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
                        const uint32_t sid = morton(uint32_t(jx), uint32_t(jy));
                        if (tr.sc(l, sid) == 0) continue;
                        const C2* mb = mult[size_t(l)].data() + size_t(sid) * n;
                        mv_acc(o.xl[size_t((dx + 3) + 7 * (dy + 3))], mb, ab, n);
                        qsum += mb[0].re;
                    }
                }
            }
            ab[0].re += qsum * logs;
        });
    }
    for (int l = 2; l < L; ++l) {
        pfor((int64_t(1) << (2 * (l + 1))), [&](int64_t cid) {
            if (tr.tc(l + 1, cid) == 0) return;
            const size_t pid = size_t(cid) >> 2;
            mv_acc(o.down[size_t(cid & 3)], loc[size_t(l)].data() + pid * n,
                   loc[size_t(l + 1)].data() + size_t(cid) * n, n);
        });
    }
    const int nb = 1 << L;
    pfor(nleaf, [&](int64_t b) {
        if (tr.tc(L, b) == 0) return;
        double cx, cy;
        tr.center(L, uint32_t(b), cx, cy);
        const double inv_s = 1.0 / tr.bside(L);
        const C2* ab = loc[size_t(L)].data() + size_t(b) * n;
        const int ix = int(deinterleave(uint32_t(b)));
        const int iy = int(deinterleave(uint32_t(b) >> 1));
        for (int e = tr.toff[size_t(b)]; e < tr.toff[size_t(b) + 1]; ++e) {
            const int i = tr.tids[size_t(e)];
            const double tx = tp[2 * i], ty = tp[2 * i + 1];
            const C2 u{(tx - cx) * inv_s, (ty - cy) * inv_s};
            C2 val = ab[P];
            for (int l = P - 1; l >= 0; --l) val = cadd(cmul(val, u), ab[l]);
            double pot = -kOneOverTwoPi * val.re;
            for (int jy = std::max(0, iy - 1); jy <= std::min(nb - 1, iy + 1); ++jy)
                for (int jx = std::max(0, ix - 1); jx <= std::min(nb - 1, ix + 1); ++jx) {
                    const uint32_t sid = morton(uint32_t(jx), uint32_t(jy));
                    for (int f = tr.soff[sid]; f < tr.soff[sid + 1]; ++f) {
                        const int j = tr.sids[size_t(f)];
                        const double dx = tx - sp[2 * j], dy = ty - sp[2 * j + 1];
                        const double r2 = dx * dx + dy * dy;
                        if (r2 == 0.0) continue;
                        pot += q[j] * green_r2(0, 0.0, r2);
                    }
                }
            out[i] = pot;
        }
    });
}

// summation.cpp:356-414 restated
struct HLevel {
    int m = 0;
    std::vector<double> x, bw;
};
struct HOps {
    int min_level = 2;
    double skip_x = 40.0;
    std::vector<HLevel> lv;
};

HOps helm_ops(double eps, double lambda, const OTree& tr) {
    HOps o;
    o.min_level = 2;
    while (o.min_level <= tr.L && lambda * tr.bside(o.min_level) > 5.0) ++o.min_level;
    o.skip_x = std::log(1.0 / eps) + 12.0;
    const int base = 8 + std::max(0, static_cast<int>(std::ceil(std::log(1.15e-8 / eps) / 1.97)));
    o.lv.resize(size_t(tr.L + 1));
    for (int l = o.min_level; l <= tr.L; ++l) {
        const double ls = lambda * tr.bside(l);
        const int bump = ls <= 0.5 ? 0 : (ls <= 2.0 ? 2 : 5);
        HLevel& v = o.lv[size_t(l)];
        v.m = std::min(base + bump, 26);
        v.x.resize(size_t(v.m));
        v.bw.resize(size_t(v.m));
        for (int a = 0; a < v.m; ++a) {
            const double th = (2 * a + 1) * 3.14159265358979323846 / (2 * v.m);
            v.x[size_t(a)] = std::cos(th);
            v.bw[size_t(a)] = (a % 2 ? -1.0 : 1.0) * std::sin(th);
        }
    }
    return o;
}

void bary(const HLevel& v, double x, double* w) {
    const int m = v.m;
    for (int a = 0; a < m; ++a)
        if (x == v.x[size_t(a)]) {
            std::fill(w, w + m, 0.0);
            w[a] = 1.0;
            return;
        }
    double s = 0.0;
    for (int a = 0; a < m; ++a) {
        w[a] = v.bw[size_t(a)] / (x - v.x[size_t(a)]);
        s += w[a];
    }
    const double inv = 1.0 / s;
    for (int a = 0; a < m; ++a) w[a] *= inv;
}

// summation.cpp:416-497 restated
void helm_apply(const OTree& tr, const HOps& o, double lambda, const double* sp,
                const double* q, const double* tp, int64_t nt, double* out) {
    const int L = tr.L;
    std::vector<std::vector<double>> W(size_t(L + 1));
    for (int l = o.min_level; l <= L; ++l) {
        const HLevel& v = o.lv[size_t(l)];
        const int m = v.m, mm = m * m;
        W[size_t(l)].assign((size_t(1) << (2 * l)) * mm, 0.0);
        const int shift = 2 * (L - l);
        pfor((int64_t(1) << (2 * l)), [&](int64_t b) {
            if (tr.sc(l, b) == 0) return;
            double cx, cy;
            tr.center(l, uint32_t(b), cx, cy);
            const double inv_h = 2.0 / tr.bside(l);
            double* wb = W[size_t(l)].data() + size_t(b) * mm;
            double lx[32], ly[32];
            const int e0 = tr.soff[size_t(b) << shift];
            const int e1 = tr.soff[(size_t(b) + 1) << shift];
            for (int e = e0; e < e1; ++e) {
                const int j = tr.sids[size_t(e)];
                bary(v, (sp[2 * j] - cx) * inv_h, lx);
                bary(v, (sp[2 * j + 1] - cy) * inv_h, ly);
                const double qj = q[j];
                for (int a = 0; a < m; ++a) {
                    const double f = qj * lx[a];
                    for (int bb = 0; bb < m; ++bb) wb[a * m + bb] += f * ly[bb];
                }
            }
        });
    }
    pfor(nt, [&](int64_t i) {
        const double tx = tp[2 * i], ty = tp[2 * i + 1];
        double pot = 0.0;
        uint64_t stack[128];
        int top = 0;
        stack[top++] = 0;
        while (top > 0) {
            const uint64_t ent = stack[--top];
            const int l = int(ent >> 32);
            const uint32_t id = uint32_t(ent);
            if (tr.sc(l, id) == 0) continue;
            const double s = tr.bside(l);
            double cx, cy;
            tr.center(l, id, cx, cy);
            const double dx = tx - cx, dy = ty - cy;
            const double d2 = dx * dx + dy * dy;
            const double rbox = s * 0.7071067811865476;
            if (lambda * (std::sqrt(d2) - rbox) > o.skip_x) continue;
            if (l >= o.min_level && d2 >= 4.5 * s * s) {
                const HLevel& v = o.lv[size_t(l)];
                const int m = v.m;
                const double* wb = W[size_t(l)].data() + size_t(id) * m * m;
                const double h = 0.5 * s;
                for (int a = 0; a < m; ++a) {
                    const double nx = cx + h * v.x[size_t(a)];
                    for (int bb = 0; bb < m; ++bb) {
                        const double ny = cy + h * v.x[size_t(bb)];
                        const double ex = tx - nx, ey = ty - ny;
                        pot += wb[a * m + bb] * green_r2(1, lambda, ex * ex + ey * ey);
                    }
                }
            } else if (l == L) {
                for (int f = tr.soff[id]; f < tr.soff[id + 1]; ++f) {
                    const int j = tr.sids[size_t(f)];
                    const double ex = tx - sp[2 * j], ey = ty - sp[2 * j + 1];
                    const double r2 = ex * ex + ey * ey;
                    if (r2 == 0.0) continue;
                    pot += q[j] * green_r2(1, lambda, r2);
                }
            } else {
                for (int cc = 0; cc < 4; ++cc)
                    stack[top++] = (uint64_t(l + 1) << 32) | ((uint64_t(id) << 2) | uint64_t(cc));
            }
        }
        out[i] = pot;
    });
}

struct ThreadScope {
    int saved;
    explicit ThreadScope(int n) : saved(g_threads) { g_threads = n; }
    ~ThreadScope() { g_threads = saved; }
};

}  // namespace

extern "C" {

int vo_plan_params(int family, double lambda, const double* src, int64_t ns,
                   const double* tgt, int64_t nt, double eps, vo_params* out) {
    vo_params p{};
    p.eps = std::clamp(eps, 1e-12, 1e-3);
    double xlo = 0, xhi = 0, ylo = 0, yhi = 0;
    bool first = true;
    for (int pass = 0; pass < 2; ++pass) {
        const double* pts = pass == 0 ? src : tgt;
        const int64_t n = pass == 0 ? ns : nt;
        for (int64_t i = 0; i < n; ++i) {
            const double x = pts[2 * i], y = pts[2 * i + 1];
            if (first) {
                xlo = xhi = x;
                ylo = yhi = y;
                first = false;
            } else {
                xlo = std::min(xlo, x);
                xhi = std::max(xhi, x);
                ylo = std::min(ylo, y);
                yhi = std::max(yhi, y);
            }
        }
    }
    const double side = std::max(xhi - xlo, yhi - ylo);
    p.direct = (side <= 0.0 || double(ns) * double(nt) <= 4e6) ? 1 : 0;
    if (!p.direct) {
        const double big = static_cast<double>(std::max(ns, nt));
        p.levels = std::clamp(
            static_cast<int>(std::ceil(std::log(big / 32.0) / std::log(4.0))), 2, 7);
        p.x0 = xlo;
        p.y0 = ylo;
        p.side = side * (1.0 + 1e-12);
        if (family == 0) {
            p.order = order_for(p.eps);
        } else {
            OTree t;
            t.L = p.levels;
            t.side = p.side;
            HOps h = helm_ops(p.eps, lambda, t);
            for (const HLevel& v : h.lv) p.order = std::max(p.order, v.m);
        }
    }
    *out = p;
    return 0;
}

void vo_bin_points(const double* pts, int64_t n, int levels, double x0,
                   double y0, double side, int32_t* off, int32_t* ids) {
    bin(pts, n, levels, x0, y0, side, off, ids);
}

void vo_count_levels(int levels, const int32_t* leaf_off, int32_t* cnt_all) {
    levels_count(levels, leaf_off, cnt_all);
}

int64_t vo_m2l_list(int levels, int l, const int32_t* scnt_all,
                    const int32_t* tcnt_all, int32_t* ntbox, int32_t* tbox,
                    int32_t* toff, int32_t* src, int32_t* oidx) {
    (void)levels;
    const int nb = 1 << l;
    const int32_t* sc = scnt_all + level_base(l);
    const int32_t* tc = tcnt_all + level_base(l);
    int64_t ne = 0;
    int32_t nt = 0;
    if (toff) toff[0] = 0;
    for (int64_t b = 0; b < (int64_t(1) << (2 * l)); ++b) {
        if (tc[b] == 0) continue;
        const int ix = int(deinterleave(uint32_t(b))), iy = int(deinterleave(uint32_t(b) >> 1));
        const int px = ix >> 1, py = iy >> 1;
        for (int qy = py - 1; qy <= py + 1; ++qy) {
            if (qy < 0 || qy > (nb >> 1) - 1) continue;
            for (int qx = px - 1; qx <= px + 1; ++qx) {
                if (qx < 0 || qx > (nb >> 1) - 1) continue;
                for (int c = 0; c < 4; ++c) {
                    const int jx = 2 * qx + (c & 1), jy = 2 * qy + ((c & 2) >> 1);
                    const int dx = jx - ix, dy = jy - iy;
                    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
                    const uint32_t sid = morton(uint32_t(jx), uint32_t(jy));
                    if (sc[sid] == 0) continue;
                    if (src) src[ne] = int32_t(sid);
                    if (oidx) oidx[ne] = (dx + 3) + 7 * (dy + 3);
                    ++ne;
                }
            }
        }
        if (tbox) tbox[nt] = int32_t(b);
        ++nt;
        if (toff) toff[nt] = int32_t(ne);
    }
    if (ntbox) *ntbox = nt;
    return ne;
}

int64_t vo_p2p_pairs(int L, const int32_t* soff, const int32_t* toff) {
    const int nb = 1 << L;
    int64_t total = 0;
    for (int64_t b = 0; b < (int64_t(1) << (2 * L)); ++b) {
        const int64_t ntb = toff[b + 1] - toff[b];
        if (ntb == 0) continue;
        const int ix = int(deinterleave(uint32_t(b))), iy = int(deinterleave(uint32_t(b) >> 1));
        int64_t nsrc = 0;
        for (int jy = std::max(0, iy - 1); jy <= std::min(nb - 1, iy + 1); ++jy)
            for (int jx = std::max(0, ix - 1); jx <= std::min(nb - 1, ix + 1); ++jx) {
                const uint32_t sid = morton(uint32_t(jx), uint32_t(jy));
                nsrc += soff[sid + 1] - soff[sid];
            }
        total += ntb * nsrc;
    }
    return total;
}

int vo_plan_sum(int family, double lambda, const double* src, const double* q,
                int64_t ns, const double* tgt, int64_t nt, double eps,
                double* out, int nthreads) {
    if (family != 0 && !(lambda > 0.0)) return 1;
    ThreadScope ts(nthreads);
    vo_params pr;
    vo_plan_params(family, lambda, src, ns, tgt, nt, eps, &pr);
    if (pr.direct) {
        pfor(nt, [&](int64_t i) {
            const double tx = tgt[2 * i], ty = tgt[2 * i + 1];
            double acc = 0.0;
            for (int64_t j = 0; j < ns; ++j) {
                const double dx = tx - src[2 * j], dy = ty - src[2 * j + 1];
                const double r2 = dx * dx + dy * dy;
                if (r2 == 0.0) continue;
                acc += q[j] * green_r2(family, lambda, r2);
            }
            out[i] = acc;
        });
        return 0;
    }
    const OTree tr = make_tree(src, ns, tgt, nt, pr);
    if (family == 0) {
        const LapOps o = lap_ops(pr.eps);
        lap_apply(tr, o, src, q, tgt, out);
    } else {
        const HOps o = helm_ops(pr.eps, lambda, tr);
        helm_apply(tr, o, lambda, src, q, tgt, nt, out);
    }
    return 0;
}

int vo_direct_sum(int family, double lambda, const double* src,
                  const double* q, int64_t ns, const double* tgt, int64_t nt,
                  double* out, int64_t* ci, int64_t* cj, int nthreads) {
    if (family != 0 && !(lambda > 0.0)) return 1;
    ThreadScope ts(nthreads);
    std::atomic<uint64_t> clash(~uint64_t(0));
    pfor(nt, [&](int64_t i) {
        const double tx = tgt[2 * i], ty = tgt[2 * i + 1];
        double acc = 0.0;
        bool hit = false;
        for (int64_t j = 0; j < ns; ++j) {
            const double dx = tx - src[2 * j], dy = ty - src[2 * j + 1];
            const double r2 = dx * dx + dy * dy;
            if (r2 == 0.0) {
                const uint64_t key = (uint64_t(i) << 32) | uint64_t(j);
                uint64_t cur = clash.load();
                while (key < cur && !clash.compare_exchange_weak(cur, key)) {
                }
                hit = true;
                break;
            }
            acc += q[j] * green_r2(family, lambda, r2);
        }
        out[i] = hit ? 0.0 : acc;
    });
    const uint64_t key = clash.load();
    if (key != ~uint64_t(0)) {
        if (ci) *ci = int64_t(key >> 32);
        if (cj) *cj = int64_t(key & 0xFFFFFFFFu);
        return 2;
    }
    return 0;
}

void vo_pairwise_sum_ld(int family, double lambda, const double* src,
                        const double* q, int64_t ns, const double* tgt,
                        int64_t nt, double* out, int nthreads) {
    ThreadScope ts(nthreads);
    const long double c = -0.25L / std::numbers::pi_v<long double>;
    pfor(nt, [&](int64_t i) {
        const long double tx = tgt[2 * i], ty = tgt[2 * i + 1];
        long double acc = 0.0L;
        for (int64_t j = 0; j < ns; ++j) {
            const long double dx = tx - src[2 * j], dy = ty - src[2 * j + 1];
            const long double r2 = dx * dx + dy * dy;
            if (r2 == 0.0L) continue;
            if (family == 0)
                acc += q[j] * (c * std::log(r2));
            else
                acc += static_cast<long double>(q[j]) *
                       green_r2(1, lambda, static_cast<double>(r2));
        }
        out[i] = static_cast<double>(acc);
    });
}

double vo_bessel_k0(double x) { return k0(x); }

double vo_radial_r2(int family, double lambda, double r2) {
    return green_r2(family, lambda, r2);
}

void vo_correction_apply(int64_t nt, const int32_t* blk_off,
                         const int32_t* blk_cell, const int32_t* blk_pool,
                         const int64_t* pool_off, const double* pool_vals,
                         const int32_t* node_off, const double* f, double* out,
                         int nthreads) {
    ThreadScope ts(nthreads);
    pfor(nt, [&](int64_t t) {
        double corr = 0;
        for (int k = blk_off[t]; k < blk_off[t + 1]; ++k) {
            const int64_t r0 = pool_off[blk_pool[k]], r1 = pool_off[blk_pool[k] + 1];
            const double* fc = f + node_off[blk_cell[k]];
            double dot = 0;
            for (int64_t e = r0; e < r1; ++e) dot += pool_vals[e] * fc[e - r0];
            corr += dot;
        }
        out[t] += corr;
    });
}

void vo_build_charges(int64_t ncell, const int32_t* cell_type,
                      const int32_t* node_off, const int32_t* src_off,
                      const double* over0, int np0, int nq0,
                      const double* over1, int np1, int nq1,
                      const double* src_wj, const double* f, double* charges, int nthreads) {
    ThreadScope ts(nthreads);
    pfor(ncell, [&](int64_t c) {  // potential.cpp:400 parallel_try over cells
        const bool t0 = cell_type[c] == 0;
        const double* O = t0 ? over0 : over1;
        const int np = t0 ? np0 : np1, nq = t0 ? nq0 : nq1;
        const double* fc = f + node_off[c];
        const int base = src_off[c];
        for (int s = 0; s < nq; ++s) {
            double v = 0;
            for (int i = 0; i < np; ++i) v += O[size_t(s) * np + i] * fc[i];
            charges[base + s] = src_wj[base + s] * v;
        }
    });
}


double vo_bessel_k1(double x) { return k1(x); }

// bie.cpp:112-135
void vo_trig_upsample(const double* f, int n, int factor, double* out) {
    constexpr double kTwoPi = 2.0 * std::numbers::pi;
    const int half = n / 2;
    std::vector<double> a(size_t(half) + 1, 0.0), b(size_t(half), 0.0);
    for (int m = 0; m <= half; ++m) {
        double ca = 0.0, cb = 0.0;
        for (int j = 0; j < n; ++j) {
            const double ang = kTwoPi * m * j / n;
            ca += f[j] * std::cos(ang);
            cb += f[j] * std::sin(ang);
        }
        a[size_t(m)] = 2.0 * ca / n;
        if (m >= 1 && m < half) b[size_t(m)] = 2.0 * cb / n;
    }
    a[0] *= 0.5;
    a[size_t(half)] *= 0.5;
    for (int j = 0; j < n * factor; ++j) {
        const double t = kTwoPi * j / (n * factor);
        double s = a[0] + a[size_t(half)] * std::cos(half * t);
        for (int m = 1; m < half; ++m) s += a[size_t(m)] * std::cos(m * t) + b[size_t(m)] * std::sin(m * t);
        out[j] = s;
    }
}

// bie.cpp:383-461 with dlp_entry (bie.cpp:43-50); kFineFactor 8, kFineReach
// 5, kCollarFraction 0.02 (bie.cpp:18-20)
int vo_layer_eval(int family, double lambda, const vo_curve* curves, int ncurves, int n_density,
                  int n_aux, const double* coeffs, int64_t ncoeffs, const double* tgt, int64_t nt,
                  int allow_close, double* out, int nthreads) {
    constexpr double kTwoPi = 2.0 * std::numbers::pi;
    constexpr int kFine = 8;
    constexpr double kReach = 5.0, kCollar = 0.02;
    if (ncoeffs != int64_t(n_density) + n_aux) return 1;
    g_threads = nthreads;
    std::vector<std::vector<double>> fine_phi(static_cast<size_t>(ncurves));
    for (int c = 0; c < ncurves; ++c) {
        const vo_curve& B = curves[c];
        fine_phi[size_t(c)].resize(size_t(B.n) * kFine);
        vo_trig_upsample(coeffs + B.offset, B.n, kFine, fine_phi[size_t(c)].data());
    }
    auto dlp = [&](double x0, double x1, const double* y, const double* ny, double speed) {
        const double d0 = y[0] - x0, d1 = y[1] - x1;
        const double r2 = d0 * d0 + d1 * d1;
        const double dn = d0 * ny[0] + d1 * ny[1];
        if (family == 0) return -dn / (kTwoPi * r2) * speed;
        const double r = std::sqrt(r2);
        return -(lambda / kTwoPi) * k1(lambda * r) * (dn / r) * speed;
    };
    std::atomic<int> reject{0};
    pfor(nt, [&](int64_t ti) {
        const double x0 = tgt[2 * ti], x1 = tgt[2 * ti + 1];
        double acc = 0.0;
        for (int c = 0; c < ncurves; ++c) {
            const vo_curve& B = curves[c];
            const double h = B.length / B.n;
            const double collar = allow_close ? 0.0 : kCollar * B.diam;
            double d2 = 1e300;
            for (int j = 0; j < B.n; ++j) {
                const double e0 = x0 - B.x[2 * j], e1 = x1 - B.x[2 * j + 1];
                d2 = std::min(d2, e0 * e0 + e1 * e1);
            }
            double d = std::sqrt(d2);
            bool fine = false;
            if (d - 0.75 * h <= std::max(collar, kReach * h)) {
                d2 = 1e300;
                for (int j = 0; j < B.n * kFine; ++j) {
                    const double e0 = x0 - B.fine_x[2 * j], e1 = x1 - B.fine_x[2 * j + 1];
                    d2 = std::min(d2, e0 * e0 + e1 * e1);
                }
                d = std::sqrt(d2);
                if (d == 0.0) {
                    reject.store(2);
                    return;
                }
                if (d < collar) {
                    int want = 0;
                    reject.compare_exchange_strong(want, 1);
                    return;
                }
                fine = d <= kReach * h;
            }
            if (fine) {
                const int nf = B.n * kFine;
                const double w = kTwoPi / nf;
                const double* phi = fine_phi[size_t(c)].data();
                for (int j = 0; j < nf; ++j)
                    acc += w * phi[j] * dlp(x0, x1, B.fine_x + 2 * j, B.fine_normal + 2 * j, B.fine_speed[j]);
            } else {
                const double w = kTwoPi / B.n;
                for (int j = 0; j < B.n; ++j)
                    acc += w * coeffs[B.offset + j] * dlp(x0, x1, B.x + 2 * j, B.normal + 2 * j, B.speed[j]);
            }
        }
        for (int k = 0; k < n_aux; ++k) {
            const double d0 = x0 - curves[k + 1].log_center[0], d1 = x1 - curves[k + 1].log_center[1];
            acc += coeffs[n_density + k] * (-std::log(std::sqrt(d0 * d0 + d1 * d1)) / kTwoPi);
        }
        out[ti] = acc;
    });
    const int r = reject.load();
    return r == 2 ? 2 : r == 1 ? 3 : 0;
}

}  // extern "C"
