// layer.cu -- double-layer potential evaluation at volume targets
// (eval_layer_potential, bie.cpp:383-468): u_H(x) = sum over curves of the
// trapezoidal Nystrom sum of phi_j dG(y_j, x)/dn(y_j) |gamma'| (2 pi / n),
// switching to the 8x trig-upsampled density and geometry within 5 node
// spacings of a curve, plus the log-completion terms of the holes.
//
// Layout (vpg_layer, uploaded once per boundary system): coarse and fine
// geometry of all curves concatenated as interleaved xy / normals and
// speeds; per-curve metadata (CurveDev).  Per eval (stream-ordered scratch):
//   1. ups_coef_kernel   a warp per (curve, m): the Fourier coefficients of
//                        the density (bie.cpp:115-127), lanes over j.
//   2. records_kernel    a thread per node: fine density by the
//                        zero-padded series (bie.cpp:128-134) and one 32-B
//                        record (y, B n) per coarse and fine node with
//                        B = -w phi speed / 2pi (Laplace) or
//                        -w phi speed lambda / 2pi (modified Helmholtz), so a
//                        pair costs dn / r^2 (dn K1(lambda r) / r).
//   3. coarse_kernel     two targets per thread, 256-record smem tiles: the
//                        coarse min distance and the coarse sum of every curve
//                        in one pass; targets whose coarse distance asks for
//                        the refined check (bie.cpp:414) are appended to the
//                        curve's fine list.
//   4. fine_kernel       two listed targets per thread over the curve's 8n fine
//                        records: refined distance, the reject rules
//                        (bie.cpp:417-425) and the fine sum.
//   5. finalize_kernel   out = per-curve values in curve order + aux logs.
// Every per-target sum runs in node order on one thread: results are
// run-to-run identical.  No CPU path.
#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "k0.cuh"
#include "plan.cuh"

struct vpg_layer;

namespace vpg {
namespace {

constexpr double kTwoPiL = 6.283185307179586476925286766559;  // bie.cpp:17
constexpr int kFineFactor = 8;      // bie.cpp:18
constexpr double kFineReach = 5.0;  // bie.cpp:19
constexpr double kCollarFraction = 0.02;  // bie.cpp:20
constexpr int kLayerTile = 256;  // records per smem tile
#ifndef VPG_LAYER_UNROLL
#define VPG_LAYER_UNROLL 4
#endif
constexpr int kLayerUnroll = VPG_LAYER_UNROLL;
#ifndef VPG_LAYER_CT
#define VPG_LAYER_CT 256
#endif
#ifndef VPG_LAYER_CTPT
#define VPG_LAYER_CTPT 1
#endif
#ifndef VPG_LAYER_FT
#define VPG_LAYER_FT 256
#endif
#ifndef VPG_LAYER_FTPT
#define VPG_LAYER_FTPT 1
#endif
constexpr int kCoarseThreads = VPG_LAYER_CT, kCoarseTPT = VPG_LAYER_CTPT;  // CTA size, targets per thread
constexpr int kFineThreads = VPG_LAYER_FT, kFineTPT = VPG_LAYER_FTPT;

struct CurveDev {
    int n, offset;
    int cbase, fbase;  // first coarse / fine node in the concatenated arrays
    int ubase;         // first Fourier coefficient slot (half + 1 per curve)
    int pad;
    double h, diam;    // length / n, node-set diameter
    double lcx, lcy;   // log_center
};

inline unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ int curve_of(const CurveDev* cv, int nc, int idx, int CurveDev::*base) {
    int c = 0;
    while (c + 1 < nc && cv[c + 1].*base <= idx) ++c;
    return c;
}

// bie.cpp:115-127: a[m] = 2/n sum f_j cos(2 pi m j / n), b likewise (m in
// [1, half)), a[0] and a[half] halved.  Angle as the reference forms it.
__global__ void ups_coef_kernel(const CurveDev* cv, int nc, int ncoef, const double* coeffs,
                                double2* ab) {
    const int w = int((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= ncoef) return;
    const int c = curve_of(cv, nc, w, &CurveDev::ubase);
    const CurveDev C = cv[c];
    const int m = w - C.ubase, n = C.n, half = n / 2;
    const double* f = coeffs + C.offset;
    double ca = 0.0, cb = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double ang = kTwoPiL * m * j / n;
        double sn, cs;
        sincos(ang, &sn, &cs);
        ca = fma(f[j], cs, ca);
        cb = fma(f[j], sn, cb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ca += __shfl_xor_sync(0xffffffffu, ca, o);
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
    }
    if (lane == 0) {
        double a = 2.0 * ca / n;
        const double b = (m >= 1 && m < half) ? 2.0 * cb / n : 0.0;
        if (m == 0 || m == half) a *= 0.5;
        ab[w] = make_double2(a, b);
    }
}

// One record per node: (y, B n).  Nodes [0, ncoarse) coarse, then fine.
template <int kFamily>
__global__ void records_kernel(const CurveDev* cv, int nc, int64_t ncoarse, int64_t nfine,
                               const double* coeffs, const double2* ab, const double2* x,
                               const double2* nrm, const double* speed, const double2* fx,
                               const double2* fnrm, const double* fspeed, double lambda,
                               double4* crec, double4* frec) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= ncoarse + nfine) return;
    const double kscale = kFamily == VPG_LAPLACE ? 1.0 : lambda;
    if (g < ncoarse) {
        const int c = curve_of(cv, nc, int(g), &CurveDev::cbase);
        const CurveDev C = cv[c];
        const int j = int(g) - C.cbase;
        const double w = kTwoPiL / C.n;
        const double B = -(w * coeffs[C.offset + j]) * speed[g] * kscale * (1.0 / kTwoPiL);
        const double2 y = x[g], nv = nrm[g];
        crec[g] = make_double4(y.x, y.y, B * nv.x, B * nv.y);
        return;
    }
    const int64_t gf = g - ncoarse;
    const int c = curve_of(cv, nc, int(gf), &CurveDev::fbase);
    const CurveDev C = cv[c];
    const int j = int(gf) - C.fbase;
    const int n = C.n, half = n / 2, nf = n * kFineFactor;
    const double2* a = ab + C.ubase;
    // bie.cpp:128-134, in the reference's term order
    const double t = kTwoPiL * j / nf;
    double s = a[0].x + a[half].x * cos(half * t);
    for (int m = 1; m < half; ++m) {
        double sn, cs;
        sincos(m * t, &sn, &cs);
        s += a[m].x * cs + a[m].y * sn;
    }
    const double w = kTwoPiL / nf;
    const double B = -(w * s) * fspeed[gf] * kscale * (1.0 / kTwoPiL);
    const double2 y = fx[gf], nv = fnrm[gf];
    frec[gf] = make_double4(y.x, y.y, B * nv.x, B * nv.y);
}

// Sum over records [r0, r1) for two targets per thread: min r^2 and the sum
// of B dn / r^2 (Laplace) or B dn K1(lambda r) / r (modified Helmholtz).
// Records are staged in kLayerTile-entry smem tiles by the whole CTA; each
// staged record serves both targets of a thread (two independent chains).
template <int kFamily>
__device__ __forceinline__ void pair_acc(const double4& r, double tx, double ty, double lambda,
                                         const double* k1tab, double& d2min, double& acc) {
    const double dx = r.x - tx, dy = r.y - ty;
    const double r2 = fma(dy, dy, dx * dx);
    d2min = fmin(d2min, r2);
    const double dn = fma(dy, r.w, dx * r.z);
    if (kFamily == VPG_LAPLACE) {
        acc = fma(dn, rcp_nr(r2), acc);
    } else {
        const double rr = sqrt(r2);
        acc = fma(dn * k1_dev(lambda * rr, k1tab), rcp_nr(rr), acc);
    }
}

template <int kFamily, int TPT>
__device__ __forceinline__ void tile_sum(const double4* rec, int r0, int r1, const double (&tx)[TPT],
                                         const double (&ty)[TPT], bool active, double lambda,
                                         const double* k1tab, double4* sm, double (&d2min)[TPT],
                                         double (&acc)[TPT]) {
    for (int b = r0; b < r1; b += kLayerTile) {
        const int cnt = min(kLayerTile, r1 - b);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) sm[i] = rec[b + i];
        __syncthreads();
        if (!active) continue;
#pragma unroll kLayerUnroll
        for (int k = 0; k < cnt; ++k) {
            const double4 r = sm[k];
#pragma unroll
            for (int u = 0; u < TPT; ++u) pair_acc<kFamily>(r, tx[u], ty[u], lambda, k1tab, d2min[u], acc[u]);
        }
    }
}

// Targets t + u * blockDim.x (u < TPT) of a TPT * blockDim.x tile per thread.
template <int kFamily, int TPT>
__global__ void __launch_bounds__(512)
coarse_kernel(const CurveDev* cv, int nc, const double4* crec, const double2* tgt, int64_t nt,
              int allow_close, double lambda, const double* k1tab, double* cval, int* fcount,
              int32_t* flist, uint8_t* fflag) {
    __shared__ double4 sm[kLayerTile];
    const int64_t t0 = int64_t(blockIdx.x) * TPT * blockDim.x + threadIdx.x;
    const bool active = t0 < nt;
    double tx[TPT], ty[TPT];
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
        const double2 p = tgt[min(t0 + u * int64_t(blockDim.x), nt - 1)];
        tx[u] = p.x;
        ty[u] = p.y;
    }
    for (int c = 0; c < nc; ++c) {
        const CurveDev C = cv[c];
        double d2[TPT], acc[TPT];
#pragma unroll
        for (int u = 0; u < TPT; ++u) d2[u] = 1e300, acc[u] = 0.0;
        tile_sum<kFamily, TPT>(crec, C.cbase, C.cbase + C.n, tx, ty, active, lambda, k1tab, sm, d2, acc);
        const double collar = allow_close ? 0.0 : kCollarFraction * C.diam;
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
            const int64_t t = t0 + u * int64_t(blockDim.x);
            if (t >= nt) continue;
            cval[int64_t(c) * nt + t] = acc[u];
            fflag[int64_t(c) * nt + t] = 0;
            const double d = sqrt(d2[u]);
            if (d - 0.75 * C.h <= fmax(collar, kFineReach * C.h)) {  // bie.cpp:414
                const int slot = atomicAdd(&fcount[c], 1);
                flist[int64_t(c) * nt + slot] = int32_t(t);
            }
        }
    }
}

template <int kFamily, int TPT>
__global__ void __launch_bounds__(512)
fine_kernel(const CurveDev* cv, int c, const double4* frec, const double2* tgt, int64_t nt,
            int allow_close, double lambda, const double* k1tab, const int* fcount,
            const int32_t* flist, double* fval, uint8_t* fflag, int* reject) {
    __shared__ double4 sm[kLayerTile];
    const CurveDev C = cv[c];
    const int cnt = fcount[c];
    const int nf = C.n * kFineFactor;
    const double collar = allow_close ? 0.0 : kCollarFraction * C.diam;
    const int64_t tile = int64_t(TPT) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * tile; base < cnt; base += int64_t(gridDim.x) * tile) {
        int64_t t[TPT];
        double tx[TPT], ty[TPT];
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
            const int64_t i = base + threadIdx.x + u * int64_t(blockDim.x);
            t[u] = i < cnt ? flist[int64_t(c) * nt + i] : -1;
            const double2 p = tgt[t[u] >= 0 ? t[u] : 0];
            tx[u] = p.x;
            ty[u] = p.y;
        }
        double d2[TPT], acc[TPT];
#pragma unroll
        for (int u = 0; u < TPT; ++u) d2[u] = 1e300, acc[u] = 0.0;
        tile_sum<kFamily, TPT>(frec, C.fbase, C.fbase + nf, tx, ty, t[0] >= 0, lambda, k1tab, sm, d2, acc);
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
            if (t[u] < 0) continue;
            const double d = sqrt(d2[u]);
            if (d == 0.0) {  // bie.cpp:417-420
                atomicMax(reject, 2);
            } else if (d < collar) {  // bie.cpp:421-424
                atomicMax(reject, 1);
            } else if (d <= kFineReach * C.h) {  // bie.cpp:425
                fval[int64_t(c) * nt + t[u]] = acc[u];
                fflag[int64_t(c) * nt + t[u]] = 1;
            }
        }
    }
}

// Per-curve values in curve order, then the log-completion terms
// (bie.cpp:443-446).
__global__ void finalize_kernel(const CurveDev* cv, int nc, int n_density, int n_aux,
                                const double* coeffs, const double2* tgt, int64_t nt,
                                const double* cval, const double* fval, const uint8_t* fflag,
                                double* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    double acc = 0.0;
    for (int c = 0; c < nc; ++c) {
        const int64_t k = int64_t(c) * nt + t;
        acc += fflag[k] ? fval[k] : cval[k];
    }
    const double2 p = tgt[t];
    for (int a = 0; a < n_aux; ++a) {
        const CurveDev C = cv[a + 1];
        const double dx = p.x - C.lcx, dy = p.y - C.lcy;
        acc += coeffs[n_density + a] * (-log(sqrt(dx * dx + dy * dy)) / kTwoPiL);
    }
    out[t] = acc;
}

template <typename T>
void upload_l(DBuf<T>& d, const std::vector<T>& h) {
    d.alloc(h.size());
    if (!h.empty()) VPG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

template <typename F>
int guarded_l(F&& f) {
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

}  // namespace
}  // namespace vpg

struct vpg_layer {
    int device = 0;
    int family = 0;
    double lambda = 0.0;
    int nc = 0, n_density = 0, n_aux = 0;
    int64_t ncoarse = 0, nfine = 0;
    int ncoef = 0;
    std::vector<vpg::CurveDev> meta;
    vpg::DBuf<vpg::CurveDev> meta_d;
    vpg::DBuf<double2> x, nrm, fx, fnrm;
    vpg::DBuf<double> speed, fspeed;
    const double* k1tab = nullptr;
};

using namespace vpg;

extern "C" {

int vpg_layer_create(int family, double lambda, const vpg_curve_block* curves, int ncurves,
                     int n_density, int n_aux, int device, vpg_layer** out) {
    return guarded_l([&] {
        if (!out) throw Error{VPG_ERR_INVALID_ARGUMENT, "layer is NULL"};
        *out = nullptr;
        if (family != VPG_LAPLACE && family != VPG_MODIFIED_HELMHOLTZ)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown kernel family"};
        if (family == VPG_MODIFIED_HELMHOLTZ && !(lambda > 0.0))  // kernel.cpp:195-196
            throw Error{VPG_ERR_INVALID_ARGUMENT, "make_kernel: modified Helmholtz needs lambda > 0"};
        if (ncurves < 1 || !curves) throw Error{VPG_ERR_INVALID_ARGUMENT, "need at least one curve"};
        if (n_aux < 0 || n_aux > ncurves - 1)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "n_aux must be in [0, ncurves - 1]"};
        auto L = std::make_unique<vpg_layer>();
        L->device = device;
        L->family = family;
        L->lambda = lambda;
        L->nc = ncurves;
        L->n_density = n_density;
        L->n_aux = n_aux;
        std::vector<double2> x, nrm, fx, fnrm;
        std::vector<double> sp, fsp;
        int cb = 0, fb = 0, ub = 0;
        for (int c = 0; c < ncurves; ++c) {
            const vpg_curve_block& B = curves[c];
            if (B.n < 16 || B.n % 2)  // bie.cpp:170-173
                throw Error{VPG_ERR_INVALID_ARGUMENT, "assemble_nystrom: node counts must be even and >= 16"};
            if (B.offset < 0 || int64_t(B.offset) + B.n > n_density)
                throw Error{VPG_ERR_INVALID_ARGUMENT, "curve block outside the density range"};
            if (!B.x || !B.normal || !B.speed || !B.fine_x || !B.fine_normal || !B.fine_speed)
                throw Error{VPG_ERR_INVALID_ARGUMENT, "curve geometry array is NULL"};
            if (!(B.length > 0.0)) throw Error{VPG_ERR_INVALID_ARGUMENT, "curve length must be positive"};
            CurveDev C{};
            C.n = B.n;
            C.offset = B.offset;
            C.cbase = cb;
            C.fbase = fb;
            C.ubase = ub;
            C.h = B.length / B.n;  // bie.cpp:406
            C.diam = B.diam;
            C.lcx = B.log_center[0];
            C.lcy = B.log_center[1];
            L->meta.push_back(C);
            for (int j = 0; j < B.n; ++j) {
                x.push_back(make_double2(B.x[2 * j], B.x[2 * j + 1]));
                nrm.push_back(make_double2(B.normal[2 * j], B.normal[2 * j + 1]));
                sp.push_back(B.speed[j]);
            }
            for (int j = 0; j < B.n * kFineFactor; ++j) {
                fx.push_back(make_double2(B.fine_x[2 * j], B.fine_x[2 * j + 1]));
                fnrm.push_back(make_double2(B.fine_normal[2 * j], B.fine_normal[2 * j + 1]));
                fsp.push_back(B.fine_speed[j]);
            }
            cb += B.n;
            fb += B.n * kFineFactor;
            ub += B.n / 2 + 1;
        }
        L->ncoarse = cb;
        L->nfine = fb;
        L->ncoef = ub;
        use_device(device);
        upload_l(L->meta_d, L->meta);
        upload_l(L->x, x);
        upload_l(L->nrm, nrm);
        upload_l(L->fx, fx);
        upload_l(L->fnrm, fnrm);
        upload_l(L->speed, sp);
        upload_l(L->fspeed, fsp);
        if (family == VPG_MODIFIED_HELMHOLTZ) L->k1tab = k1_table_dev();
        *out = L.release();
    });
}

int vpg_layer_eval(const vpg_layer* L, const double* coeffs, int64_t ncoeffs, const double* tgt_xy,
                   int64_t nt, int allow_close, double* out, unsigned flags, void* stream) {
    return guarded_l([&] {
        if (!L) throw Error{VPG_ERR_INVALID_ARGUMENT, "layer is NULL"};
        if (ncoeffs != int64_t(L->n_density) + L->n_aux)  // bie.cpp:387-388
            throw Error{VPG_ERR_INVALID_ARGUMENT, "eval_layer_potential: coefficient length mismatch"};
        if (nt < 0 || (nt && (!tgt_xy || !out)) || !coeffs)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad arrays"};
        VPG_CUDA(cudaSetDevice(L->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        bool owned = false;
        if (!s) {
            VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamDefault));  // orders after the legacy stream
            owned = true;
        }
        struct SG {
            cudaStream_t s;
            bool o;
            ~SG() {
                if (o) cudaStreamDestroy(s);
            }
        } sg{s, owned};
        const bool dev = flags & VPG_DEVICE_POINTERS;
        const int nc = L->nc;
        // one scratch block: coefficients, records, per-curve values and lists
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t n_ab = al(sizeof(double2) * size_t(L->ncoef));
        const size_t n_cr = al(sizeof(double4) * size_t(L->ncoarse));
        const size_t n_fr = al(sizeof(double4) * size_t(L->nfine));
        const size_t n_val = al(sizeof(double) * size_t(nt) * nc);
        const size_t n_list = al(sizeof(int32_t) * size_t(nt) * nc);
        const size_t n_flag = al(size_t(nt) * nc);
        const size_t n_cnt = al(sizeof(int) * size_t(nc + 1));
        const size_t n_io = dev ? 0 : al(sizeof(double) * size_t(ncoeffs)) + al(sizeof(double2) * size_t(nt)) +
                                          al(sizeof(double) * size_t(nt));
        const size_t total = n_ab + n_cr + n_fr + 2 * n_val + n_list + n_flag + n_cnt + n_io;
        char* base = nullptr;
        VPG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), total, s));
        struct Free {
            void* p;
            cudaStream_t s;
            ~Free() {
                if (p) cudaFreeAsync(p, s);
            }
        } fr{base, s};
        char* cur = base;
        auto take = [&](size_t b) {
            char* p = cur;
            cur += b;
            return p;
        };
        double2* ab = reinterpret_cast<double2*>(take(n_ab));
        double4* crec = reinterpret_cast<double4*>(take(n_cr));
        double4* frec = reinterpret_cast<double4*>(take(n_fr));
        double* cval = reinterpret_cast<double*>(take(n_val));
        double* fval = reinterpret_cast<double*>(take(n_val));
        int32_t* flist = reinterpret_cast<int32_t*>(take(n_list));
        uint8_t* fflag = reinterpret_cast<uint8_t*>(take(n_flag));
        int* cnt = reinterpret_cast<int*>(take(n_cnt));  // [nc] list counts, [nc] reject
        const double* cf = coeffs;
        const double2* tg = reinterpret_cast<const double2*>(tgt_xy);
        double* od = out;
        if (!dev) {
            double* cfd = reinterpret_cast<double*>(take(al(sizeof(double) * size_t(ncoeffs))));
            double2* tgd = reinterpret_cast<double2*>(take(al(sizeof(double2) * size_t(nt))));
            od = reinterpret_cast<double*>(take(al(sizeof(double) * size_t(nt))));
            VPG_CUDA(cudaMemcpyAsync(cfd, coeffs, sizeof(double) * size_t(ncoeffs), cudaMemcpyHostToDevice, s));
            if (nt) VPG_CUDA(cudaMemcpyAsync(tgd, tgt_xy, sizeof(double2) * size_t(nt), cudaMemcpyHostToDevice, s));
            cf = cfd;
            tg = tgd;
        }
        VPG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(nc + 1), s));
        const CurveDev* cv = L->meta_d.p;
        ups_coef_kernel<<<nblk(int64_t(L->ncoef) * 32, 256), 256, 0, s>>>(cv, nc, L->ncoef, cf, ab);
        VPG_LAUNCH_CHECK();
        const int64_t nrec = L->ncoarse + L->nfine;
        const bool lap = L->family == VPG_LAPLACE;
        (lap ? records_kernel<VPG_LAPLACE> : records_kernel<VPG_MODIFIED_HELMHOLTZ>)
            <<<nblk(nrec, 128), 128, 0, s>>>(cv, nc, L->ncoarse, L->nfine, cf, ab, L->x.p, L->nrm.p,
                                             L->speed.p, L->fx.p, L->fnrm.p, L->fspeed.p, L->lambda, crec,
                                             frec);
        VPG_LAUNCH_CHECK();
        if (nt) {
            (lap ? coarse_kernel<VPG_LAPLACE, kCoarseTPT> : coarse_kernel<VPG_MODIFIED_HELMHOLTZ, kCoarseTPT>)
                <<<nblk(nt, kCoarseTPT * kCoarseThreads), kCoarseThreads, 0, s>>>(cv, nc, crec, tg, nt, allow_close,
                                                                   L->lambda, L->k1tab, cval, cnt, flist,
                                                                   fflag);
            VPG_LAUNCH_CHECK();
            int sms = 148;
            VPG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, L->device));
            const unsigned fgrid =
                unsigned(std::min<int64_t>(nblk(nt, kFineTPT * kFineThreads), int64_t(sms) * (2048 / kFineThreads)));
            for (int c = 0; c < nc; ++c) {
                (lap ? fine_kernel<VPG_LAPLACE, kFineTPT> : fine_kernel<VPG_MODIFIED_HELMHOLTZ, kFineTPT>)
                    <<<fgrid, kFineThreads, 0, s>>>(cv, c, frec, tg, nt, allow_close, L->lambda, L->k1tab,
                                                     cnt, flist, fval, fflag, cnt + nc);
                VPG_LAUNCH_CHECK();
            }
            finalize_kernel<<<nblk(nt, 256), 256, 0, s>>>(cv, nc, L->n_density, L->n_aux, cf, tg, nt, cval,
                                                         fval, fflag, od);
            VPG_LAUNCH_CHECK();
        }
        int reject = 0;
        VPG_CUDA(cudaMemcpyAsync(&reject, cnt + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
        if (!dev && nt)
            VPG_CUDA(cudaMemcpyAsync(out, od, sizeof(double) * size_t(nt), cudaMemcpyDeviceToHost, s));
        VPG_CUDA(cudaStreamSynchronize(s));
        if (reject == 2)  // bie.cpp:450-457
            throw Error{VPG_ERR_INVALID_ARGUMENT, "eval_layer_potential: target lies on a boundary node"};
        if (reject == 1)
            throw Error{VPG_ERR_INVALID_ARGUMENT,
                        "eval_layer_potential: target inside the close-evaluation collar "
                        "(0.02 of the curve diameter); refine the boundary grid and "
                        "evaluate with solve_bvp, or move the target"};
    });
}

int vpg_layer_destroy(vpg_layer* L) {
    return guarded_l([&] {
        if (!L) return;
        cudaSetDevice(L->device);
        delete L;
    });
}

}  // extern "C"
