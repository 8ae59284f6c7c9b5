// common.cuh -- shared device/host helpers for libvolpot_b200.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "volpot_b200.h"

namespace vpg {

// ---------------------------------------------------------------- errors --
// Thread-local message behind vpg_last_error().
void set_error(const std::string& msg);
const char* get_error();

struct Error {
    int status;
    std::string msg;
};

#define VPG_CUDA(call)                                                       \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) {                                             \
            (void)cudaGetLastError();                                        \
            throw ::vpg::Error{e_ == cudaErrorMemoryAllocation               \
                                   ? VPG_ERR_OUT_OF_MEMORY                   \
                                   : VPG_ERR_CUDA,                           \
                               std::string(#call) + ": " +                   \
                                   cudaGetErrorString(e_)};                  \
        }                                                                    \
    } while (0)

#define VPG_LAUNCH_CHECK() VPG_CUDA(cudaGetLastError())

// Verifies that `device` is a usable sm_100 device and makes it current.
void use_device(int device);

// ------------------------------------------------------------- constants --
constexpr double kInv2Pi = 0.15915494309189533577;   // summation.cpp:15
constexpr double kInv4Pi = 0.07957747154594766788;   // 0.25/pi, kernel.cpp:183
constexpr double kLn2Hi = 6.93147180369123816490e-01;  // ln2 split, hi has
constexpr double kLn2Lo = 1.90821492927058770002e-10;  // 21 trailing zeros

// ------------------------------------------------------------ Morton ids --
// Bit interleave of the reference (summation.cpp:45-62): x in even bits.
__host__ __device__ inline uint32_t spread2(uint32_t v) {
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__host__ __device__ inline uint32_t mort(uint32_t ix, uint32_t iy) {
    return spread2(ix) | (spread2(iy) << 1);
}
__host__ __device__ inline uint32_t squash2(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0F0F0F0Fu;
    v = (v | (v >> 4)) & 0x00FF00FFu;
    v = (v | (v >> 8)) & 0x0000FFFFu;
    return v;
}
// Offset of level l in the concatenated per-level box arrays.
__host__ __device__ inline int64_t lvl_base(int l) {
    return ((int64_t(1) << (2 * l)) - 1) / 3;
}

// --------------------------------------------------------------- complex --
struct cplx {
    double re, im;
};
__host__ __device__ inline cplx cmul(cplx a, cplx b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ inline cplx cadd(cplx a, cplx b) {
    return {a.re + b.re, a.im + b.im};
}

// ------------------------------------------------------------ fast log --
// Natural log for the P2P inner loop, split as ln(x) = e*ln2 + t so the
// caller can accumulate sum(q*t) and sum(q*e) separately and apply ln2 once
// (hi/lo split) per target.  x = 2^e * m, m in [1,2); m is rounded to the
// nearest centre c = 1 + i/512 (i = 0..512, from the top mantissa bits) and
// ln(m) = -ln(1/c) + log1p(m * RN(1/c) - 1) with |m/c - 1| <= 2^-10; log1p by
// a degree-4 polynomial (truncation 2^-50/5 < 2e-16 absolute; one DFMA per
// pair less than the 8-bit table with degree 5, -6% near-field time on
// cfg4; VPG_LOG_BITS=8 selects that variant).  Centre i = 0
// is c = 1 exactly (RN(1/c) = 1, ln = 0), so ln(1) and ln(2^k) come out
// exact.  The table (RN(1/c), -ln RN(1/c)) lives in shared memory replicated
// 8x so the eight lanes of every quarter-warp 128-bit access hit distinct
// bank groups whatever the indices (conflict-free).
#ifndef VPG_LOG_BITS
#define VPG_LOG_BITS 9
#endif
constexpr int kLogTableBits = VPG_LOG_BITS;
constexpr int kLogTableSize = (1 << kLogTableBits) + 1;
#ifndef VPG_LOG_COPIES
#define VPG_LOG_COPIES 8
#endif
constexpr int kLogTableCopies = VPG_LOG_COPIES;
constexpr int kLogTableBytes = kLogTableSize * kLogTableCopies * 16;

// Host-built table (inv_c, -ln(inv_c)) in global memory (one per device,
// see log_table_dev()), replicated into shared memory by each CTA.
__device__ inline void log_table_to_smem(double2* sm, const double2* gtab) {
    for (int i = threadIdx.x; i < kLogTableSize * kLogTableCopies; i += blockDim.x)
        sm[i] = gtab[i / kLogTableCopies];
}

// Polynomial coefficients live in constant memory so every DFMA takes them
// as a c[][] operand (no register materialisation inside the hot loop).
static __constant__ double c_log1p5[4] = {0.2, -0.25, 0.33333333333333333333, -0.5};
static __constant__ double c_magic_bias = 4503599627371519.0;  // 2^52 + 1023

__device__ __forceinline__ double2 lds_f64x2(uint32_t saddr) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(saddr));
    return v;
}

// Shared-window byte address of this lane's copy of table entry 0, biased
// by -(0x3FF << bits) entries: fast_log_split indexes with the mantissa
// word 0x3FF00000 | mant (see there); uint32 wrap-around cancels.
constexpr uint32_t kLogTableBias = uint32_t(0x3FF << kLogTableBits) * uint32_t(16 * kLogTableCopies);
__device__ __forceinline__ uint32_t log_table_lane_addr(const double2* tab, int lane8) {
    return uint32_t(__cvta_generic_to_shared(tab)) + uint32_t(lane8) * 16u - kLogTableBias;
}

// Returns t with ln(x) = ed*ln2 + t; ed = exponent as a double.
// Integer side (6 instructions): the mantissa word mhi = 0x3FF00000 | mant
// is one 3-input LOP3; v = (mhi + half) >> (20 - bits) = (0x3FF << bits) +
// idx (a rounding carry gives idx = 2^bits, the table's last entry), so the
// byte address is tab_lane + 128 v with the bias folded into tab_lane
// (log_table_lane_addr); the unbiased exponent is (hi - 0x3FF00000) >> 20
// (arithmetic shift), converted by I2F.F64 (conversion pipe, not FP64).
__device__ __forceinline__ double fast_log_split(double x, uint32_t tab_lane, double& ed) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    const uint32_t v = uint32_t(mhi + (1 << (19 - kLogTableBits))) >> (20 - kLogTableBits);
    const double m = __hiloint2double(mhi, lo);
    ed = __int2double_rn((hi - 0x3FF00000) >> 20);
    const double2 tc = lds_f64x2(tab_lane + v * uint32_t(16 * kLogTableCopies));
    const double r = fma(m, tc.x, -1.0);
#if VPG_LOG_BITS >= 9
    // |r| <= 2^-10: degree 4 (truncation 2^-50/5 < 2e-16 absolute)
    double p = fma(r, c_log1p5[1], c_log1p5[2]);
#else
    double p = fma(r, c_log1p5[0], c_log1p5[1]);
    p = fma(r, p, c_log1p5[2]);
#endif
    p = fma(r, p, c_log1p5[3]);
    const double r2 = r * r;
    return tc.y + fma(r2, p, r);
}

// ln(x) as one double, for the near-field loops: the same reduction as
// fast_log_split, with the exponent term folded into the polynomial's
// addend, w = e ln2 + (-ln RN(1/c)) (one DFMA, the product exact inside it),
// and log1p by Horner in r (c_flog), so the last DFMA adds r p(r) to w:
// ln x = fma(r, p, w), six FP64 instructions (fast_log_split plus combining
// its split result: eight).  Error: truncation < 1.2e-17, p's rounding
// scaled by |r| <= 2^-10, ln2's representation error times |e|, and two
// roundings (w, the result): <= 1.3e-16 absolute for |ln x| < 1, <= 1.3
// ulp above, exact 0 at x = 1 (mpmath check of this exact arithmetic over
// 1e-30..1e3 and the interval edges).
#ifndef VPG_LOG_FOLD
#define VPG_LOG_FOLD 1
#endif
constexpr double kLn2 = 0.69314718055994530942;
// The table of fast_log (lap_log_table_dev): the centres of fast_log_split,
// c = 1 + i/512 (i = 0..512, the mantissa ROUNDED to its top 9 bits, |m/c -
// 1| <= 2^-10, centre 0 exactly 1 so ln(2^k) = fl(k ln2) and ln 1 = 0 as
// the SPEC examples need), entries (RN(1/c), -ln RN(1/c) - i ln2/512).  The
// exponent goes in together with the index: with t = hi + half-an-index,
// g = (t >> 11) - (0x3FF << 9) = e 512 + i exactly (a rounding carry into
// the exponent field gives (e + 1) 512 + 0 = e 512 + 512, the same number),
// and w = fma(g, ln2/512, entry) = e ln2 - ln RN(1/c), the product exact
// inside the DFMA.  Integer side (8): IADD + LEA.HI for g, I2F.F64; the
// mantissa word (LOP3) and, rounded, its index scaled to the 128-byte
// entry stride (IADD, SHF, IMAD; bias folded into tab_lane as in
// fast_log_split); the register-pair move for m.
constexpr double kLn2Over512 = 0.69314718055994530942 / 512.0;
// log1p(r) = r p(r), p = c1 + r(-1/2 + r(c3 - r/4)): the Taylor terms with
// r^5/5 economised over |r| <= h = 2^-10 (Chebyshev: r^5 ~ (5/4)h^2 r^3 -
// (5/16)h^4 r), c1 = 1 - h^4/16, c3 = 1/3 + h^2/4; truncation < 1.2e-17.
// DFMA takes these as c[][] operands (no register materialisation).
static __constant__ double c_flog[4] = {0.3333335717519124, kLn2Over512, -0.25, 0.99999999999994315658};
__device__ __forceinline__ double fast_log(double x, uint32_t tab_lane) {
    constexpr int kHalf = 1 << (19 - kLogTableBits);
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double g = __int2double_rn(((hi + kHalf) >> 11) - (0x3FF << 9));
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    uint32_t idx, addr;  // explicit shift + multiply-add: one IMAD, no mask
    asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi + kHalf));
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
    const double m = __hiloint2double(mhi, lo);
    const double2 tc = lds_f64x2(addr);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}
static_assert(kLogTableBits == 9 && kLogTableCopies == 8, "fast_log assumes the 9-bit, 8-copy layout");

// fast_log with the table read from global memory (lap_log_table_dev, one
// copy): the same arithmetic on the same table values, so it returns the
// same bits as the smem form -- for rare paths (coincidence fix-ups) in
// kernels that do not stage the 66 KB table.
__device__ __forceinline__ double fast_log(double x, const double2* gtab) {
    constexpr int kHalf = 1 << (19 - kLogTableBits);
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double g = __int2double_rn(((hi + kHalf) >> 11) - (0x3FF << 9));
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    const uint32_t idx = (uint32_t(mhi + kHalf) >> 11) - uint32_t(0x3FF << kLogTableBits);
    const double m = __hiloint2double(mhi, lo);
    const double2 tc = __ldg(gtab + idx);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}

// The near-field form of fast_log (VPG_LOG_TRUNC, default): the mantissa's
// top 9 bits TRUNCATED select the centre c = 1 + (i + 1/2)/512 (i = 0..511,
// again |m/c - 1| <= 2^-10), so the exponent-and-index word g = e 512 + i
// is (hi >> 11) - bias without the rounding add and the mantissa word
// indexes the table as it is: two integer instructions fewer per pair
// (logvar_bench: +4% pairs/s), same six DFMAs, same error bound.  No centre
// is exactly 1, so ln 1 comes out as a rounding error (1.1e-17) instead of
// 0: the all-pairs kernel, which has to return the SPEC's exact zeros, keeps
// fast_log.  Table lap_log_table_dev(): (RN(1/c), -ln RN(1/c) - i ln2/512).
#ifndef VPG_LOG_TRUNC
#define VPG_LOG_TRUNC 1
#endif
__device__ __forceinline__ double trunc_log(double x, uint32_t tab_lane) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double g = __int2double_rn((hi >> 11) - (0x3FF << 9));
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    uint32_t idx, addr;
    asm("shr.b32 %0, %1, 11;" : "=r"(idx) : "r"(mhi));
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(addr) : "r"(idx), "r"(tab_lane));
    const double m = __hiloint2double(mhi, lo);
    const double2 tc = lds_f64x2(addr);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}
__device__ __forceinline__ double trunc_log(double x, const double2* gtab) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const double g = __int2double_rn((hi >> 11) - (0x3FF << 9));
    int mhi;
    asm("lop3.b32 %0, %1, 0x000FFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x3FF00000));
    const uint32_t idx = (uint32_t(mhi) >> 11) - uint32_t(0x3FF << kLogTableBits);
    const double m = __hiloint2double(mhi, lo);
    const double2 tc = __ldg(gtab + idx);
    const double r = fma(m, tc.x, -1.0);
    const double w = fma(g, c_flog[1], tc.y);
    double p = fma(r, c_flog[2], c_flog[0]);
    p = fma(r, p, -0.5);
    p = fma(r, p, c_flog[3]);
    return fma(r, p, w);
}
// ln x of the near-field kernels (one function, so every kernel of a plan
// returns the same bits for the same pair)
template <class Tab>
__device__ __forceinline__ double near_log(double x, Tab tab) {
#if VPG_LOG_TRUNC
    return trunc_log(x, tab);
#else
    return fast_log(x, tab);
#endif
}

// ----------------------------------------------- programmatic launches --
// Kernels of one apply are chained with programmatic dependent launch: the
// next grid may start (and stage its constant operators / tables) while the
// previous one drains; it calls pdl_wait() before touching the
// predecessor's outputs.  pdl_trigger() lets the successor launch early.
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VPG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// ------------------------------------------------ TMA bulk copies (1-D) --
// cp.async.bulk global -> shared with mbarrier completion (sm_90+ async
// proxy).  Sizes and addresses must be multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Whole-CTA staging of a contiguous global block into smem with 1-D bulk
// copies (one issuing thread, <= 32 KB per copy) -- replaces the dependent
// load/store loops whose L2 latency dominated the small per-level kernels.
// Must be called by every thread of the CTA; bar is a __shared__ word.
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar, uint32_t phase) {
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768u) {
            const uint32_t len = bytes - off < 32768u ? bytes - off : 32768u;
            tma_load_1d(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len, bar);
        }
    }
    mbar_wait(bar, phase);
}

// Cooperative launch (all CTAs co-resident: grid-wide barriers allowed).
template <typename... KArgs, typename... Args>
void launch_coop(void (*kern)(KArgs...), int grid, dim3 block, size_t smem, cudaStream_t st,
                 Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VPG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Per-device constant tables, built on first use (api.cu).
const double2* log_table_dev();  // kLogTableSize entries (inv_c, -ln inv_c): fast_log_split
const double2* lap_log_table_dev();  // the near-field table: near_log's (VPG_LOG_FOLD=0: log_table_dev)
const double2* lap_log_table_rn_dev();  // fast_log's table (all-pairs kernel)
const double* k0_table_dev();    // K0 Chebyshev fits, see k0.cuh
const double* k1_table_dev();    // K1 Chebyshev fits (same layout)
const double* k0_fast_table_dev();  // quarter-octave K0 fits (k0_fast)

// Opt a kernel into > 48 KB dynamic shared memory once per device.
void smem_optin(const void* func, int bytes);

}  // namespace vpg
