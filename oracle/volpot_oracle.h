/*
 * volpot_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load libvolpot_oracle.so, and only as the
 * checker.  The product library (paper_2203_05933_b200/libvolpot_b200.so)
 * never links or loads it.
 *
 * Every function restates one piece of the reference (arxiv 2203.05933
 * artifact, /root/reference/proj) and cites the file:line it follows.  The
 * restatement is pinned against the reference itself (oracle/_ref, built
 * from the unmodified sources) by tests/test_oracle_pins.py and against the
 * committed golden vectors in tests/golden/.
 *
 * Point arrays are interleaved xy doubles (the reference Vec2 is a 16-byte
 * POD, common.hpp:13-14).  Level-indexed box arrays ("cnt_all") concatenate
 * levels 0..L, level l starting at (4^l - 1)/3.
 */
#ifndef VOLPOT_ORACLE_H
#define VOLPOT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int direct;   /* 1: pairwise fallback (summation.cpp:578) */
    int levels;   /* leaf level L (summation.cpp:580-583) */
    int order;    /* P (summation.cpp:155-157) or max Chebyshev m */
    double eps;   /* clamped epsilon (summation.cpp:557) */
    double x0, y0, side; /* root box, side already scaled by (1+1e-12) */
} vo_params;

/* summation.cpp:551-591 -- plan parameters exactly as the ctor derives them. */
int vo_plan_params(int family, double lambda, const double* src, int64_t ns,
                   const double* tgt, int64_t nt, double eps, vo_params* out);

/* summation.cpp:81-100 -- leaf CSR (stable counting sort by Morton leaf). */
void vo_bin_points(const double* pts, int64_t n, int levels, double x0,
                   double y0, double side, int32_t* off, int32_t* ids);

/* summation.cpp:102-115 -- per-level counts, levels 0..L concatenated. */
void vo_count_levels(int levels, const int32_t* leaf_off, int32_t* cnt_all);

/* summation.cpp:271-303 -- explicit M2L list of one level, in the reference
 * enumeration order: target boxes in Morton order (tgt_cnt > 0), then
 * (qy, qx, child) loops.  Returns the entry count; writes when arrays are
 * non-NULL.  tbox[i], toff[i..i+1] is the target CSR (ntbox entries + 1),
 * src[e]/oidx[e] the source box and offset index (dx+3)+7*(dy+3). */
int64_t vo_m2l_list(int levels, int level, const int32_t* src_cnt_all,
                    const int32_t* tgt_cnt_all, int32_t* ntbox,
                    int32_t* tbox, int32_t* toff, int32_t* src, int32_t* oidx);

/* Number of enumerated near-field (P2P) pairs, self pairs included
 * (summation.cpp:330-344). */
int64_t vo_p2p_pairs(int levels, const int32_t* src_off, const int32_t* tgt_off);

/* summation.cpp:542-643 -- whole SummationPlan (ctor + apply) restated:
 * pairwise, Laplace FMM or modified-Helmholtz treecode.  Returns 0, or 1 on
 * a kernel/size error. */
int vo_plan_sum(int family, double lambda, const double* src, const double* q,
                int64_t ns, const double* tgt, int64_t nt, double eps,
                double* out, int nthreads);

/* summation.cpp:501-540 -- direct_sum.  Returns 0, or 2 with the smallest
 * coincident (i, j) in ci, cj. */
int vo_direct_sum(int family, double lambda, const double* src,
                  const double* q, int64_t ns, const double* tgt, int64_t nt,
                  double* out, int64_t* ci, int64_t* cj, int nthreads);

/* Pairwise sum with the r^2 == 0 skip (summation.cpp:619-635), accumulated
 * in long double.  The accuracy oracle for >= 1M points. */
void vo_pairwise_sum_ld(int family, double lambda, const double* src,
                        const double* q, int64_t ns, const double* tgt,
                        int64_t nt, double* out, int nthreads);

/* kernel.cpp:17-172 -- K0 (series below 2, Chebyshev fits above). */
double vo_bessel_k0(double x);
/* kernel.cpp:181-186 */
double vo_radial_r2(int family, double lambda, double r2);

/* potential.cpp:446-462 -- correction apply: out[t] += sum over blocks of
 * pool row . f[node_off[cell] ..]. Rows live in a flat pool (pool_off CSR). */
void vo_correction_apply(int64_t nt, const int32_t* blk_off,
                         const int32_t* blk_cell, const int32_t* blk_pool,
                         const int64_t* pool_off, const double* pool_vals,
                         const int32_t* node_off, const double* f,
                         double* out, int nthreads);

/* potential.cpp:397-412 -- charges = src_wj * (O_type(cell) * f_cell).
 * over_* are row-major (nq x np) oversampling maps per cell type. */
void vo_build_charges(int64_t ncell, const int32_t* cell_type,
                      const int32_t* node_off, const int32_t* src_off,
                      const double* over0, int np0, int nq0,
                      const double* over1, int np1, int nq1,
                      const double* src_wj, const double* f, double* charges, int nthreads);

/* kernel.cpp:174-179 -- K1 (series below 2, Chebyshev fits above). */
double vo_bessel_k1(double x);

/* bie.cpp:112-135 -- trig_upsample: zero-padded Fourier interpolation of n
 * (even) periodic samples onto factor*n points. */
void vo_trig_upsample(const double* f, int n, int factor, double* out);

/* One curve block of BoundarySystem (bie.hpp:30-47): the fields that
 * eval_layer_potential reads.  x/normal are n interleaved xy, speed n;
 * fine_* the 8n-point refined geometry (bie.cpp:206-215). */
typedef struct {
    int n;
    int offset;
    double length;
    double diam;
    const double* x;
    const double* normal;
    const double* speed;
    const double* fine_x;
    const double* fine_normal;
    const double* fine_speed;
    double log_center[2];
} vo_curve;

/* bie.cpp:383-461 -- eval_layer_potential(sys, coeffs, targets,
 * allow_close).  Returns 0, 1 (coefficient length mismatch), 2 (a target
 * lies on a boundary node) or 3 (a target inside the collar); 2 wins over 3
 * when both occur (the reference keeps whichever store came last). */
int vo_layer_eval(int family, double lambda, const vo_curve* curves,
                  int ncurves, int n_density, int n_aux,
                  const double* coeffs, int64_t ncoeffs, const double* tgt,
                  int64_t nt, int allow_close, double* out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
