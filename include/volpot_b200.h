/*
 * volpot_b200.h -- C ABI of the B200-native FMM-step library
 * (paper_2203_05933_b200/libvolpot_b200.so, sm_100a only).
 *
 * This is the drop-in boundary for the hot path of the arxiv 2203.05933
 * volume-potential artifact (/root/reference/proj):
 *
 *   reference symbol                                  replaced by
 *   ------------------------------------------------  ---------------------------
 *   SummationPlan::SummationPlan  (summation.hpp:36-37,
 *                                  summation.cpp:551-591)  vpg_plan_create
 *   SummationPlan::apply          (summation.hpp:42,
 *                                  summation.cpp:610-643)  vpg_plan_apply
 *   SummationPlan::num_sources/num_targets/levels/
 *                  expansion_order (summation.hpp:44-50)   vpg_plan_info
 *   SummationPlan::~SummationPlan (summation.hpp:38)       vpg_plan_destroy
 *   direct_sum                    (summation.hpp:22-23,
 *                                  summation.cpp:501-540)  vpg_direct_sum
 *   accelerated_sum               (summation.hpp:58-61)    create+apply+destroy
 *   bessel_k0                     (kernel.hpp:11)          vpg_bessel_k0 (device)
 *   correction loop of VolumePotentialOperator::apply
 *                                 (potential.cpp:446-462)  vpg_corr_create/apply
 *   build_charges                 (potential.cpp:397-412)  vpg_charges_create/apply
 *   VolumePotentialOperator::apply (potential.cpp:431-470) vpg_operator_create/apply
 *   eval_layer_potential          (bie.hpp:87-90,
 *                                  bie.cpp:383-468)       vpg_layer_create/eval
 *
 * Conventions
 *   - Point arrays are interleaved xy float64 (the reference Vec2 is a
 *     16-byte POD, common.hpp:13-14), so a std::vector<Vec2>::data() can be
 *     passed zero-copy.
 *   - Every entry point returns a vpg_status; on failure vpg_last_error()
 *     returns a thread-local message using the reference's wording where the
 *     reference throws (e.g. "SummationPlan::apply: charge count N does not
 *     match source count M", summation.cpp:613-617).
 *   - apply is const: a plan is immutable after creation and may be applied
 *     concurrently from several host threads with distinct charge vectors
 *     (summation.hpp:32-33).  Scratch is stream-ordered per call.
 *   - Results are run-to-run bit-identical: no floating-point atomics, every
 *     sum is reduced in a fixed order.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with VPG_ERR_CUDA.
 */
#ifndef VOLPOT_B200_H
#define VOLPOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPG_ABI_VERSION 3  /* 2: vpg_plan_info_t.near_symmetric, vpg_layer_*; 3: near_lattice (was reserved) */

typedef enum {
    VPG_OK = 0,
    VPG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    VPG_ERR_COINCIDENT = 2,       /* direct_sum coincidence (summation.cpp:535-538) */
    VPG_ERR_DOMAIN = 3,           /* std::domain_error (kernel.cpp:169) */
    VPG_ERR_CUDA = 4,
    VPG_ERR_OUT_OF_MEMORY = 5
} vpg_status;

typedef enum { VPG_LAPLACE = 0, VPG_MODIFIED_HELMHOLTZ = 1 } vpg_family;

/* Tree policy.  REFERENCE reproduces the reference plan bit-exactly (same
 * bounding box, depth clamp(ceil(log4(max(ns,nt)/32)),2,7), same P, same
 * pairwise threshold ns*nt <= 4e6), so trees and interaction lists can be
 * compared entry by entry.  NATIVE departs from the reference algorithm
 * where a B200-first one is faster, with parity to the requested tolerance:
 *   Laplace: an adaptive quadtree -- a box splits while it holds more than
 *     96 sources or targets, down to depth 16 -- with U/V/W/X interaction
 *     lists (P2P, M2L, M2P, P2L), so clustered points stay O(n); the
 *     uniform-tree dumps and leaf shards are not available.
 *   Modified Helmholtz: the reference tree with a compressed Chebyshev-
 *     interpolation FMM (SVD-based M2L) instead of the proxy treecode;
 *     expansion_order then reports the Chebyshev nodes per dimension.
 * The pairwise threshold (ns*nt <= 4e6) is the reference's in both modes. */
typedef enum { VPG_MODE_REFERENCE = 0, VPG_MODE_NATIVE = 1 } vpg_mode;

/* vpg_plan_apply flags */
#define VPG_DEVICE_POINTERS 1u /* q and out are device pointers (no copies) */
#define VPG_NO_SYNC 2u         /* return without synchronising the stream */

typedef struct vpg_plan vpg_plan;
typedef struct vpg_corr vpg_corr;
typedef struct vpg_charges vpg_charges;
typedef struct vpg_operator vpg_operator;

typedef struct {
    int64_t num_sources, num_targets;
    int32_t levels;          /* 0 = pairwise (summation.hpp:46-47) */
    int32_t expansion_order; /* P, or max Chebyshev m (summation.hpp:48-50) */
    int32_t family, mode, device;
    double epsilon;          /* clamped to [1e-12, 1e-3] (summation.cpp:557) */
    double x0, y0, side;     /* root box */
    int64_t m2l_pairs;       /* (target box, source box) translations */
    int64_t p2p_pairs;       /* enumerated near-field pairs, self included */
    int64_t m2m_children, l2l_children;
    int64_t device_bytes;    /* resident plan footprint */
    int32_t near_symmetric;  /* 1: near field by unordered pairs (fmm.cu p2p_sym_kernel) */
    int32_t near_lattice;    /* 1: near field as dense K_o q products of translation-invariant leaves (lattice.cu) */
} vpg_plan_info_t;

/* Phase timings of the most recent apply on a plan with profiling on, in
 * milliseconds (CUDA events on the apply stream). */
typedef enum {
    VPG_PHASE_UPLOAD = 0,  /* H2D of charges (host-pointer apply only) */
    VPG_PHASE_GATHER,      /* charges into Morton order */
    VPG_PHASE_P2M,
    VPG_PHASE_M2M,
    VPG_PHASE_M2L,
    VPG_PHASE_L2L,
    VPG_PHASE_P2P,         /* fused L2P + near field (or pairwise / treecode) */
    VPG_PHASE_DOWNLOAD,    /* D2H of potentials */
    VPG_PHASE_COUNT
} vpg_phase;

const char* vpg_last_error(void);
int vpg_abi_version(void);
/* Number of visible devices usable by this library (sm_100). */
int vpg_device_count(int* count);

int vpg_plan_create(int family, double lambda, const double* src_xy,
                    int64_t ns, const double* tgt_xy, int64_t nt,
                    double epsilon, int mode, int device, vpg_plan** plan);
/* q: ns charges; out: nt potentials in original target order.  Host
 * pointers unless VPG_DEVICE_POINTERS.  stream: cudaStream_t or NULL for a
 * library-owned per-call stream. */
int vpg_plan_apply(const vpg_plan* plan, const double* q, int64_t nq,
                   double* out, unsigned flags, void* stream);
int vpg_plan_info(const vpg_plan* plan, vpg_plan_info_t* info);
int vpg_plan_set_profiling(vpg_plan* plan, int on);
int vpg_plan_phase_times(const vpg_plan* plan, float* ms /* VPG_PHASE_COUNT */);
/* Kernel launches issued by the most recent apply. */
int vpg_plan_last_launches(const vpg_plan* plan, int64_t* launches);
/* Copies the device tree back for the bit-exact check.
 * src_off/tgt_off: 4^L + 1 ints, src_ids: ns, tgt_ids: nt,
 * src_cnt/tgt_cnt: sum_{l<=L} 4^l ints (levels concatenated, level l at
 * (4^l-1)/3).  Any pointer may be NULL.  Fails for pairwise plans. */
int vpg_plan_dump_tree(const vpg_plan* plan, int32_t* src_off,
                       int32_t* src_ids, int32_t* tgt_off, int32_t* tgt_ids,
                       int32_t* src_cnt, int32_t* tgt_cnt);
/* M2L interaction list of one level in the reference enumeration order
 * (summation.cpp:271-303): *ntbox target boxes (tbox, toff CSR of ntbox+1)
 * and *nent entries (src box, offset index (dx+3)+7*(dy+3)).  Call with NULL
 * arrays to get the sizes. */
int vpg_plan_dump_m2l(const vpg_plan* plan, int level, int32_t* ntbox,
                      int64_t* nent, int32_t* tbox, int32_t* toff,
                      int32_t* src, int32_t* oidx);
/* Multi-GPU target sharding (one process per GPU): restricts
 * the target side of later applies (M2L, L2L, L2P+P2P, and M2P / P2L on
 * adaptive trees) to the shard units [unit_begin, unit_end); the upward pass
 * stays complete.  Units are the 4^levels Morton leaves of a reference-mode
 * tree, or the leaves holding targets (in target order) of an adaptive tree;
 * vpg_plan_shard_units gives their count and a work estimate per unit for
 * balancing.  Outputs of targets outside the shard are written as 0.0, so
 * summing the shards' outputs (one all-reduce) reproduces the unsharded plan
 * bit for bit.  Not to be called concurrently with apply.  [0, nunits)
 * restores the full plan.  Modified-Helmholtz plans shard their target side
 * too (treecode: the traversal; Chebyshev FMM: L2P and near field). */
int vpg_plan_set_shard(vpg_plan* plan, int64_t unit_begin, int64_t unit_end);
int vpg_plan_shard_units(const vpg_plan* plan, int64_t* nunits, double* costs /* [nunits] or NULL */);
int vpg_plan_destroy(vpg_plan* plan);

/* direct_sum (summation.cpp:501-540).  skip_coincident = 0: reference
 * semantics, returns VPG_ERR_COINCIDENT and the smallest (i, j) when a
 * target coincides with a source; 1: pairwise-mode semantics, r^2 == 0
 * pairs are skipped (summation.cpp:630).  Host pointers unless
 * VPG_DEVICE_POINTERS. */
int vpg_direct_sum(int family, double lambda, const double* src_xy,
                   const double* q, int64_t ns, const double* tgt_xy,
                   int64_t nt, double* out, int skip_coincident,
                   int64_t* clash_i, int64_t* clash_j, int device,
                   unsigned flags, void* stream);

/* K0 on the device (kernel.cpp:167-172); x <= 0 -> VPG_ERR_DOMAIN with the
 * reference message.  Host arrays. */
int vpg_bessel_k0(const double* x, int64_t n, double* out, int device);

/* Correction map (potential.cpp:92-110, 446-462): out[t] += sum over blocks
 * k in [blk_off[t], blk_off[t+1]) of pool_row(blk_pool[k]) . f[node_off[cell]
 * ..]. Rows are a flat pool with pool_off CSR (shared box-lattice rows are
 * stored once). */
int vpg_corr_create(int64_t nt, const int32_t* blk_off, int64_t nblocks,
                    const int32_t* blk_cell, const int32_t* blk_pool,
                    int64_t npool, const int64_t* pool_off,
                    const double* pool_vals, int64_t ncell,
                    const int32_t* node_off, int device, vpg_corr** corr);
/* f: ndofs samples, out: nt values accumulated into (out += C f). */
int vpg_corr_apply(const vpg_corr* corr, const double* f, int64_t nf,
                   double* out, unsigned flags, void* stream);
int vpg_corr_destroy(vpg_corr* corr);

/* build_charges (potential.cpp:397-412): charges[src_off[c] + s] =
 * src_wj[...] * sum_i O_type(c)[s][i] f[node_off[c] + i].  Two cell types
 * (0 = box, 1 = triangle), O row-major nq x np. */
int vpg_charges_create(int64_t ncell, const int32_t* cell_type,
                       const int32_t* node_off, const int32_t* src_off,
                       const double* over0, int np0, int nq0,
                       const double* over1, int np1, int nq1,
                       const double* src_wj, int device, vpg_charges** ch);
int vpg_charges_apply(const vpg_charges* ch, const double* f, int64_t nf,
                      double* charges, unsigned flags, void* stream);
int vpg_charges_destroy(vpg_charges* ch);

/* The operator-level apply of VolumePotentialOperator::apply
 * (potential.cpp:431-470), device-resident end to end:
 *   out = plan.apply(build_charges(f)) + C f
 * with the charge map, the plan and the correction map borrowed (they must
 * outlive the operator; ch may be NULL when the plan's sources are the
 * samples themselves with unit weights, i.e. charges = f).  The operator
 * owns persistent device buffers, so its FMM step replays the plan's cached
 * CUDA graph.  timings_ms (may be NULL) receives {smooth, correction} in
 * milliseconds, split like ApplyTimings (smooth includes build_charges,
 * potential.cpp:440-444); asking for timings synchronises. */
int vpg_operator_create(const vpg_plan* plan, const vpg_charges* ch, const vpg_corr* corr,
                        vpg_operator** op);
int vpg_operator_apply(const vpg_operator* op, const double* f, int64_t nf, double* out,
                       unsigned flags, void* stream, float* timings_ms);
int vpg_operator_destroy(vpg_operator* op);

/* Correction-row generation on the device: the rows of the
 * operator's correction map, built by VolumePotentialOperator::Impl::
 * build_corrections (potential.cpp:133-349) from SingularTargetRule::row
 * (singular.cpp:383-415), reduce_to_rays + apply_ray_quadrature
 * (singular.cpp:274-310), box_correction_table (singular.cpp:586-646) and
 * smooth_potential_row (singular.cpp:428-456).
 *
 * vpg_rows_create takes the mesh the rows integrate over: curves (kind 0
 * circle {cx, cy, r}, 1 ellipse {cx, cy, a, b, angle}, 2 star {cx, cy, r0,
 * amp, arms, phase}; 6 doubles each, geometry.hpp:31-72), cells (type 0
 * straight triangle, 1 curved triangle, 2 box; cell_curve the curve of a
 * curved cell; cell_v 3 vertices, cell_t (ta, tb), cell_ch (centre, h):
 * geometry.hpp:90-100), and the basis data of order p and source order q
 * (TriangleBasisTable nodes and C, BoxBasisTable C, the triangle source rule:
 * basis.hpp:13-56; row-major).  The context owns device copies. */
typedef struct vpg_rows vpg_rows;
int vpg_rows_create(int family, double lambda, int p, int q, int64_t ncurve, const int32_t* curve_kind,
                    const double* curve_par, int64_t ncell, const int32_t* cell_type, const int32_t* cell_curve,
                    const double* cell_v, const double* cell_t, const double* cell_ch, const double* tri_nodes,
                    const double* tri_C, const double* box_C, int64_t ntri_src, const double* tri_src_xy,
                    const double* tri_src_w, int device, vpg_rows** rows);
int vpg_rows_destroy(vpg_rows* rows);
/* One of the context's 1-D rules (0 Gauss-Legendre 16, 1 / 2 the 20-point
 * Gauss rules for -t log t / t, 3 the singular ray rule, 4.. the near ray
 * rules per decade bucket -2..9): x, w may be NULL to size. */
int vpg_rows_rule(const vpg_rows* rows, int which, double* x, double* w, int64_t* n);
/* Row tasks (host arrays, one entry per task): job 0 self rule at zeta0,
 * 1 ray rule (zeta0, zstar), 2 smooth row (aux 30: the 30x30 box rule),
 * 3..6 operator rows (TriSelfNode with aux = node, TriNearSnap, SelfGeneric,
 * NearGeneric: potential.cpp:157-333, geometry resolved on the device),
 * 7 lattice row (aux = offset * 256 + node, r0 = the node's point; the table
 * for lattice_h), 8/9 lattice-table entries; cell -1 = the reference box.
 * Rows are written back to back (p*p for box cells, p(p+1)/2 otherwise);
 * out = NULL only sizes (*out_len). */
int vpg_rows_eval(vpg_rows* rows, int64_t ntask, const int32_t* job, const int32_t* cell, const int32_t* aux,
                  const double* r0, const double* zeta0, const double* zstar, double lattice_h, double* out,
                  int64_t* out_len);

/* The whole correction map of VolumePotentialOperator (build_corrections,
 * potential.cpp:133-349) for targets tgt_xy: classify_target with near
 * distance D * h (mesh.cpp:410-448) on the device, the reference's task list
 * and pool slots on the host (node-coincident targets found by exact bits in
 * nodes_xy, the dof layout of mesh_nodes with node_off per cell; shared box
 * lattice rows), every row on the device; the map is created on the rows
 * context's device.  stats (may be NULL, 13 doubles): classification ms,
 * task/table ms, row ms, blocks, pool rows, pool doubles, then the block
 * counts of TriSelfNode, TriNearSnap, SelfGeneric, NearGeneric, BoxLattice,
 * then the quadrature nodes the row kernels evaluated on triangle and on box
 * cells (13 doubles).
 * Errors: the reference's classify_target messages (VPG_ERR_INVALID_ARGUMENT). */
int vpg_corr_build(vpg_rows* rows, int64_t ndofs, const double* nodes_xy, const int32_t* node_off, int64_t nt,
                   const double* tgt_xy, double D, vpg_corr** corr, double* stats);
/* The context's mesh mapped on the host: which = 0 the order-p interpolation
 * nodes of every cell in cell order (mesh_nodes, potential.cpp:63-74: xy);
 * 1 the order-q source rule (build_sources, potential.cpp:133-151: xy and
 * w * jacobian).  *n receives the point count; xy / wj may be NULL. */
int vpg_rows_map(const vpg_rows* rows, int which, double* xy, double* wj, int64_t* n);
/* Copies a correction map back to the host (any pointer may be NULL);
 * sizes (5 int64, may be NULL): nt, nblocks, npool, pool doubles, ndofs. */
int vpg_corr_export(const vpg_corr* corr, int32_t* blk_off, int32_t* blk_cell, int32_t* blk_pool,
                    int64_t* pool_off, double* pool_vals, int64_t* sizes);

/* Double-layer potential at volume targets, eval_layer_potential
 * (bie.hpp:87-90, bie.cpp:383-468): the trapezoidal Nystrom sum of every
 * curve, the 8x trig-upsampled rule within 5 node spacings (bie.cpp:414-
 * 440), plus the log-completion terms of the holes (bie.cpp:443-446).
 * A curve block carries the BoundarySystem::CurveBlock fields the
 * evaluation reads (bie.hpp:30-47): n nodes (even, >= 16) with interleaved
 * xy positions and outward normals and speeds, the 8n-point refined
 * geometry, total arclength, node-set diameter and log_center (holes). */
typedef struct vpg_layer vpg_layer;
typedef struct {
    int n;
    int offset; /* first density coefficient of the curve */
    double length;
    double diam;
    const double* x;           /* [n][2] */
    const double* normal;      /* [n][2] */
    const double* speed;       /* [n] */
    const double* fine_x;      /* [8n][2] */
    const double* fine_normal; /* [8n][2] */
    const double* fine_speed;  /* [8n] */
    double log_center[2];
} vpg_curve_block;
/* Uploads the boundary geometry once (the BoundarySystem is immutable). */
int vpg_layer_create(int family, double lambda, const vpg_curve_block* curves,
                     int ncurves, int n_density, int n_aux, int device,
                     vpg_layer** layer);
/* coeffs: n_density + n_aux values (density then log coefficients);
 * targets nt interleaved xy.  Errors with the reference messages:
 * "eval_layer_potential: coefficient length mismatch", "... target lies on a
 * boundary node", "... target inside the close-evaluation collar ..."
 * (VPG_ERR_INVALID_ARGUMENT; the on-node error wins when both occur).
 * The call always synchronises its stream before returning: the reject
 * rules are decided on the device and reported through the status. */
int vpg_layer_eval(const vpg_layer* layer, const double* coeffs,
                   int64_t ncoeffs, const double* tgt_xy, int64_t nt,
                   int allow_close, double* out, unsigned flags, void* stream);
int vpg_layer_destroy(vpg_layer* layer);

#ifdef __cplusplus
}
#endif
#endif /* VOLPOT_B200_H */
