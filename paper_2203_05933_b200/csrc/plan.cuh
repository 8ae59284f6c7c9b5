// plan.cuh -- device-resident SummationPlan state (the pimpl behind the
// C ABI; the reference keeps the same information in SummationPlan::Impl,
// summation.cpp:542-549).
#pragma once

#include <memory>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace vpg {

// Owning device buffer (cudaMalloc at plan build; plans are immutable).
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) VPG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// M2L work unit: a run of consecutive non-empty target boxes (one level)
// whose interaction lists together hold <= kM2LPairs entries.
struct M2LBatch {
    int32_t level;
    int32_t tfirst;  // index into the concatenated target-box list
    int32_t tcount;
    int32_t efirst;  // first list entry
    int32_t ecount;
};
constexpr int kP2PCoopSources = 768;  // neighbourhood size for CTA-cooperative chunks
constexpr int kM2LPairs = 54;  // two interior target boxes (27 each); 2 * pairs columns

// P2M work unit: the sources [e0, e1) (Morton-sorted) of one box at one
// level; direct = the box is a single item (write the expansion in place).
struct P2MItem {
    int32_t level;
    int32_t box;    // Morton id at `level` (centre)
    int32_t row;    // expansion row (mult + row * (P+1))
    int32_t e0, e1;
    int32_t direct;
};
// A box whose sources span several items: partials summed in item order.
struct P2MSplit {
    int32_t row;
    int32_t first;
    int32_t count;
};
constexpr int kP2MItemCap = 256;  // sources per P2M item

// P2P work unit: up to chunk targets of one leaf (Morton-sorted order).
struct P2PChunk {
    int32_t tbegin;
    int32_t tcount;
    int32_t pad;     // neighbourhood source count (schedule cost estimate)
    int32_t rfirst;  // near source ranges [rfirst, rfirst + rcount) in near_ranges
    int32_t rcount;  // <= kMaxNearRanges
    int32_t rself;   // index (within the list) of the target's own leaf
    int32_t lfirst;  // local-expansion rows the targets evaluate (L2P chain):
    int32_t lcount;  //   l2p_rows[lfirst, lfirst + lcount), leaf first
    int32_t part;    // split chunks: this task's share of the flat source list,
    int32_t nparts;  //   part of nparts (1 = whole chunk, written directly)
    int32_t slot;    //   counter of the split chunk (last finisher reduces)
    int32_t pbase;   //   first partial-sum row of the split chunk
};
constexpr int kMaxNearRanges = 64;

// Symmetric near field (uniform Laplace or Chebyshev-FMM Helmholtz trees whose first ns targets are the
// sources, the volume-potential case "targets = nodes"): every unordered pair
// of near points is evaluated ONCE -- log r^2 feeds target i (with q_j) and
// target j (with q_i).  Leaf A owns the pairs {A, B} with its neighbours B
// when it is the larger leaf (ties: smaller Morton id); its flat column list
// is A itself, then the owned neighbours.  The (rows of A) x (columns) block
// is cut into subtasks of one row group (whole tiles of 32 R rows) x one
// column chunk, sized to the GPU's fair share.  A subtask writes its
// partials: row sums of A's targets into A's row slot of the chunk, column
// sums (accumulated over the group's row tiles) into the column target's
// slot for (owner A, row group).  Each (target, slot) has exactly one
// writer and the final per-target sum runs over the leaf's slots in a fixed
// order (fmm.cu, p2p_sym_kernel / sym_finalize_kernel).  Partial layout per
// leaf A: pbase(A) + slot * n_A + k; slots: A's column chunks (row sums),
// A's row groups (self columns), then per owning neighbour its row groups.
struct SymTask {
    int32_t a_src, na;     // rows: leaf A's sources = its first na targets
    int32_t r0, r1;        // row group [r0, r1): whole row tiles of 32 R rows
    int32_t c0, c1;        // flat column chunk [c0, c1) (multiples of 32, c1 may be ncol)
    int32_t rfirst, rcount;  // column ranges sym_ranges[rfirst, +rcount), the first is A
    int64_t a_part;        // row partial of row i: part[a_part + i]
    int32_t rg, rows2;     // row group index (column slots: b_part + rg * nb); R = 1 << rows2
};
struct SymRange {
    int32_t b_src, coff, nb, pad;  // sorted source of the range, flat offset, leaf size
    int64_t b_part;                // column j -> part[b_part + rt * nb + (j - coff)]
};
struct SymLeaf {
    int64_t pbase;   // first partial of the leaf
    int32_t tgt, n;  // first matched target (sorted) and count
    int32_t nslot;
    int32_t t1;      // end of the leaf's targets: [tgt + n, t1) are unmatched
    int32_t rfirst, rcount;  // the leaf's 3x3 source ranges in near_ranges (unmatched targets)
    int32_t lfirst, lcount;  // the leaf's L2P chain in l2p_rows (the fused far field of sym_finalize_kernel)
};
constexpr int kSymMaxN = 4096;    // largest leaf (sources) the symmetric path takes
constexpr int kSymMaxRanges = 9;
// most rows per lane of the Laplace symmetric kernel (sym.cuh; tree.cu picks R per leaf
// size up to this).  8 is built on request only: on cfg4 it measured slower than 4 (5.20 vs
// 4.71 ms: three warps per scheduler leave fixed-latency waits exposed and the eight extra
// diagonal-tile instances cost instruction fetches), on cfg3's 4,096-point leaves 3% faster.
#ifndef VPG_SYM_MAXR
#define VPG_SYM_MAXR 4
#endif
constexpr int kSymLapMaxR = VPG_SYM_MAXR;
// M2L by offset (m2lgrid.cu): up to 32 target boxes of one level and one position in the parent
struct GridTile {
    int32_t level, cls, first, count;  // first: index into gt_rows / gt_nbr rows
};

struct LeafNear {  // per-leaf near-field data of the last schedule (host)
    int32_t leaf, t0, t1, rfirst, rcount, rself, lfirst, lcount;
};

// One captured apply (CUDA graph) with its own persistent workspace, keyed
// by the device pointers it was captured for (host-pointer applies use the
// entry's staging buffers).  `done` orders successive uses of the entry.
struct GraphEntry {
    const double* q = nullptr;
    double* out = nullptr;
    bool host = false;
    void* work = nullptr;
    double* qstage = nullptr;
    double* ostage = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;
    uint64_t last_use = 0;
    int64_t launches = 0;
    GraphEntry() = default;
    GraphEntry(const GraphEntry&) = delete;
    GraphEntry& operator=(const GraphEntry&) = delete;
    ~GraphEntry() {
        if (done) cudaEventSynchronize(done);
        if (exec) cudaGraphExecDestroy(exec);
        if (done) cudaEventDestroy(done);
        if (work) cudaFree(work);
        if (qstage) cudaFree(qstage);
        if (ostage) cudaFree(ostage);
    }
};

struct Plan {
    int device = 0;
    int sm_count = 148;
    int shift_grid = 148;  // co-resident CTAs of the cooperative M2M/L2L passes
    int family = VPG_LAPLACE;
    int mode = VPG_MODE_REFERENCE;
    double lambda = 0.0, eps = 1e-12;
    int64_t ns = 0, nt = 0;
    bool direct = true;
    int L = 0, P = 0;
    double x0 = 0, y0 = 0, side = 1;

    // Original-order points (pairwise mode) and Morton-sorted points.
    DBuf<double2> src, tgt;
    DBuf<double2> src_sorted, tgt_sorted;
    DBuf<int32_t> src_off, src_ids, tgt_off, tgt_ids;  // leaf CSR
    DBuf<int32_t> src_cnt, tgt_cnt;                    // all levels
    // Expansion rows: every box that carries an expansion has a row
    // (mult/loc + row * (P+1)).  Uniform trees: levels 2..L dense, row =
    // exp_off[l]/(P+1) + Morton id.  Adaptive trees: one row per box.
    DBuf<int32_t> row_level, row_morton, row_parent;  // parent = -1 above level 2
    int64_t n_rows = 0;
    DBuf<int32_t> tgt_row;  // leaf row of every Morton-sorted target

    // M2L lists (levels 2..L concatenated): target boxes and entries.
    std::vector<int64_t> lvl_tfirst;  // per level: first target-box index
    DBuf<int32_t> m2l_tbox, m2l_toff, m2l_src, m2l_oidx;
    int64_t n_tbox = 0, n_m2l = 0;
    DBuf<M2LBatch> m2l_batches;
    int64_t n_m2l_batches = 0;
    // uniform trees: the by-offset M2L schedule (m2lgrid.cu); 0 tiles: m2l_kernel runs the batches
    DBuf<GridTile> gt_tiles;
    DBuf<int32_t> gt_rows, gt_nbr, gt_oidx;  // target rows; [row][27] source rows or -1; [4][27] offset ids
    int64_t n_gt_tiles = 0;

    // Laplace operators (summation.cpp:150-222), uploaded once.
    DBuf<double> m2m_ops, l2l_ops;  // binomial triangles of the factorised M2M / L2L
    DBuf<double> h_t;               // H^T: P x RP (k-major), real
    DBuf<double2> dpow;             // 49 x (2P+1): d^-j per offset
    DBuf<double2> logmd;            // 49: log(-d)
    DBuf<double2> m2l_canon;        // 7 x (P+1): c^-j for the canonical offsets
    DBuf<int32_t> m2l_omap;         // 49: offset -> canonical | conj<<3 | quarter turns<<4
    int RP = 0;                     // rows padded to a multiple of 8
    int KP = 0;                     // P padded to a multiple of 4 (DMMA k-steps)

    // Upward/downward expansion level sizes.
    std::vector<int64_t> exp_off;  // per level offset (in complex) into scratch
    DBuf<int64_t> exp_off_dev;
    int64_t exp_total = 0;         // complex count for one of mult/loc

    // P2P schedule.
    int p2p_tpt = 1;
    DBuf<P2PChunk> p2p_chunks;
    DBuf<int2> near_ranges;  // (first sorted source, count) per near leaf
    // Laplace near field: (target, own-leaf source) pairs with r^2 zero or
    // subnormal, CSR over sorted targets (fmm.cu, build_coincidences)
    DBuf<int32_t> coin_off, coin_src;
    bool coin_ready = false;
    // symmetric near field (see SymTask); unmatched targets are summed
    // one-sided by sym_finalize_kernel (p2p_chunks keeps every target for L2P)
    bool matched = false;  // tgt[0, ns) == src bitwise (set at plan creation)
    bool sym = false;
    int32_t sym_min = -1;   // whole-tree choice: -1 off, 0 every pair symmetric, T: pairs of leaves >= T (hybrid)
    bool sym_hybrid = false;
    DBuf<P2PChunk> hyb_chunks;  // hybrid: one-sided chunks over the non-symmetric ranges
    DBuf<int2> hyb_ranges;
    int64_t n_hyb_chunks = 0;
    DBuf<SymTask> sym_tasks;
    DBuf<SymRange> sym_ranges;
    DBuf<SymLeaf> sym_leaves;
    int64_t n_sym_tasks = 0, n_sym_leaves = 0;
    bool sym_unmatched = false;  // some leaf has targets beyond its sources (summed one-sided in the finalize)
    int64_t sym_nparts = 0;   // partial doubles per apply
    int32_t sym_chunk = 0;    // column chunk (whole-tree decision, shards reuse it)
    bool sym_l2p_single = false;  // every symmetric leaf evaluates one local expansion (its own)
    double sym_fair = 0.0;    // pairs per subtask (whole-tree decision)
    // translation-invariant leaves (lattice.cu): the near field as dense GEMMs K_o . q on the
    // FP64 tensor cores; sym_leaves then holds one-slot leaves for the finalize
    bool lat = false;
    int lat_m = 0, lat_nt = 64;   // points per leaf, column tile of the kernel
    int64_t lat_ncol = 0;         // target leaves of the schedule
    double lat_pairs_exec = 0.0;  // m^2 x 9 x leaves: multiply-adds per apply (boundary zeros included)
    DBuf<double> lat_K;           // [9][m / 32][32][m + 4]
    DBuf<int32_t> lat_nbr;        // [leaf][9]: first sorted charge of the neighbour leaf, -1 outside
    // lattice P2M: power sums of the pattern by one GEMM, per-leaf binomial shift (lattice.cu)
    bool lat_p2m = false;
    int64_t lat_p2m_ncol = 0, lat_near_parts = 0;
    int lat_shift_terms = 0;      // the shift series keeps k - i <= this
    DBuf<double> lat_V;           // [m / 32][32][128 + 4]: re / im rows of w0^i
    DBuf<double> lat_binom;       // [51][51] binomial coefficients of the shift
    DBuf<int32_t> lat_p2m_src, lat_p2m_rows;  // per non-empty leaf: first sorted charge, multipole row
    DBuf<double2> lat_drift;      // per non-empty leaf: (translation - box-centre offset) / box side
    std::vector<LeafNear> h_leafnear;
    int64_t n_p2p_chunks = 0;
    int64_t n_p2p_heavy = 0;  // split chunks (counters)
    int64_t n_p2p_parts = 0;  // partial-sum rows of the split chunks
    double near_fair = 0.0;   // split threshold, fixed by the whole-tree schedule
                              // (shards must split chunks identically)
    int64_t p2p_pairs = 0;
    int64_t m2m_children = 0, l2l_children = 0;

    // Leaf ids with src_cnt > 0 (P2M work list) and parents per level for
    // M2M (src_cnt > 0) / L2L (tgt_cnt > 0).
    DBuf<P2MItem> p2m_items;
    int64_t n_p2m_items = 0;
    DBuf<P2MSplit> p2m_splits;
    int64_t n_p2m_splits = 0;
    // Multilevel passes (small problems): P2M at every level instead of the
    // M2M chain, L2P of every ancestor instead of the L2L chain -- one
    // launch each instead of one per level (tree.cu, choose_passes).
    bool multilevel_up = false, multilevel_down = false;
    // Uniform trees: hybrid pass thresholds.  A box with <= up_cap sources
    // gets its multipole by direct P2M, a larger non-leaf box by M2M; a
    // non-leaf box with > dn_cap targets pushes its local down by L2L, the
    // others are evaluated directly on the L2P chain.  0 = the classical
    // chain (summation.cpp:257-267, 305-312), INT32_MAX = multilevel.
    int32_t up_cap = 0, dn_cap = 0;
    // Adaptive trees (VPG_MODE_NATIVE, adaptive.cu): W-list M2P and X-list
    // P2L work on top of the V (M2L) and U (near-field) lists.
    bool adaptive = false;
    DBuf<int4> m2p_work;    // (target begin, count, first W row, W count)
    DBuf<int32_t> m2p_rows;
    int64_t n_m2p_work = 0, m2p_evals = 0;
    DBuf<int4> p2l_work;    // (receiving row, first range, range count, 0)
    // adaptive shards (vpg_plan_set_shard): host copies of the full
    // target-side schedules, filtered per target range
    std::vector<int4> ad_rng;             // per row (src begin, end, tgt begin, end)
    std::vector<int32_t> ad_level, ad_vc;
    std::vector<int64_t> ad_vp;
    int64_t ad_nv = 0;
    std::vector<P2PChunk> ad_chunks;      // unsplit near-field chunks
    std::vector<int4> ad_m2p, ad_p2l;     // full M2P / P2L work
    std::vector<int32_t> ad_ud_boxes;     // M2M parents, then L2L parents (rows)
    std::vector<int4> ad_ud_kids;
    std::vector<int64_t> ad_m2m_first, ad_m2m_count, ad_l2l_first, ad_l2l_count;
    std::vector<int32_t> ad_leaves;       // leaves with targets, in target order (shard units)
    DBuf<int2> p2l_ranges;  // X-leaf source ranges
    int64_t n_p2l_work = 0, p2l_sources = 0;
    std::vector<int64_t> m2m_first, m2m_count;  // into updown_boxes, per level
    std::vector<int64_t> l2l_first, l2l_count;
    DBuf<int32_t> updown_boxes;  // parent rows of the M2M / L2L passes
    DBuf<double2> shift_tab;      // [4][P+1] t_c^j, then [4][P+1] (2 t_c)^-j
    int KPd = 0;                  // L2L k-extent (multiple of 4, >= P+1)
    // adaptive trees: child rows per quadrant (-1 = no child / empty) of the
    // updown_boxes parents, and the L2P ancestor chain (next row whose local
    // expansion a target still evaluates; -1 once the parent pushed its local
    // down by L2L)
    DBuf<int4> updown_kids;
    DBuf<int32_t> row_chain;
    DBuf<int32_t> l2p_rows;  // per-leaf L2P chains (P2PChunk::lfirst/lcount)

    // Modified Helmholtz, native mode: compressed Chebyshev-interpolation FMM
    // (helm.cu, build_helm_fmm): n x n Chebyshev nodes per box at levels
    // hf_lmin..L, M2L through a rank-k SVD basis per level.
    bool hf = false;
    int hf_n = 0, hf_k = 0, hf_lmin = 0;
    bool hf_k0_fast = false;   // near-field K0 by the series (every near pair has lambda r <= 1)
    int hf_k0_deg = 9;         // series degree of that form (k0_series_degree)
    double hf_k0_qmax = 0.25;  // bound of q = (lambda r / 2)^2 over the near pairs
    DBuf<double> hf_tab;            // nodes[n], bw[n], S[2][n][n]
    DBuf<double> hf_Vt, hf_Vc;      // per level: V as [n2][k] (row-major) and [k][n2]
    DBuf<double> hf_C;              // per level and offset: C [k][k], C[j*k + i] = C_ij
    std::vector<int64_t> hf_V_off, hf_C_off, hf_row_base;  // per level
    DBuf<int32_t> hf_tbox, hf_toff, hf_esrc, hf_eop;       // M2L target rows CSR; entries (src row, C block)
    std::vector<int64_t> hf_lvl_t0;                        // per level first index into hf_tbox
    std::vector<std::vector<int2>> hf_offs;                // per level: the M2L offsets (T - S in box units)
    DBuf<int32_t> hf_srcof;  // per level [targets][offsets]: source row or -1
    DBuf<int4> hf_tiles;     // M2L tiles, 2 x int4: (first target, count, srcof base, noff),
                             // (first offset, end offset, partial slot or -1, C block base)
    DBuf<int2> hf_splits;    // split targets: (target row, first partial slot); nparts per split
    int64_t hf_ntiles = 0, hf_nsplit = 0, hf_nparts = 0;
    int hf_split_parts = 0;
    int64_t hf_rows = 0, hf_ntbox = 0, hf_nent = 0;

    // Modified Helmholtz (treecode) state.
    int helm_min_level = 2;
    double helm_skip_x = 40.0;
    std::vector<int> helm_m;          // per level
    DBuf<double> helm_nodes;          // per level, 32 slots
    DBuf<double> helm_bw;             // per level, 32 slots
    std::vector<int64_t> helm_w_off;  // per level offset into proxy weights
    int64_t helm_w_total = 0;

    // Host copies used to (re)build the schedules (tree.cu build_schedules).
    std::vector<int32_t> h_tflag, h_ecount;   // per box of levels 2..L
    std::vector<int64_t> h_epos, h_tpos;
    std::vector<int32_t> h_scnt, h_tcnt, h_soff, h_toff;
    int64_t shard_lb = 0, shard_le = 0, shard_m2l = 0;
    int64_t shard_t0 = 0, shard_t1 = 0;  // Morton-sorted target range of the shard

    // Profiling.
    bool profiling = false;
    mutable std::mutex prof_mu;
    mutable float phase_ms[VPG_PHASE_COUNT] = {};
    mutable std::atomic<int64_t> last_launches{0};  // written by concurrent applies
    // CUDA-graph cache of the apply (api.cu); declared last so it is torn
    // down before the buffers it references
    mutable std::mutex graph_mu;
    mutable std::vector<std::unique_ptr<GraphEntry>> graphs;
    mutable uint64_t graph_clock = 0;
    mutable uint32_t host_rr = 0;   // host-pointer applies alternate between two staged graphs
    mutable bool graph_broken = false;  // capture unsupported: plain launches

    int64_t device_bytes() const;
};

// tree.cu
void build_tree(Plan& pl);
void build_schedules(Plan& pl, int64_t leaf_begin, int64_t leaf_end);
void schedule_near_chunks(Plan& pl, std::vector<P2PChunk>& chunks);
void build_sym_near(Plan& pl, int64_t leaf_begin, int64_t leaf_end);
void choose_passes(Plan& pl);
// adaptive.cu
void build_adaptive(Plan& pl, cudaStream_t st);
void adaptive_set_targets(Plan& pl, int64_t leaf_begin, int64_t leaf_end);  // shard
// fmm.cu
void build_laplace_ops(Plan& pl);
struct LaplaceWork {
    double* qs;
    double2* mult;
    double2* loc;
    double* pot_far;
    int* ticket;
    double* partial_p2p;
    int* pcount;
    double2* p2m_partial;
    double* sym_part;  // slot partials of the symmetric near field (SymLeaf::pbase)
};
size_t laplace_work_bytes(const Plan& pl);
LaplaceWork laplace_work_at(const Plan& pl, void* base);
void laplace_issue(const Plan& pl, const double* q_dev, double* out_dev, const LaplaceWork& w,
                   cudaStream_t st, cudaEvent_t* ev, int64_t& launches, cudaStream_t side,
                   cudaEvent_t fork, cudaEvent_t join, cudaEvent_t far_done);
void laplace_apply(const Plan& pl, const double* q_dev, double* out_dev,
                   cudaStream_t st, cudaEvent_t* ev, int64_t& launches);
// direct.cu
void pairwise_apply(const Plan& pl, const double* q_dev, double* out_dev,
                    cudaStream_t st, int64_t& launches);
void direct_sum_device(int family, double lambda, const double2* src,
                       const double* q, int64_t ns, const double2* tgt,
                       int64_t nt, double* out, bool skip,
                       unsigned long long* clash, cudaStream_t st);
// helm.cu
void build_helm_ops(Plan& pl);
void build_m2l_grid(Plan& pl, int64_t lb, int64_t le);  // m2lgrid.cu
void m2l_grid_issue(const Plan& pl, const double2* mult, double2* loc, cudaStream_t st);
bool build_lattice_near(Plan& pl, int64_t lb, int64_t le);  // lattice.cu
void lattice_near_issue(const Plan& pl, const double* qs, double* near, cudaStream_t st);
void lattice_p2m_issue(const Plan& pl, const double* qs, double* S, double2* mult, cudaStream_t st);
void build_helm_fmm(Plan& pl);  // native mode (helm.cu)
void hf_build_m2l(Plan& pl, int64_t lb, int64_t le);  // its M2L schedule for the targets of a leaf range
size_t helm_work_bytes(const Plan& pl);  // Chebyshev FMM apply scratch (helm.cu)
void helm_fmm_issue(const Plan& pl, const double* q_dev, double* out_dev, void* work, cudaStream_t st,
                    cudaEvent_t* ev, int64_t& launches, cudaStream_t side, cudaEvent_t fork, cudaEvent_t join,
                    cudaEvent_t far_done);
void helm_apply(const Plan& pl, const double* q_dev, double* out_dev,
                cudaStream_t st, cudaEvent_t* ev, int64_t& launches);
void k0_device(const double* x, int64_t n, double* out, cudaStream_t st);
void ensure_k0_table();

}  // namespace vpg
