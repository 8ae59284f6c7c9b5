// api.cu -- the extern "C" boundary (include/volpot_b200.h): argument
// checks with the reference's error semantics, device selection, per-device
// tables, stream handling and host<->device staging around the kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "k0.cuh"

#include "maps.cuh"
#include "plan.cuh"

struct vpg_plan {
    vpg::Plan impl;
};

namespace vpg {

namespace {
thread_local std::string t_err;
std::mutex g_mu;
struct DeviceTables {
    double2* log_tab = nullptr;
    double2* log_tab2 = nullptr;  // fast_log's table (round-to-nearest centres)
    double2* log_tab3 = nullptr;  // trunc_log's table (mid-point centres)
    double* k0_tab = nullptr;
    double* k0f_tab = nullptr;
    double* k1_tab = nullptr;
};
std::map<int, DeviceTables> g_tables;
std::map<std::pair<const void*, int>, int> g_optin;  // (kernel, device) -> opted-in dynamic smem
std::set<int> g_ready;
}  // namespace

void set_error(const std::string& msg) { t_err = msg; }
const char* get_error() { return t_err.c_str(); }

void use_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        (void)cudaGetLastError();
        throw Error{VPG_ERR_CUDA, std::string("no CUDA device available: ") +
                                      (e == cudaSuccess ? "device count 0" : cudaGetErrorString(e))};
    }
    if (device < 0 || device >= count)
        throw Error{VPG_ERR_INVALID_ARGUMENT, "device " + std::to_string(device) + " out of range"};
    VPG_CUDA(cudaSetDevice(device));
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_ready.count(device)) return;
    cudaDeviceProp prop;
    VPG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw Error{VPG_ERR_CUDA, std::string("libvolpot_b200 is built for sm_100a; device is ") +
                                      prop.name + " sm_" + std::to_string(prop.major) +
                                      std::to_string(prop.minor)};
    // Keep stream-ordered scratch in the pool between applies.
    cudaMemPool_t pool;
    VPG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~uint64_t(0);
    VPG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_ready.insert(device);
}

static DeviceTables& tables_locked(int dev) {
    DeviceTables& t = g_tables[dev];
    if (!t.log_tab) {
        // (RN(1/c), -ln RN(1/c)) at the centres c = 1 + i/256, i = 0..256
        std::vector<double2> h(kLogTableSize);
        for (int i = 0; i < kLogTableSize; ++i) {
            const long double c = 1.0L + (long double)i / (kLogTableSize - 1);
            const double inv = double(1.0L / c);
            h[size_t(i)] = make_double2(inv, double(-std::log((long double)inv)));
        }
        VPG_CUDA(cudaMalloc(&t.log_tab, sizeof(double2) * h.size()));
        VPG_CUDA(cudaMemcpy(t.log_tab, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    }
    if (!t.log_tab2) {
        // centres c = 1 + i/512 (fast_log): (RN(1/c), -ln RN(1/c) - i ln2/512)
        std::vector<double2> h(kLogTableSize);
        const long double ln2_512 = (long double)kLn2Over512;
        for (int i = 0; i < kLogTableSize; ++i) {
            const long double c = 1.0L + (long double)i / (kLogTableSize - 1);
            const double inv = double(1.0L / c);
            h[size_t(i)] = make_double2(inv, double(-std::log((long double)inv) - (long double)i * ln2_512));
        }
        VPG_CUDA(cudaMalloc(&t.log_tab2, sizeof(double2) * h.size()));
        VPG_CUDA(cudaMemcpy(t.log_tab2, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    }
    if (!t.log_tab3) {
        // centres c = 1 + (i + 1/2)/512 (trunc_log): (RN(1/c), -ln RN(1/c) - i ln2/512);
        // entry 512 is never indexed (the index is the truncated mantissa)
        std::vector<double2> h(kLogTableSize);
        const long double ln2_512 = (long double)kLn2Over512;
        for (int i = 0; i < kLogTableSize; ++i) {
            const long double c = 1.0L + ((long double)i + 0.5L) / (kLogTableSize - 1);
            const double inv = double(1.0L / c);
            h[size_t(i)] = make_double2(inv, double(-std::log((long double)inv) - (long double)i * ln2_512));
        }
        VPG_CUDA(cudaMalloc(&t.log_tab3, sizeof(double2) * h.size()));
        VPG_CUDA(cudaMemcpy(t.log_tab3, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    }
    if (!t.k0_tab) {
        std::vector<double> h(size_t(kK0Intervals) * kK0Coeffs);
        k0_fit_host(h.data());
        VPG_CUDA(cudaMalloc(&t.k0_tab, sizeof(double) * h.size()));
        VPG_CUDA(cudaMemcpy(t.k0_tab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    }
    if (!t.k1_tab) {
        std::vector<double> h(size_t(kK0Intervals) * kK0Coeffs);
        k1_fit_host(h.data());
        VPG_CUDA(cudaMalloc(&t.k1_tab, sizeof(double) * h.size()));
        VPG_CUDA(cudaMemcpy(t.k1_tab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    }
    if (!t.k0f_tab) {
        std::vector<double> h(size_t(kK0FastIntervals) * kK0FastStride, 0.0);
        k0_fit_fast_host(h.data());
        VPG_CUDA(cudaMalloc(&t.k0f_tab, sizeof(double) * h.size()));
        VPG_CUDA(cudaMemcpy(t.k0f_tab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    }
    return t;
}

const double2* log_table_dev() {
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).log_tab;
}
const double2* lap_log_table_rn_dev() {
#if VPG_LOG_FOLD
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).log_tab2;
#else
    return log_table_dev();
#endif
}
const double2* lap_log_table_dev() {
#if VPG_LOG_FOLD && VPG_LOG_TRUNC
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).log_tab3;
#else
    return lap_log_table_rn_dev();
#endif
}
const double* k0_fast_table_dev() {
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).k0f_tab;
}
const double* k1_table_dev() {
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).k1_tab;
}
const double* k0_table_dev() {
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    return tables_locked(dev).k0_tab;
}

void smem_optin(const void* func, int bytes) {
    int dev = 0;
    VPG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_optin.find({func, dev});
    if (it != g_optin.end() && it->second >= bytes) return;  // raised only, never lowered
    VPG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    g_optin[{func, dev}] = bytes;
}

int64_t Plan::device_bytes() const {
    return int64_t(src.bytes() + tgt.bytes() + src_sorted.bytes() + tgt_sorted.bytes() +
                   src_off.bytes() + src_ids.bytes() + tgt_off.bytes() + tgt_ids.bytes() +
                   src_cnt.bytes() + tgt_cnt.bytes() + m2l_tbox.bytes() + m2l_toff.bytes() +
                   m2l_src.bytes() + m2l_oidx.bytes() + m2l_batches.bytes() + m2m_ops.bytes() +
                   l2l_ops.bytes() + h_t.bytes() + dpow.bytes() + logmd.bytes() +
                   p2p_chunks.bytes() + near_ranges.bytes() + row_level.bytes() + row_morton.bytes() +
                   row_parent.bytes() + tgt_row.bytes() + p2m_items.bytes() + p2m_splits.bytes() + updown_boxes.bytes() + updown_kids.bytes() + row_chain.bytes() +
                   helm_nodes.bytes() + helm_bw.bytes() + exp_off_dev.bytes() + sym_tasks.bytes() + sym_ranges.bytes() +
                   sym_leaves.bytes() + lat_K.bytes() + lat_nbr.bytes() + lat_V.bytes() + lat_binom.bytes() +
                   lat_p2m_src.bytes() + lat_p2m_rows.bytes() + lat_drift.bytes() + gt_tiles.bytes() + gt_rows.bytes() +
                   gt_nbr.bytes() + gt_oidx.bytes());
}

// Runs f, mapping exceptions to status codes + thread-local message.
template <typename F>
int guarded(F&& f) {
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

// Stream to run on: the caller's, or a private one for this call.
struct CallStream {
    cudaStream_t s = nullptr;
    bool owned = false;
    explicit CallStream(void* user) {
        if (user) {
            s = static_cast<cudaStream_t>(user);
        } else {
            // blocking: orders after work already queued on the legacy
            // default stream (e.g. a q written there by the caller)
            VPG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamDefault));
            owned = true;
        }
    }
    ~CallStream() {
        if (owned) cudaStreamDestroy(s);
    }
};

template <typename T>
struct Scratch {  // stream-ordered device scratch
    T* p = nullptr;
    cudaStream_t s;
    Scratch(size_t n, cudaStream_t st) : s(st) {
        if (n) VPG_CUDA(cudaMallocAsync(&p, n * sizeof(T), st));
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

// Graph-cached Laplace apply: the kernel sequence of laplace_issue is
// captured into a CUDA graph and replayed with one cudaGraphLaunch -- at
// ~0.5 ms per step the dozen launches and stream-ordered allocations of a
// plain apply cost ~10%.  Entries are keyed by the (q, out) device pointers
// they were captured for (host-pointer applies use the entry's own staging
// buffers).  At most kMaxGraphs entries per plan, each with its persistent
// workspace allocated once: a new pointer pair beyond that re-captures into
// the least recently used entry of the same kind and patches its executable
// in place (cudaGraphExecUpdate, in-flight launches unaffected), so steady
// state applies with fresh output tensors never allocate, free or
// instantiate.  Caller holds pl.graph_mu.
constexpr size_t kMaxGraphs = 4;

bool plan_is_sharded(const Plan& pl) {
    if (pl.adaptive) return pl.shard_t0 != 0 || pl.shard_t1 != pl.nt;
    return pl.shard_lb != 0 || pl.shard_le != (int64_t(1) << (2 * pl.L));
}

// Captures laplace_issue (or helm_fmm_issue) for e's pointers; nullptr when
// capture is not supported here (the caller falls back to plain launches).
static cudaGraph_t capture_apply(const Plan& pl, GraphEntry& e) {
    const double* qd = e.host ? e.qstage : e.q;
    double* od = e.host ? e.ostage : e.out;
    cudaStream_t cap = nullptr, side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, far_done = nullptr;
    static const bool prio = [] {  // VPG_PRIO=0: equal priorities (A/B)
        const char* v = std::getenv("VPG_PRIO");
        return !(v && v[0] == '0');
    }();
    if (prio) {  // far-field chain ahead of the side-stream near field (cfg2: -3%)
        int lo = 0, hi = 0;
        VPG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VPG_CUDA(cudaStreamCreateWithPriority(&cap, cudaStreamNonBlocking, hi));
        VPG_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
    } else {
        VPG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        VPG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    }
    VPG_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    VPG_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    VPG_CUDA(cudaEventCreateWithFlags(&far_done, cudaEventDisableTiming));
    struct StreamGuard {
        cudaStream_t s, t;
        cudaEvent_t f, j, d;
        ~StreamGuard() {
            cudaStreamDestroy(s);
            cudaStreamDestroy(t);
            cudaEventDestroy(f);
            cudaEventDestroy(j);
            cudaEventDestroy(d);
        }
    } sg{cap, side, fork, join, far_done};
    VPG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t g = nullptr;
    try {
        if (plan_is_sharded(pl) && pl.nt)
            VPG_CUDA(cudaMemsetAsync(od, 0, sizeof(double) * size_t(pl.nt), cap));
        static const bool no_fork = [] {
            const char* v = std::getenv("VPG_NO_FORK");
            return v && v[0] == '1';
        }();
        int64_t launches = 0;
        if (pl.family == VPG_LAPLACE)
            laplace_issue(pl, qd, od, laplace_work_at(pl, e.work), cap, nullptr, launches,
                          no_fork ? nullptr : side, fork, join, far_done);
        else
            helm_fmm_issue(pl, qd, od, e.work, cap, nullptr, launches, no_fork ? nullptr : side, fork, join,
                           far_done);
        e.launches = launches;
    } catch (...) {
        cudaStreamEndCapture(cap, &g);
        if (g) cudaGraphDestroy(g);
        (void)cudaGetLastError();
        return nullptr;
    }
    VPG_CUDA(cudaStreamEndCapture(cap, &g));
    return g;
}

static bool instantiate(GraphEntry& e, cudaGraph_t g) {
    const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, cudaGraphInstantiateFlagUseNodePriority);
    if (ie != cudaSuccess) {
        (void)cudaGetLastError();
        e.exec = nullptr;
        return false;
    }
    return true;
}

GraphEntry* graph_entry(const Plan& pl, const double* q, double* out, bool host) {
    for (auto& e : pl.graphs)
        if (e->host == host && e->q == q && e->out == out) return e.get();
    GraphEntry* lru = nullptr;
    size_t same_kind = 0;
    for (auto& e : pl.graphs) {
        if (e->host != host) continue;
        ++same_kind;
        if (!lru || e->last_use < lru->last_use) lru = e.get();
    }
    if (lru && (same_kind >= kMaxGraphs - 1 || pl.graphs.size() >= kMaxGraphs)) {
        // re-target the least recently used entry: same workspace, patched exec
        lru->q = q;
        lru->out = out;
        cudaGraph_t g = capture_apply(pl, *lru);
        if (!g) return nullptr;
        cudaGraphExecUpdateResultInfo info;
        bool ok = cudaGraphExecUpdate(lru->exec, g, &info) == cudaSuccess;
        if (!ok) {
            (void)cudaGetLastError();
            VPG_CUDA(cudaEventSynchronize(lru->done));  // not in flight before it goes
            cudaGraphExecDestroy(lru->exec);
            ok = instantiate(*lru, g);
        }
        cudaGraphDestroy(g);
        if (!ok) return nullptr;
        return lru;
    }
    auto e = std::make_unique<GraphEntry>();
    e->q = q;
    e->out = out;
    e->host = host;
    VPG_CUDA(cudaMalloc(&e->work, pl.family == VPG_LAPLACE ? laplace_work_bytes(pl) : helm_work_bytes(pl)));
    if (host) {
        VPG_CUDA(cudaMalloc(&e->qstage, sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1))));
        VPG_CUDA(cudaMalloc(&e->ostage, sizeof(double) * size_t(std::max<int64_t>(pl.nt, 1))));
    }
    VPG_CUDA(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
    cudaGraph_t g = capture_apply(pl, *e);
    if (!g) return nullptr;
    const bool ok = instantiate(*e, g);
    cudaGraphDestroy(g);
    if (!ok) return nullptr;
    pl.graphs.push_back(std::move(e));
    return pl.graphs.back().get();
}

bool graphs_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("VPG_NO_GRAPH");
        return !(v && v[0] == '1');
    }();
    return on;
}

}  // namespace vpg

using namespace vpg;

extern "C" {

const char* vpg_last_error(void) { return get_error(); }
int vpg_abi_version(void) { return VPG_ABI_VERSION; }

int vpg_device_count(int* count) {
    return guarded([&] {
        if (!count) throw Error{VPG_ERR_INVALID_ARGUMENT, "count is NULL"};
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            (void)cudaGetLastError();
            n = 0;
        }
        int usable = 0;
        for (int d = 0; d < n; ++d) {
            cudaDeviceProp p;
            if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++usable;
        }
        *count = usable;
    });
}

int vpg_plan_create(int family, double lambda, const double* src_xy, int64_t ns,
                    const double* tgt_xy, int64_t nt, double epsilon, int mode,
                    int device, vpg_plan** plan) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        *plan = nullptr;
        if (family != VPG_LAPLACE && family != VPG_MODIFIED_HELMHOLTZ)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown kernel family"};
        if (family == VPG_MODIFIED_HELMHOLTZ && !(lambda > 0.0))  // kernel.cpp:195-196
            throw Error{VPG_ERR_INVALID_ARGUMENT, "make_kernel: modified Helmholtz needs lambda > 0"};
        if (ns < 0 || nt < 0 || (ns > 0 && !src_xy) || (nt > 0 && !tgt_xy))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "bad point arrays"};
        if (ns > INT32_MAX || nt > INT32_MAX)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "point count exceeds int32 indexing"};
        if (mode != VPG_MODE_REFERENCE && mode != VPG_MODE_NATIVE)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown tree mode"};
        use_device(device);
        auto holder = std::make_unique<vpg_plan>();
        Plan& pl = holder->impl;
        pl.device = device;
        VPG_CUDA(cudaDeviceGetAttribute(&pl.sm_count, cudaDevAttrMultiProcessorCount, device));
        pl.family = family;
        pl.lambda = family == VPG_LAPLACE ? 0.0 : lambda;
        pl.mode = mode;
        pl.eps = std::min(std::max(epsilon, 1e-12), 1e-3);  // summation.cpp:557
        if (std::isnan(epsilon)) pl.eps = 1e-12;
        pl.ns = ns;
        pl.nt = nt;
        pl.src.alloc(size_t(ns));
        pl.tgt.alloc(size_t(nt));
        if (ns) VPG_CUDA(cudaMemcpy(pl.src.p, src_xy, sizeof(double2) * size_t(ns), cudaMemcpyHostToDevice));
        if (nt) VPG_CUDA(cudaMemcpy(pl.tgt.p, tgt_xy, sizeof(double2) * size_t(nt), cudaMemcpyHostToDevice));
        // "targets = nodes": the first ns targets are the sources, bitwise
        // (enables the symmetric near field, plan.cuh SymTask)
        pl.matched = ns > 0 && ns <= nt && std::memcmp(src_xy, tgt_xy, sizeof(double2) * size_t(ns)) == 0;
        build_tree(pl);
        if (!pl.direct) {
            if (family == VPG_LAPLACE) {
                build_laplace_ops(pl);
            } else {
                build_helm_ops(pl);                           // reference treecode
                if (mode == VPG_MODE_NATIVE) build_helm_fmm(pl);  // Chebyshev FMM when applicable
            }
        }
        (void)log_table_dev();
        (void)lap_log_table_dev();
        (void)k0_table_dev();
        VPG_CUDA(cudaDeviceSynchronize());
        *plan = holder.release();
    });
}

int vpg_plan_apply(const vpg_plan* plan, const double* q, int64_t nq, double* out,
                   unsigned flags, void* stream) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        const Plan& pl = plan->impl;
        if (nq != pl.ns)  // summation.cpp:613-617
            throw Error{VPG_ERR_INVALID_ARGUMENT,
                        "SummationPlan::apply: charge count " + std::to_string(nq) +
                            " does not match source count " + std::to_string(pl.ns)};
        if ((pl.ns > 0 && !q) || (pl.nt > 0 && !out))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL charge or output array"};
        VPG_CUDA(cudaSetDevice(pl.device));
        CallStream cs(stream);
        cudaStream_t st = cs.s;
        const bool dev = flags & VPG_DEVICE_POINTERS;
        if (!pl.direct && (pl.family == VPG_LAPLACE || pl.hf) && !pl.profiling && graphs_enabled()) {
            std::unique_lock<std::mutex> lk(pl.graph_mu);
            // host pointers: two staged graphs used in turn, so applies issued on
            // two streams overlap one's copies with the other's kernels
            const double* hkey = reinterpret_cast<const double*>(uintptr_t(1 + (pl.host_rr++ & 1u)));
            GraphEntry* e = pl.graph_broken ? nullptr : graph_entry(pl, dev ? q : hkey, dev ? out : nullptr, !dev);
            if (e) {
                e->last_use = ++pl.graph_clock;
                VPG_CUDA(cudaStreamWaitEvent(st, e->done, 0));  // previous use of this workspace
                if (!dev && pl.ns)
                    VPG_CUDA(cudaMemcpyAsync(e->qstage, q, sizeof(double) * size_t(pl.ns), cudaMemcpyHostToDevice, st));
                VPG_CUDA(cudaGraphLaunch(e->exec, st));
                if (!dev && pl.nt)
                    VPG_CUDA(cudaMemcpyAsync(out, e->ostage, sizeof(double) * size_t(pl.nt), cudaMemcpyDeviceToHost, st));
                VPG_CUDA(cudaEventRecord(e->done, st));
                pl.last_launches.store(e->launches, std::memory_order_relaxed);
                lk.unlock();
                if (!(flags & VPG_NO_SYNC) || cs.owned) VPG_CUDA(cudaStreamSynchronize(st));
                return;
            }
            pl.graph_broken = true;
        }
        Scratch<double> qd(dev ? 0 : size_t(pl.ns), st), od(dev ? 0 : size_t(pl.nt), st);
        const double* q_dev = dev ? q : qd.p;
        double* out_dev = dev ? out : od.p;

        const bool prof = pl.profiling;
        cudaEvent_t ev[VPG_PHASE_COUNT + 1] = {};
        if (prof)
            for (auto& e : ev) VPG_CUDA(cudaEventCreate(&e));
        struct EvGuard {
            cudaEvent_t* e;
            bool on;
            ~EvGuard() {
                if (on)
                    for (int i = 0; i <= VPG_PHASE_COUNT; ++i) cudaEventDestroy(e[i]);
            }
        } eg{ev, prof};
        // event i marks the start of phase i; ev[PHASE_COUNT] the end
        if (prof) VPG_CUDA(cudaEventRecord(ev[VPG_PHASE_UPLOAD], st));
        if (!dev && pl.ns)
            VPG_CUDA(cudaMemcpyAsync(qd.p, q, sizeof(double) * size_t(pl.ns), cudaMemcpyHostToDevice, st));
        int64_t launches = 0;
        cudaEvent_t* inner = prof ? ev + 1 : nullptr;  // GATHER .. DOWNLOAD
        if (!pl.direct && plan_is_sharded(pl) && pl.nt)
            VPG_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double) * size_t(pl.nt), st));
        if (pl.direct) {
            if (prof)
                for (int i = 0; i < 6; ++i) VPG_CUDA(cudaEventRecord(inner[i], st));
            pairwise_apply(pl, q_dev, out_dev, st, launches);
            if (prof) VPG_CUDA(cudaEventRecord(inner[6], st));
        } else if (pl.family == VPG_LAPLACE) {
            laplace_apply(pl, q_dev, out_dev, st, inner, launches);
        } else {
            helm_apply(pl, q_dev, out_dev, st, inner, launches);
        }
        if (!dev && pl.nt)
            VPG_CUDA(cudaMemcpyAsync(out, od.p, sizeof(double) * size_t(pl.nt), cudaMemcpyDeviceToHost, st));
        if (prof) VPG_CUDA(cudaEventRecord(ev[VPG_PHASE_COUNT], st));
        const bool sync = !(flags & VPG_NO_SYNC) || cs.owned || prof;
        if (sync) VPG_CUDA(cudaStreamSynchronize(st));
        if (prof) {
            std::lock_guard<std::mutex> lk(pl.prof_mu);
            for (int i = 0; i < VPG_PHASE_COUNT; ++i)
                VPG_CUDA(cudaEventElapsedTime(&pl.phase_ms[i], ev[i], ev[i + 1]));
        }
        pl.last_launches.store(launches, std::memory_order_relaxed);
    });
}

int vpg_plan_info(const vpg_plan* plan, vpg_plan_info_t* info) {
    return guarded([&] {
        if (!plan || !info) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL argument"};
        const Plan& pl = plan->impl;
        vpg_plan_info_t r{};
        r.num_sources = pl.ns;
        r.num_targets = pl.nt;
        r.levels = pl.direct ? 0 : pl.L;
        r.expansion_order = pl.direct ? 0 : pl.P;
        r.family = pl.family;
        r.mode = pl.mode;
        r.device = pl.device;
        r.epsilon = pl.eps;
        r.x0 = pl.x0;
        r.y0 = pl.y0;
        r.side = pl.side;
        r.m2l_pairs = pl.direct ? 0 : pl.shard_m2l;
        r.p2p_pairs = pl.direct ? pl.ns * pl.nt : pl.p2p_pairs;
        r.m2m_children = pl.m2m_children;
        r.l2l_children = pl.l2l_children;
        r.device_bytes = pl.device_bytes();
        r.near_symmetric = pl.sym ? 1 : 0;
        r.near_lattice = pl.lat ? 1 : 0;
        *info = r;
    });
}

int vpg_plan_set_profiling(vpg_plan* plan, int on) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        plan->impl.profiling = on != 0;
    });
}

int vpg_plan_phase_times(const vpg_plan* plan, float* ms) {
    return guarded([&] {
        if (!plan || !ms) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL argument"};
        std::lock_guard<std::mutex> lk(plan->impl.prof_mu);
        std::memcpy(ms, plan->impl.phase_ms, sizeof(float) * VPG_PHASE_COUNT);
    });
}

int vpg_plan_last_launches(const vpg_plan* plan, int64_t* launches) {
    return guarded([&] {
        if (!plan || !launches) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL argument"};
        *launches = plan->impl.last_launches.load(std::memory_order_relaxed);
    });
}

int vpg_plan_dump_tree(const vpg_plan* plan, int32_t* src_off, int32_t* src_ids,
                       int32_t* tgt_off, int32_t* tgt_ids, int32_t* src_cnt,
                       int32_t* tgt_cnt) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        const Plan& pl = plan->impl;
        if (pl.direct) throw Error{VPG_ERR_INVALID_ARGUMENT, "pairwise plan has no tree"};
        if (pl.adaptive)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "adaptive (native) plan has no uniform leaf table"};
        VPG_CUDA(cudaSetDevice(pl.device));
        auto cp = [](int32_t* dst, const DBuf<int32_t>& s, size_t n) {
            if (dst && n) VPG_CUDA(cudaMemcpy(dst, s.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        };
        const size_t nleaf = size_t(1) << (2 * pl.L);
        cp(src_off, pl.src_off, nleaf + 1);
        cp(tgt_off, pl.tgt_off, nleaf + 1);
        cp(src_ids, pl.src_ids, size_t(pl.ns));
        cp(tgt_ids, pl.tgt_ids, size_t(pl.nt));
        cp(src_cnt, pl.src_cnt, size_t(lvl_base(pl.L + 1)));
        cp(tgt_cnt, pl.tgt_cnt, size_t(lvl_base(pl.L + 1)));
    });
}

int vpg_plan_dump_m2l(const vpg_plan* plan, int level, int32_t* ntbox, int64_t* nent,
                      int32_t* tbox, int32_t* toff, int32_t* src, int32_t* oidx) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        const Plan& pl = plan->impl;
        if (pl.direct || level < 2 || level > pl.L)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "level out of range"};
        if (pl.adaptive)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "adaptive (native) plan has no per-level M2L table"};
        VPG_CUDA(cudaSetDevice(pl.device));
        const int64_t t0 = pl.lvl_tfirst[size_t(level)], t1 = pl.lvl_tfirst[size_t(level + 1)];
        std::vector<int32_t> off(size_t(t1 - t0 + 1));
        VPG_CUDA(cudaMemcpy(off.data(), pl.m2l_toff.p + t0, off.size() * sizeof(int32_t),
                            cudaMemcpyDeviceToHost));
        const int64_t e0 = off.front(), e1 = off.back();
        if (ntbox) *ntbox = int32_t(t1 - t0);
        if (nent) *nent = e1 - e0;
        // lists hold expansion rows; report Morton ids of the level
        const int32_t rowbase = int32_t(lvl_base(level) - lvl_base(2));
        if (tbox && t1 > t0) {
            VPG_CUDA(cudaMemcpy(tbox, pl.m2l_tbox.p + t0, size_t(t1 - t0) * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < t1 - t0; ++i) tbox[i] -= rowbase;
        }
        if (toff)
            for (size_t i = 0; i < off.size(); ++i) toff[i] = int32_t(off[i] - e0);
        if (src && e1 > e0) {
            VPG_CUDA(cudaMemcpy(src, pl.m2l_src.p + e0, size_t(e1 - e0) * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < e1 - e0; ++i) src[i] -= rowbase;
        }
        if (oidx && e1 > e0)
            VPG_CUDA(cudaMemcpy(oidx, pl.m2l_oidx.p + e0, size_t(e1 - e0) * sizeof(int32_t),
                                cudaMemcpyDeviceToHost));
    });
}

int vpg_plan_set_shard(vpg_plan* plan, int64_t leaf_begin, int64_t leaf_end) {
    return guarded([&] {
        if (!plan) throw Error{VPG_ERR_INVALID_ARGUMENT, "plan is NULL"};
        Plan& pl = plan->impl;
        if (pl.direct) throw Error{VPG_ERR_INVALID_ARGUMENT, "pairwise plan cannot be sharded"};
        const int64_t nleaf = pl.adaptive ? int64_t(pl.ad_leaves.size()) : int64_t(1) << (2 * pl.L);
        if (leaf_begin < 0 || leaf_end > nleaf || leaf_begin > leaf_end)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "shard leaf range out of bounds"};
        VPG_CUDA(cudaSetDevice(pl.device));
        {
            std::lock_guard<std::mutex> lk(pl.graph_mu);
            pl.graphs.clear();  // captured schedules are stale
        }
        if (pl.adaptive) adaptive_set_targets(pl, leaf_begin, leaf_end);
        else build_schedules(pl, leaf_begin, leaf_end);
    });
}

int vpg_plan_shard_units(const vpg_plan* plan, int64_t* nunits, double* costs) {
    return guarded([&] {
        if (!plan || !nunits) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL argument"};
        const Plan& pl = plan->impl;
        if (pl.direct) throw Error{VPG_ERR_INVALID_ARGUMENT, "pairwise plan cannot be sharded"};
        const double P = pl.P;
        if (pl.adaptive) {
            *nunits = int64_t(pl.ad_leaves.size());
            if (!costs) return;
            std::map<int32_t, size_t> at;  // target begin -> leaf position
            for (size_t i = 0; i < pl.ad_leaves.size(); ++i) {
                at[pl.ad_rng[size_t(pl.ad_leaves[i])].z] = i;
                costs[i] = 0.0;
            }
            for (const P2PChunk& c : pl.ad_chunks) {
                auto it = at.upper_bound(c.tbegin);
                const size_t i = std::prev(it)->second;
                // near field + local evaluation of the chain + ~27 M2L entries
                costs[i] += double(c.tcount) * (double(c.pad) * 14.0 + 4.0 * (P + 1) * c.lcount) +
                            (c.tbegin == pl.ad_rng[size_t(pl.ad_leaves[i])].z ? 27.0 * 4.0 * P * (P + 1) : 0.0);
            }
            return;
        }
        const int L = pl.L;
        const int64_t nleaf = int64_t(1) << (2 * L);
        *nunits = nleaf;
        if (!costs) return;
        const int nb = 1 << L;
        for (int64_t b = 0; b < nleaf; ++b) {
            const int64_t ntgt = pl.h_toff[size_t(b) + 1] - pl.h_toff[size_t(b)];
            const int ix = int(squash2(uint32_t(b))), iy = int(squash2(uint32_t(b) >> 1));
            int64_t nsrc = 0;
            for (int jy = std::max(0, iy - 1); jy <= std::min(nb - 1, iy + 1); ++jy)
                for (int jx = std::max(0, ix - 1); jx <= std::min(nb - 1, ix + 1); ++jx) {
                    const uint32_t sid = mort(uint32_t(jx), uint32_t(jy));
                    nsrc += pl.h_soff[sid + 1] - pl.h_soff[sid];
                }
            costs[b] = double(ntgt) * double(nsrc) * 14.0 + double(ntgt) * 4.0 * (P + 1) +
                       (ntgt > 0 ? 27.0 * 4.0 * P * (P + 1) : 0.0);
        }
    });
}

int vpg_plan_destroy(vpg_plan* plan) {
    return guarded([&] {
        if (!plan) return;
        cudaSetDevice(plan->impl.device);
        delete plan;
    });
}

int vpg_direct_sum(int family, double lambda, const double* src_xy, const double* q,
                   int64_t ns, const double* tgt_xy, int64_t nt, double* out,
                   int skip_coincident, int64_t* clash_i, int64_t* clash_j, int device,
                   unsigned flags, void* stream) {
    return guarded([&] {
        if (family != VPG_LAPLACE && family != VPG_MODIFIED_HELMHOLTZ)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "unknown kernel family"};
        if (family == VPG_MODIFIED_HELMHOLTZ && !(lambda > 0.0))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "make_kernel: modified Helmholtz needs lambda > 0"};
        if (ns < 0 || nt < 0 || (ns && (!src_xy || !q)) || (nt && (!tgt_xy || !out)))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "direct_sum: points/charges size mismatch"};
        if (ns > INT32_MAX || nt > INT32_MAX)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "point count exceeds int32 indexing"};
        if (clash_i) *clash_i = -1;
        if (clash_j) *clash_j = -1;
        use_device(device);
        CallStream cs(stream);
        cudaStream_t st = cs.s;
        const bool dev = flags & VPG_DEVICE_POINTERS;
        Scratch<double2> sd(dev ? 0 : size_t(ns), st), td(dev ? 0 : size_t(nt), st);
        Scratch<double> qd(dev ? 0 : size_t(ns), st), od(dev ? 0 : size_t(nt), st);
        Scratch<unsigned long long> clash(1, st);
        const double2* s_p = dev ? reinterpret_cast<const double2*>(src_xy) : sd.p;
        const double2* t_p = dev ? reinterpret_cast<const double2*>(tgt_xy) : td.p;
        const double* q_p = dev ? q : qd.p;
        double* o_p = dev ? out : od.p;
        if (!dev) {
            if (ns) {
                VPG_CUDA(cudaMemcpyAsync(sd.p, src_xy, sizeof(double2) * size_t(ns), cudaMemcpyHostToDevice, st));
                VPG_CUDA(cudaMemcpyAsync(qd.p, q, sizeof(double) * size_t(ns), cudaMemcpyHostToDevice, st));
            }
            if (nt) VPG_CUDA(cudaMemcpyAsync(td.p, tgt_xy, sizeof(double2) * size_t(nt), cudaMemcpyHostToDevice, st));
        }
        VPG_CUDA(cudaMemsetAsync(clash.p, 0xFF, sizeof(unsigned long long), st));
        if (nt) {
            if (ns)
                direct_sum_device(family, lambda, s_p, q_p, ns, t_p, nt, o_p,
                                  skip_coincident != 0, clash.p, st);
            else
                VPG_CUDA(cudaMemsetAsync(o_p, 0, sizeof(double) * size_t(nt), st));
        }
        unsigned long long key = ~0ull;
        VPG_CUDA(cudaMemcpyAsync(&key, clash.p, sizeof(key), cudaMemcpyDeviceToHost, st));
        if (!dev && nt)
            VPG_CUDA(cudaMemcpyAsync(out, od.p, sizeof(double) * size_t(nt), cudaMemcpyDeviceToHost, st));
        VPG_CUDA(cudaStreamSynchronize(st));
        if (!skip_coincident && key != ~0ull) {  // summation.cpp:533-538
            const int64_t i = int64_t(key >> 32), j = int64_t(key & 0xFFFFFFFFull);
            if (clash_i) *clash_i = i;
            if (clash_j) *clash_j = j;
            throw Error{VPG_ERR_COINCIDENT, "direct_sum: target " + std::to_string(i) +
                                                " coincides with source " + std::to_string(j)};
        }
    });
}

int vpg_bessel_k0(const double* x, int64_t n, double* out, int device) {
    return guarded([&] {
        if (n < 0 || (n && (!x || !out))) throw Error{VPG_ERR_INVALID_ARGUMENT, "bad arrays"};
        for (int64_t i = 0; i < n; ++i)
            if (!(x[i] > 0.0))  // kernel.cpp:169
                throw Error{VPG_ERR_DOMAIN, "bessel_k0: argument must be positive"};
        use_device(device);
        CallStream cs(nullptr);
        Scratch<double> xd(size_t(n), cs.s), od(size_t(n), cs.s);
        if (n) VPG_CUDA(cudaMemcpyAsync(xd.p, x, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, cs.s));
        k0_device(xd.p, n, od.p, cs.s);
        if (n) VPG_CUDA(cudaMemcpyAsync(out, od.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, cs.s));
        VPG_CUDA(cudaStreamSynchronize(cs.s));
    });
}


struct vpg_operator {
    const vpg_plan* plan = nullptr;
    const vpg_charges* ch = nullptr;
    const vpg_corr* corr = nullptr;
    int device = 0;
    int64_t ndofs = 0, ns = 0, nt = 0;
    double* fd = nullptr;  // persistent device buffers: samples, charges, potentials
    double* qd = nullptr;
    double* od = nullptr;
    cudaEvent_t done = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    mutable std::mutex mu;
    ~vpg_operator() {
        if (done) cudaEventSynchronize(done);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (done) cudaEventDestroy(done);
        cudaFree(fd);
        cudaFree(qd);
        cudaFree(od);
    }
};

int vpg_operator_create(const vpg_plan* plan, const vpg_charges* ch, const vpg_corr* corr,
                        vpg_operator** op) {
    return guarded([&] {
        if (!plan || !corr || !op) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL argument"};
        const Plan& pl = plan->impl;
        const int64_t ndofs = corr->ndofs;
        if (corr->nt != pl.nt)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "operator: correction map has " + std::to_string(corr->nt) +
                                                      " targets, plan has " + std::to_string(pl.nt)};
        if (ch ? (ch->nsrc != pl.ns || ch->ndofs != ndofs) : (pl.ns != ndofs))
            throw Error{VPG_ERR_INVALID_ARGUMENT, "operator: charge map does not match the plan's sources"};
        if ((ch && ch->device != pl.device) || corr->device != pl.device)
            throw Error{VPG_ERR_INVALID_ARGUMENT, "operator: maps and plan on different devices"};
        VPG_CUDA(cudaSetDevice(pl.device));
        auto o = std::make_unique<vpg_operator>();
        o->plan = plan;
        o->ch = ch;
        o->corr = corr;
        o->device = pl.device;
        o->ndofs = ndofs;
        o->ns = pl.ns;
        o->nt = pl.nt;
        VPG_CUDA(cudaMalloc(&o->fd, sizeof(double) * size_t(std::max<int64_t>(ndofs, 1))));
        VPG_CUDA(cudaMalloc(&o->qd, sizeof(double) * size_t(std::max<int64_t>(pl.ns, 1))));
        VPG_CUDA(cudaMalloc(&o->od, sizeof(double) * size_t(std::max<int64_t>(pl.nt, 1))));
        VPG_CUDA(cudaEventCreateWithFlags(&o->done, cudaEventDisableTiming));
        for (cudaEvent_t& e : o->ev) VPG_CUDA(cudaEventCreate(&e));
        *op = o.release();
    });
}

int vpg_operator_apply(const vpg_operator* op, const double* f, int64_t nf, double* out,
                       unsigned flags, void* stream, float* timings_ms) {
    return guarded([&] {
        if (!op) throw Error{VPG_ERR_INVALID_ARGUMENT, "operator is NULL"};
        if (nf != op->ndofs)  // potential.cpp:434-438
            throw Error{VPG_ERR_INVALID_ARGUMENT,
                        "apply: expected " + std::to_string(op->ndofs) + " samples, got " + std::to_string(nf)};
        if ((nf > 0 && !f) || (op->nt > 0 && !out)) throw Error{VPG_ERR_INVALID_ARGUMENT, "NULL sample or output array"};
        VPG_CUDA(cudaSetDevice(op->device));
        CallStream cs(stream);
        cudaStream_t st = cs.s;
        const bool dev = flags & VPG_DEVICE_POINTERS;
        const unsigned dflags = VPG_DEVICE_POINTERS | VPG_NO_SYNC;
        std::lock_guard<std::mutex> lk(op->mu);  // persistent buffers: one use at a time per stream order
        VPG_CUDA(cudaStreamWaitEvent(st, op->done, 0));
        const double* fdev = dev ? f : op->fd;
        double* odev = dev ? out : op->od;
        if (!dev && nf)
            VPG_CUDA(cudaMemcpyAsync(op->fd, f, sizeof(double) * size_t(nf), cudaMemcpyHostToDevice, st));
        if (timings_ms) VPG_CUDA(cudaEventRecord(op->ev[0], st));
        // build_charges (potential.cpp:397-412) -> plan apply (potential.cpp:443)
        const double* q = fdev;
        if (op->ch) {
            const int rc = vpg_charges_apply(op->ch, fdev, nf, op->qd, dflags, st);
            if (rc) throw Error{rc, vpg_last_error()};
            q = op->qd;
        }
        int rc = vpg_plan_apply(op->plan, q, op->ns, odev, dflags, st);
        if (rc) throw Error{rc, vpg_last_error()};
        if (timings_ms) VPG_CUDA(cudaEventRecord(op->ev[1], st));
        // correction (potential.cpp:446-462): out += C f
        rc = vpg_corr_apply(op->corr, fdev, nf, odev, dflags, st);
        if (rc) throw Error{rc, vpg_last_error()};
        if (timings_ms) VPG_CUDA(cudaEventRecord(op->ev[2], st));
        if (!dev && op->nt)
            VPG_CUDA(cudaMemcpyAsync(out, op->od, sizeof(double) * size_t(op->nt), cudaMemcpyDeviceToHost, st));
        VPG_CUDA(cudaEventRecord(op->done, st));
        if (timings_ms || !(flags & VPG_NO_SYNC) || cs.owned || !dev) VPG_CUDA(cudaStreamSynchronize(st));
        if (timings_ms) {
            VPG_CUDA(cudaEventElapsedTime(&timings_ms[0], op->ev[0], op->ev[1]));
            VPG_CUDA(cudaEventElapsedTime(&timings_ms[1], op->ev[1], op->ev[2]));
        }
    });
}

int vpg_operator_destroy(vpg_operator* op) {
    return guarded([&] {
        if (!op) return;
        cudaSetDevice(op->device);
        delete op;
    });
}

}  // extern "C"
