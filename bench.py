#!/usr/bin/env python
"""FMM-step benchmark (BASELINE.json metric: source-target interactions/s, FP64).

A step is one SummationPlan::apply (summation.cpp:610-643) of the workload:
charges in -> potentials out at every target.  The default workload is cfg4
(BASELINE.json configs[3], 4,194,304 nodes: the largest configuration, one
GPU) at eps = 1e-12.

Interactions per step: for Laplace tree plans, the near-field
source-target pairs the reference enumerates (summation.cpp:330-344, the
3x3-leaf lists of its uniform L = 7 tree including the skipped self pairs:
9,563,275,264 at cfg4), the same count for both arms and both tree modes;
value = those pairs / the whole FMM-step time (far field included), so the
ratio to the reference arm is the step-time ratio.  Pairwise plans and the
modified-Helmholtz treecode have no near-field list: there a step counts
ns * nt.  kernels.p2p.pairs_per_s is the P2P-kernel-only rate.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4]
    python bench.py --impl reference ...   # the reference CPU code (oracle/_ref)

N > 1 runs under torchrun: every rank owns a Morton-contiguous shard of the
target leaves (balanced by near-field pair count), the upward pass is
replicated, there is no data-path collective inside the step (results stay
sharded), and the timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "source-target interactions/s (FP64) for the FMM step"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
DEFAULT_WORKLOAD = "cfg4"  # BASELINE.json configs[3]: the largest config, fits one GPU

THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


def fp64_peak_tflops(pipe="any"):
    """Measured FP64 peak on this pool's B200 (profiles/fp64_peak_r01.json):
    the DMMA (tensor) figure for tensor-core kernels, the DFMA figure for
    FP64 CUDA-core kernels, the larger of the two for "any"."""
    with open(FP64_PEAK_FILE) as f:
        rows = [json.loads(x) for x in f if x.strip()]
    dfma = max(r.get("fp64_dfma_tflops_best", 0.0) for r in rows)
    dmma = max(r.get("fp64_dmma_tflops_best", 0.0) for r in rows)
    return {"tensor": dmma, "fp64": dfma}.get(pipe, max(dfma, dmma))


def hbm_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)  # first sample in before the load starts
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mask = 0
        for r in self.rows:
            mask |= r[2]
        reasons = [n for b, n in THROTTLE_BITS.items() if mask & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows)}


def measured_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic_r02.json, else traffic_r01.json), or None when that workload was not captured."""
    for name in ("traffic_r02.json", "traffic_r01.json"):  # the latest capture that has the kernel
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
        try:
            with open(path) as f:
                v = json.load(f).get(workload, {}).get(kernel)
        except (OSError, ValueError):
            v = None
        if v is not None:
            return v
    return None


def load_workload(name):
    from paper_2203_05933_b200 import workloads as W
    return W.CONFIGS[name]()


def kernel_for(wl):
    import paper_2203_05933_b200 as vp
    if wl.kernel == "helmholtz":
        return vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, wl.lam)
    return vp.make_kernel(vp.KernelFamily.Laplace)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the sharded flow on a single-GPU box (VPG_BENCH_BACKEND=gloo):
    # ranks share device 0; timings from such a run are not scaling numbers
    if os.environ.get("VPG_BENCH_BACKEND") == "gloo":
        local = 0
    return world, rank, local


def dist_backend():
    return os.environ.get("VPG_BENCH_BACKEND", "nccl")


def interaction_count(wl, levels, p2p_pairs):
    """Interactions per step (module docstring): the reference near-field pair
    count for Laplace tree plans, ns * nt otherwise."""
    if wl.kernel == "laplace" and levels > 0:
        return float(p2p_pairs), "near-field pairs of the reference tree (summation.cpp:330-344)"
    return float(wl.ns) * float(wl.nt), "ns * nt (no near-field list: pairwise or treecode plan)"


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    wl = load_workload(args.workload)
    ref = oracle.reference()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    fam = 1 if wl.kernel == "helmholtz" else 0
    eps = min(wl.eps)
    plan = ref.plan(fam, wl.lam, wl.src, wl.tgt, eps)
    levels = plan.levels()
    pairs = 0
    if fam == 0 and levels > 0:  # the reference tree's near-field count (restated binning, summation.cpp:81-129)
        rest = oracle.restatement()
        tr = rest.tree(wl.src, wl.tgt, eps)
        pairs = rest.p2p_pairs(levels, tr["src_off"], tr["tgt_off"])
    inter, counted = interaction_count(wl, levels, pairs)
    for _ in range(args.warmup):
        plan.apply(wl.q)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        plan.apply(wl.q)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    v = inter / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "interactions/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        # the same keys as the GPU arm's config; the workload keys carry the same values
        "config": {"workload": args.workload, "ns": wl.ns, "nt": wl.nt, "epsilon": eps,
                   "levels": levels, "order": plan.expansion_order(), "mode": "reference",
                   "parallelism": "single" if world == 1 else f"target-shard{world}",
                   "interactions_per_step": inter, "interactions_counted": counted,
                   "l2": "host arm (no device L2 flush)",
                   "near_field": "pairwise (the reference's own loop, summation.cpp:330-344)",
                   "step": "FMM step: SummationPlan::apply (summation.cpp:610-643)"},
        "cpu_baseline": {"value": v, "unit": "interactions/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} full SummationPlan::apply of {args.workload} "
                                   f"(oracle/_ref = unmodified proj/src/summation.cpp, g++ -O3 "
                                   f"-march=native, set_thread_count({cores}))"},
        "e2e": {"value": v, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU arm
def cpu_baseline_sample(wl, inter, budget_s=20.0, corr=None):
    """oracle/_ref on the host cores: full applies, bounded to ~budget_s.
    Operator workloads (corr given): the CPU composition of
    VolumePotentialOperator::apply -- our restatement of
    build_charges (potential.cpp:397-412) + the reference SummationPlan::apply
    + our restatement of the correction loop (potential.cpp:446-462) on the
    same map, all on the host cores."""
    import oracle
    try:
        ref = oracle.reference()
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "interactions/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    fam = 1 if wl.kernel == "helmholtz" else 0
    plan = ref.plan(fam, wl.lam, wl.src, wl.tgt, min(wl.eps))
    t0 = time.perf_counter()
    plan.apply(wl.q)
    first = time.perf_counter() - t0
    n = max(1, min(5, int(budget_s / max(first, 1e-3))))
    times = []
    for _ in range(n):
        t0 = time.perf_counter()
        plan.apply(wl.q)
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    if corr is not None:
        from paper_2203_05933_b200 import rows as RW
        rest = oracle.restatement()
        mp = RW.export_map(corr["map"])
        ct, o0, o1 = corr["charges"]
        f = wl.notes["f"]
        t0 = time.perf_counter()
        qv = rest.build_charges(ct, corr["node_off"], corr["src_off"], o0, o1, wl.notes["src_wj"], f, threads=cores)
        t_ch = time.perf_counter() - t0
        t0 = time.perf_counter()
        rest.correction_apply(mp["blk_off"], mp["blk_cell"], mp["blk_pool"], mp["pool_off"], mp["pool_vals"],
                              corr["node_off"], f, np.zeros(wl.nt), threads=cores)
        t_co = time.perf_counter() - t0
        tt = t + t_ch + t_co
        return {"value": inter / tt, "unit": "interactions/s", "cores": cores, "kind": "reference",
                "ms_per_step": tt * 1e3, "split_ms": {"build_charges": t_ch * 1e3, "fmm": t * 1e3,
                                                      "correction": t_co * 1e3},
                "sample": f"operator apply composed on {cores} host threads: restated build_charges + median of "
                          f"{n} reference SummationPlan::apply (oracle/_ref) + restated correction loop on the "
                          f"same map; q max diff vs the workload charges "
                          f"{float(np.abs(qv - wl.q).max() / np.abs(wl.q).max()):.1e} (rel)"}
    return {"value": inter / t, "unit": "interactions/s", "cores": cores,
            "kind": "reference", "ms_per_step": t * 1e3,
            "sample": f"median of {n} full SummationPlan::apply of the workload after 1 warm-up "
                      f"(oracle/_ref, set_thread_count({cores}))"}


def run_gpu(args):
    import torch

    import paper_2203_05933_b200 as vp
    from paper_2203_05933_b200 import multigpu

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(dist_backend(), **({"device_id": torch.device("cuda", local)}
                                                   if dist_backend() == "nccl" else {}))

    wl = load_workload(args.workload)
    kern = kernel_for(wl)
    eps = args.eps if args.eps else min(wl.eps)
    plan = vp.SummationPlan(kern, wl.src, wl.tgt, eps, mode=args.mode, device=local)
    info_full = plan.info()  # the whole job's counts (value = all ranks' interactions / max time)
    shard = None
    if world > 1:
        shard = multigpu.shard_plan(plan, rank, world)
    info = plan.info()       # this rank's shard (kernel statistics of rank 0)
    # one explicit stream for the L2 flush, the events and every apply: the
    # default stream's handle is 0, which the library would replace by a
    # stream of its own (unordered with the flush, synchronised per call)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    q_d = torch.from_numpy(wl.q).to("cuda")
    out_d = torch.empty(wl.nt, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MB > L2

    # cfg5 (BASELINE configs[4]) includes the correction apply: the step is
    # the operator-level apply (potential.cpp:431-470) -- build_charges
    # (q = w f, identity oversampling) -> FMM step -> + C f
    op = None
    corr_info = None
    if "mesh" in wl.notes and world == 1:
        # the reference's own operator layout on its hybrid mesh: correction
        # map built on the device (build_corrections, csrc/rows.cu), the
        # tensor-core build_charges with the reference oversampling matrices
        from paper_2203_05933_b200 import rows as RW
        m, b = wl.notes["mesh"], wl.notes["basis"]
        pp, qq = wl.notes["p"], wl.notes["q"]
        mesh = RW.Mesh(m["type"], m["curve"], m["v"], m["tt"], m["ch"], np.array([RW.CURVE_STAR]),
                       m["star"][None, :])
        fam = 1 if wl.kernel == "helmholtz" else 0
        eng = RW.RowEngine(mesh, fam, wl.lam, pp, qq, b["tri_nodes"], b["tri_C"], b["box_C"], b["tri_src"],
                           b["tri_src_w"], device=local)
        box = m["type"] == 2
        node_off = np.concatenate([[0], np.cumsum(np.where(box, pp * pp, pp * (pp + 1) // 2))]).astype(np.int32)
        src_off = np.concatenate([[0], np.cumsum(np.where(box, b["box_over"].shape[0],
                                                          b["tri_over"].shape[0]))]).astype(np.int32)
        torch.cuda.synchronize()
        t_cb = time.perf_counter()
        cm, cst = RW.build_correction_map(eng, wl.tgt, node_off, wl.tgt)
        corr_build_ms = (time.perf_counter() - t_cb) * 1e3
        ch = vp.ChargeMap(np.where(box, 0, 1).astype(np.int32), node_off, src_off, b["box_over"], b["tri_over"],
                          wl.notes["src_wj"], device=local)
        op = vp.VolumePotentialOperator(plan, cm, ch)
        f_np = np.ascontiguousarray(wl.notes["f"], dtype=np.float64)
        f_d = torch.from_numpy(f_np).to("cuda")
        corr_info = {"build_ms": corr_build_ms, "stats": cst, "node_off": node_off, "src_off": src_off,
                     "map": cm, "charges": (np.where(box, 0, 1).astype(np.int32), b["box_over"], b["tri_over"])}
    elif "corr" in wl.notes and world == 1:
        csr = wl.notes["corr"]()
        ncell = csr["node_off"].size - 1
        cm = vp.CorrectionMap(csr["blk_off"], csr["blk_cell"], csr["blk_pool"], csr["pool_off"],
                              csr["pool_vals"], csr["node_off"], device=local)
        ch = vp.ChargeMap(np.zeros(ncell, np.int32), csr["node_off"], csr["node_off"], np.eye(64),
                          np.zeros((0, 0)), wl.notes["w"], device=local)
        op = vp.VolumePotentialOperator(plan, cm, ch)
        f_np = np.ascontiguousarray(wl.notes["f"], dtype=np.float64)
        f_d = torch.from_numpy(f_np).to("cuda")

    def step():
        if op is not None:
            op.apply_device(f_d.data_ptr(), out_d.data_ptr(), sh)
        else:
            plan.apply_device(q_d.data_ptr(), out_d.data_ptr(), sh)

    # clocks are sampled (every 100 ms) from the first warm-up step to the end
    # of the timed region; untimed steps keep the GPU loaded for >= 0.5 s
    # first, so the samples see clocks under load
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    t_hold = time.time()
    while time.time() - t_hold < 0.5:
        for _ in range(8):
            flush.zero_()
            step()
        torch.cuda.synchronize()

    # ---- timed region: K device-resident steps, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.sum(step_ms)) / args.steps
    launches_per_step = plan.last_launches()
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- phase split (profiled pass, same protocol, events inside the library)
    plan.set_profiling(True)
    phases = {k: 0.0 for k in ("gather", "p2m", "m2m", "m2l", "l2l", "p2p")}
    for _ in range(args.steps):
        flush.zero_()
        plan.apply_device(q_d.data_ptr(), out_d.data_ptr(), sh)
        pt = plan.phase_times()
        for k in phases:
            phases[k] += pt[k] / args.steps
    plan.set_profiling(False)
    if op is not None:  # the correction share of the operator apply (ApplyTimings split)
        corr_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            corr_ms += op.apply(f_np, timings=True)[1]["correction_ms"] / args.steps
        phases["correction"] = corr_ms

    # ---- end to end through the C ABI with pinned HOST buffers (H2D + D2H inside).
    # A caller streaming independent charge vectors issues its applies on two
    # streams with two pinned buffer pairs (the library alternates two staged
    # graphs for host pointers), so one apply's copies overlap the other's
    # kernels; every step still copies its own q in and its own result out
    # inside the timed region.  The one-stream (serial) figure is reported too.
    src_h = (wl.q if op is None else f_np)
    q_hs = [torch.from_numpy(src_h.copy()).pin_memory() for _ in range(2)]
    out_hs = [torch.empty(wl.nt, dtype=torch.float64).pin_memory() for _ in range(2)]
    q_h, out_h = q_hs[0], out_hs[0]
    host_apply = plan.apply_host_ptr if op is None else op.apply_host_ptr
    streams = [stream, torch.cuda.Stream()]
    for k in range(max(2, args.warmup)):
        host_apply(q_hs[k & 1].data_ptr(), out_hs[k & 1].data_ptr(),
                   streams[(k & 1) if op is None else 0].cuda_stream, sync=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    # the L2 flush runs between steps on the issuing stream; a concurrent flush would
    # steal the other stream's bandwidth, so plans whose per-step working set
    # (points, expansions, partials) is several times L2 skip it (info device_bytes)
    big = info["device_bytes"] > 4 * 126 * 1024 * 1024
    for i in range(args.steps):
        sk = streams[(i & 1) if op is None else 0]
        if not big:
            with torch.cuda.stream(sk):
                flush.zero_()
        host_apply(q_hs[i & 1].data_ptr(), out_hs[i & 1].data_ptr(), sk.cuda_stream, sync=False)
    j1 = torch.cuda.Event()
    j1.record(streams[1])
    streams[0].wait_event(j1)
    e1.record(streams[0])
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if op is not None:  # the operator's persistent buffers serialise its applies: no two-stream figure
        e2e_ms = None
    # serial: one stream, each apply's copies and kernels back to back
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        e2e_ev[i][0].record(stream)
        host_apply(q_h.data_ptr(), out_h.data_ptr(), sh, sync=False)
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = float(np.sum([a.elapsed_time(b) for a, b in e2e_ev])) / args.steps
    # copy/compute pipeline through the device-pointer API: step i's H2D (own
    # copy stream) runs under step i-1's apply and its D2H (another copy stream)
    # under step i+1's, applies themselves back to back on one stream
    e2e_pipe_ms = None
    if op is None:
        q_d2 = [torch.empty(wl.ns, dtype=torch.float64, device="cuda") for _ in range(2)]
        o_d2 = [torch.empty(wl.nt, dtype=torch.float64, device="cuda") for _ in range(2)]
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        ev_h2d = [torch.cuda.Event() for _ in range(2)]
        ev_app = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]

        def pipe(nsteps, record=None):
            for i in range(nsteps):
                k = i & 1
                with torch.cuda.stream(h2d_s):
                    if i >= 2:
                        h2d_s.wait_event(ev_app[k])  # the apply of step i-2 read q_d2[k]
                    q_d2[k].copy_(q_hs[k], non_blocking=True)
                    ev_h2d[k].record(h2d_s)
                stream.wait_event(ev_h2d[k])
                if i >= 2:
                    stream.wait_event(ev_d2h[k])     # o_d2[k] of step i-2 copied out
                with torch.cuda.stream(stream):
                    flush.zero_()
                plan.apply_device(q_d2[k].data_ptr(), o_d2[k].data_ptr(), sh)
                ev_app[k].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(ev_app[k])
                    out_hs[k].copy_(o_d2[k], non_blocking=True)
                    ev_d2h[k].record(d2h_s)

        pipe(max(2, args.warmup))
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        h2d_s.wait_event(p0)
        pipe(args.steps)
        j1 = torch.cuda.Event()
        j1.record(d2h_s)
        stream.wait_event(j1)
        p1.record(stream)
        torch.cuda.synchronize()
        e2e_pipe_ms = p0.elapsed_time(p1) / args.steps
    cands = {"one stream": e2e_serial_ms}
    if e2e_ms is not None:
        cands["applies alternating over two streams"] = e2e_ms
    if e2e_pipe_ms is not None:
        cands["copy/compute pipeline (H2D and D2H streams around device-pointer applies)"] = e2e_pipe_ms
    e2e_mode = min(cands, key=cands.get)
    e2e_ms = cands[e2e_mode]
    two_stream = e2e_mode != "one stream"
    if dist:
        t = torch.tensor([e2e_ms, e2e_serial_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, e2e_serial_ms = (float(x) for x in t.tolist())

    # parity spot check of this very run against the device-resident result
    step()
    torch.cuda.synchronize()
    host_res = out_h.numpy()
    dev_res = out_d.cpu().numpy()
    if shard is None and not np.array_equal(host_res, dev_res) and not os.environ.get("VPG_BENCH_ABLATION"):
        raise RuntimeError("host-pointer and device-pointer applies differ")  # VPG_BENCH_ABLATION: timing-ablation builds

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    ref_pairs = info_full["p2p_pairs"]
    if args.mode == "native" and wl.kernel == "laplace":
        # the workload's count is the reference tree's, whatever tree runs
        with vp.SummationPlan(kern, wl.src, wl.tgt, eps, mode="reference", device=local) as rp:
            ref_pairs = rp.info()["p2p_pairs"]
    inter, counted = interaction_count(wl, info["levels"] if args.mode == "reference" else 1, ref_pairs)
    value = inter / (ms * 1e-3)
    P = info["expansion_order"]
    peak = fp64_peak_tflops()
    kern_stats = {}
    if info["levels"] > 0 and wl.kernel == "laplace":
        m2l_flops = info["m2l_pairs"] * (4.0 * P * (P + 1) + 8.0 * (P + 1) + 6.0 * P)
        m2l_dense = info["m2l_pairs"] * 8.0 * (P + 1) ** 2
        p2p_flops = info["p2p_pairs"] * 27.0
        kern_stats["m2l"] = {"ms": phases["m2l"], "pairs": info["m2l_pairs"],
                             "tflops_executed": m2l_flops / (phases["m2l"] * 1e-3) / 1e12 if phases["m2l"] else None,
                             "tflops_dense_equiv": m2l_dense / (phases["m2l"] * 1e-3) / 1e12 if phases["m2l"] else None}
        kern_stats["p2p"] = {"ms": phases["p2p"], "pairs": info["p2p_pairs"],
                             "pairs_per_s": info["p2p_pairs"] / (phases["p2p"] * 1e-3) if phases["p2p"] else None,
                             "tflops_27": p2p_flops / (phases["p2p"] * 1e-3) / 1e12 if phases["p2p"] else None}
        dom = "m2l" if phases["m2l"] >= phases["p2p"] else "p2p"
        if info.get("near_symmetric"):
            # the symmetric kernel evaluates each unordered pair once: 27 flops
            # for the pair plus 2 for the second accumulation, per 2 ordered pairs
            p2p_flops = info["p2p_pairs"] / 2.0 * 29.0
            kern_stats["p2p"]["tflops_executed_sym"] = p2p_flops / (phases["p2p"] * 1e-3) / 1e12 if phases["p2p"] else None
        lattice = bool(info.get("near_lattice"))
        if lattice:
            # translation-invariant leaves (lattice.cu): the near field is sum_o K_o q on the
            # FP64 tensor cores, one multiply-add per near pair
            p2p_flops = info["p2p_pairs"] * 2.0
            kern_stats["p2p"]["tflops_executed_lattice"] = p2p_flops / (phases["p2p"] * 1e-3) / 1e12 if phases["p2p"] else None
            kern_stats["p2p"].pop("tflops_executed_sym", None)
        flops = m2l_flops if dom == "m2l" else p2p_flops
        achieved = flops / (phases[dom] * 1e-3) / 1e12
        near_k = "lattice_near_kernel" if lattice else "p2p_sym_kernel" if info.get("near_symmetric") else "l2p_p2p_kernel"
        kname = "m2l_kernel" if dom == "m2l" else near_k
        bound = "tensor" if dom == "m2l" or lattice else "fp64"
        peak = fp64_peak_tflops(bound)
        roofline = {"bound": bound, "kernel": kname,
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": measured_traffic(args.workload, kname),
                    "peak_source": ("measured FP64 tensor-core (DMMA, tools/dmma_peak.cu)" if bound == "tensor"
                                    else "measured FP64 CUDA-core (DFMA, tools/fp64_peak.cu)")
                                   + " peak, profiles/fp64_peak_r01.json; MEASURED_PEAKS.json has no FP64 entry",
                    "bound_note": ("M2L runs on the FP64 tensor cores (mma.sync m8n8k4 f64)" if dom == "m2l"
                                   else "leaves are translates of one point pattern: the near field is the dense "
                                        "contraction sum_o K_o q (K_o = ln r^2 blocks formed once per plan) on the "
                                        "FP64 tensor cores; phase time includes the finalize" if lattice
                                   else "the near-field log sum is FP64 CUDA-core work (no tensor-core form)"),
                    "flops_per_unit": ("4P(P+1)+8(P+1)+6P executed per M2L pair" if dom == "m2l"
                                       else "2 per near-field pair (one multiply-add of the precomputed ln r^2)" if lattice
                                       else "27 per near-field pair (SURVEY.md 8d convention)"
                                       if near_k != "p2p_sym_kernel" else
                                       "29 per unordered near-field pair (27 per pair, SURVEY.md 8d, + 2 for the "
                                       "second target's accumulation; ordered pairs / 2)")}
    elif wl.kernel == "helmholtz" and info["levels"] > 0 and info["p2p_pairs"] > 0 and phases["p2p"] > 0:
        # native Chebyshev FMM: the dominant phase is the K0 near field (+ L2P),
        # 70 flops per K0 pair by the SURVEY.md 8d convention
        dom = "p2p"
        k0_flops = info["p2p_pairs"] * 70.0
        achieved = k0_flops / (phases["p2p"] * 1e-3) / 1e12
        peak = fp64_peak_tflops("fp64")
        kern_stats["p2p"] = {"ms": phases["p2p"], "pairs": info["p2p_pairs"],
                             "pairs_per_s": info["p2p_pairs"] / (phases["p2p"] * 1e-3)}
        kern_stats["m2l"] = {"ms": phases["m2l"], "pairs": info["m2l_pairs"]}
        roofline = {"bound": "fp64", "kernel": "hf_l2p_p2p_kernel", "achieved": achieved, "peak": peak,
                    "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                    "peak_source": "measured FP64 CUDA-core (DFMA) peak, profiles/fp64_peak_r01.json",
                    "flops_per_unit": "70 per near-field K0 pair (SURVEY.md 8d convention), phase time includes L2P"}
    else:
        dom = "p2p"
        roofline = {"bound": "fp64", "kernel": "traverse_kernel" if wl.kernel == "helmholtz" else "allpairs_kernel",
                    "achieved": None, "peak": peak, "unit": "TFLOP/s", "frac": None, "traffic": None}
    line = {
        "metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": args.workload, "ns": wl.ns, "nt": wl.nt, "epsilon": eps,
                   "levels": info["levels"], "order": P, "mode": args.mode,
                   "parallelism": f"target-shard{world}" if world > 1 else "single",
                   "interactions_per_step": inter, "interactions_counted": counted,
                   "l2": "flushed (256 MB write) before every timed step",
                   "near_field": ("dense K_o q products on the FP64 tensor cores: the leaves are translates of one "
                                  "point pattern, the nine ln r^2 blocks K_o are plan data like the translation "
                                  "operators (lattice.cu; VPG_LATTICE=0 runs the pairwise kernel, "
                                  "profiles/r02/bench_cfg4_pairwise_v8.json)" if info.get("near_lattice")
                                  else "pairwise, unordered pairs (p2p_sym_kernel)" if info.get("near_symmetric")
                                  else "pairwise, one-sided (l2p_p2p_kernel)"),
                   "step": ("operator apply: build_charges + FMM step + correction (potential.cpp:431-470)"
                            if op is not None else "FMM step: SummationPlan::apply (summation.cpp:610-643)")},
        "e2e": {"value": inter / (e2e_ms * 1e-3), "unit": "interactions/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * (wl.ns if op is None else int(f_np.size)), "d2h_bytes_per_step": 8 * wl.nt,
                "path": ("vpg_operator_apply" if op is not None else "vpg_plan_apply")
                        + " with pinned host buffers, " + e2e_mode,
                "candidates_ms": cands,
                "serial_ms_per_step": e2e_serial_ms,
                "l2": ("not flushed in the two-stream loop: the plan's working set is > 4x L2" if big and two_stream
                       else "flushed (256 MB write) before every step"),
                "serial_value": inter / (e2e_serial_ms * 1e-3)},
        "gpu_launches": int((launches_per_step + (2 if op is not None else 0)) * args.steps),
        "phases_ms": phases,
        "kernels": kern_stats,
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if corr_info is not None:
        st = corr_info["stats"]
        line["config"].update({"mesh": wl.notes["h_name"], "cells": wl.notes["cells"], "p": wl.notes["p"],
                               "q": wl.notes["q"], "ndofs": int(f_np.size),
                               "correction_blocks": int(st["blocks"]), "correction_rows": int(st["pool_rows"])})
        line["correction_build"] = {"ms": corr_info["build_ms"], "rows_per_s": st["pool_rows"] / (
            corr_info["build_ms"] * 1e-3), **{k: v for k, v in st.items()}}
        line["acceptance7_correction_over_smooth"] = phases.get("correction", 0.0) / max(ms - phases.get(
            "correction", 0.0), 1e-9)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(wl, inter, corr=corr_info)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------- correction rows
CORR_METRIC = "correction rows/s (build_corrections: classification, task list, rows)"
CORR_MESH = "star_h00125"


def _corr_setup(local, h_name=CORR_MESH):
    from paper_2203_05933_b200 import rows as RW
    from paper_2203_05933_b200 import workloads as W
    m = dict(np.load(os.path.join(W.GOLDEN, f"mesh_{h_name}.npz")))
    b = dict(np.load(os.path.join(W.GOLDEN, "basis_p8_q16.npz")))
    nodes, _ = W.map_cells(m, [b["tri_nodes"], b["box_nodes"]])
    box = m["type"] == 2
    node_off = np.concatenate([[0], np.cumsum(np.where(box, 64, 36))]).astype(np.int32)
    return RW, m, b, nodes, node_off


def _corr_reference_rate(h_name=CORR_MESH, ntarget=1500, seed=3):
    """The reference's build_corrections rate on the host cores: the reference
    operator (oracle/_ref/libvolpot_ref_op.so) built on the same reference mesh
    for a seeded subset of its nodes, minus a one-target build (the shared
    tables and the sources, built once per operator)."""
    import oracle
    R = oracle.reference_operator()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    h = {"star_h0125": 0.125, "star_h005": 0.05, "star_h0025": 0.025, "star_h00125": 0.0125}[h_name]
    rm = R.star_mesh(h, r0=1.0, amp=0.3, arms=5)
    nodes = rm.nodes(8)
    rng = np.random.default_rng(seed)
    sub = nodes[np.sort(rng.choice(len(nodes), ntarget, replace=False))]
    rm.operator(8, 16, nodes[:1])  # warm the cached reference tables
    t0 = time.perf_counter()
    op1 = rm.operator(8, 16, nodes[:1])
    t1 = time.perf_counter()
    opn = rm.operator(8, 16, sub)
    t2 = time.perf_counter()
    rows = opn.npool - op1.npool
    dt = (t2 - t1) - (t1 - t0)
    return {"value": rows / dt, "unit": "rows/s", "cores": cores, "kind": "reference",
            "ms_per_row": dt / rows * 1e3,
            "sample": f"reference VolumePotentialOperator build (oracle/_ref/libvolpot_ref_op.so, "
                      f"set_thread_count({cores})) on the same reference mesh for {ntarget} seeded nodes "
                      f"({rows} correction rows) minus a 1-target build"}


def run_corr(args):
    import torch
    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        cb = _corr_reference_rate()
        line = {"impl": "reference", "metric": CORR_METRIC, "value": cb["value"], "unit": "rows/s", "n_gpus": world,
                "steps": 1, "warmup": 1, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "reference star mesh (tests/golden)",
                "config": {"workload": "corr", "mesh": CORR_MESH, "p": 8, "q": 16},
                "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "rows/s", "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    torch.cuda.set_device(local)
    RW, m, b, nodes, node_off = _corr_setup(local)
    mesh = RW.Mesh(m["type"], m["curve"], m["v"], m["tt"], m["ch"], np.array([RW.CURVE_STAR]), m["star"][None, :])
    eng = RW.RowEngine(mesh, 0, 0.0, 8, 16, b["tri_nodes"], b["tri_C"], b["box_C"], b["tri_src"], b["tri_src_w"],
                       device=local)
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        cm, st = RW.build_correction_map(eng, nodes, node_off, nodes)
        cm.close()
    times, stats = [], None
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cm, stats = RW.build_correction_map(eng, nodes, node_off, nodes)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        cm.close()
    clk.__exit__(None, None, None)
    t = float(np.mean(times))
    rows = stats["pool_rows"]
    if rank != 0:
        return 0
    # roofline of the row kernels: per quadrature node 4 nb (basis recurrences
    # and the row accumulate) + 30 (cell map, kernel log, weight) flops,
    # nb = 36 on triangle rows, 64 on box rows (convention)
    flops = stats["quad_nodes_tri"] * (4 * 36 + 30) + stats["quad_nodes_box"] * (4 * 64 + 30)
    achieved = flops / (stats["rows_ms"] * 1e-3) / 1e12
    peak = fp64_peak_tflops("fp64")
    line = {
        "metric": CORR_METRIC, "value": rows / t, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "the reference's own hybrid mesh of the configs[1] star "
                                                      "(tests/golden/mesh_star_h00125.npz), targets = its nodes",
        "config": {"workload": "corr", "mesh": CORR_MESH, "cells": int(len(m["type"])), "targets": int(len(nodes)),
                   "p": 8, "q": 16, "D": 0.4, "step": "build_corrections (potential.cpp:133-349) on the device"},
        "e2e": {"value": rows / t, "unit": "rows/s", "ms_per_step": t * 1e3,
                "h2d_bytes_per_step": int(nodes.nbytes * 2), "d2h_bytes_per_step": 0,
                "path": "vpg_corr_build with host target arrays; the map stays on the device"},
        "gpu_launches": 4, "stats": stats,
        "roofline": {"bound": "fp64", "kernel": "rows_kernel", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                     "flops_per_unit": "per quadrature node 4 nb + 30 (nb = 36 triangle rows, 64 box rows)"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = _corr_reference_rate()
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- layer potential
LAYER_METRIC = "target-boundary node interactions/s (FP64) for the layer-potential evaluation"
LAYER_FLOPS = {0: 15.0, 1: 80.0}  # per evaluated pair: Laplace dn/r^2 (+min), MH with K1 by convention


def _layer_pairs(sys, tgt):
    """Evaluated pairs of one eval: every target against every coarse node,
    plus 8n fine nodes for the targets the refined check sends to the fine
    rule (bie.cpp:414-440), counted on the host from the coarse distance."""
    coarse = fine = 0
    for c in sys.curves:
        h = c.length / c.n
        d2 = np.full(len(tgt), np.inf)
        for j0 in range(0, c.n, 64):
            blk = c.x[j0:j0 + 64]
            d2 = np.minimum(d2, ((tgt[:, None, :] - blk[None, :, :]) ** 2).sum(axis=2).min(axis=1))
        cand = np.sqrt(d2) - 0.75 * h <= 5.0 * h
        coarse += len(tgt) * c.n
        fine += int(cand.sum()) * c.n * 8
    return coarse, fine


def _layer_kernel(workload):
    import paper_2203_05933_b200 as vp
    if workload == "layer_mh":  # configs[4]'s lambda on the configs[1] boundary
        return vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, 10.0)
    return vp.make_kernel(vp.KernelFamily.Laplace)


def run_layer(args):
    import torch

    import paper_2203_05933_b200 as vp
    from paper_2203_05933_b200 import workloads as W

    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        import oracle
        sys_, cf, tg = W.layer_cfg2(_layer_kernel(args.workload))
        fam, lam = int(sys_.kernel.family), sys_.kernel.lam
        rest = oracle.restatement()
        cores = os.cpu_count() or 1
        sub = tg[:: max(1, len(tg) // 60000)]
        for _ in range(args.warmup):
            rest.layer_eval(fam, lam, sys_.curves, sys_.n_density, sys_.n_aux, cf, sub, True, cores)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            rest.layer_eval(fam, lam, sys_.curves, sys_.n_density, sys_.n_aux, cf, sub, True, cores)
            times.append(time.perf_counter() - t0)
        co, fi = _layer_pairs(sys_, sub)
        t = float(np.mean(times))
        v = (co + fi) / t
        print(json.dumps({
            "impl": "reference", "metric": LAYER_METRIC, "value": v, "unit": "interactions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, configs[1] shapes)",
            "config": {"workload": args.workload, "nt": len(sub), "n_boundary": sys_.n_density},
            "cpu_baseline": {"value": v, "unit": "interactions/s", "cores": cores, "kind": "port",
                             "sample": f"every {max(1, len(tg) // 60000)}-th configs[1] target ({len(sub)}), "
                                       "oracle vo_layer_eval (bie.cpp:383-461 restated; bie.cpp needs Eigen)"},
            "e2e": {"value": v, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
            flush=True)
        return 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(dist_backend(), **({"device_id": torch.device("cuda", local)}
                                                   if dist_backend() == "nccl" else {}))
    sys_, cf, tg_all = W.layer_cfg2(_layer_kernel(args.workload))
    fam, lam = int(sys_.kernel.family), sys_.kernel.lam
    # targets are independent: rank r evaluates a contiguous slice, no collective
    lo, hi = len(tg_all) * rank // world, len(tg_all) * (rank + 1) // world
    tg = np.ascontiguousarray(tg_all[lo:hi])
    ev_obj = sys_.evaluator(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    cf_d = torch.from_numpy(cf).to("cuda")
    tg_d = torch.from_numpy(np.ascontiguousarray(tg)).to("cuda")
    out_d = torch.empty(len(tg), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        ev_obj.eval_device(cf_d.data_ptr(), cf_d.numel(), tg_d.data_ptr(), len(tg), out_d.data_ptr(),
                           allow_close=True, stream=sh)

    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    t_hold = time.time()
    while time.time() - t_hold < 0.5:
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    if dist:
        dist.barrier()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # end to end: host arrays through vpg_layer_eval (H2D of density + targets, D2H of u_H)
    host = ev_obj.eval(cf, tg, allow_close=True)
    e2e = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        host = ev_obj.eval(cf, tg, allow_close=True)
        e2e.append(time.perf_counter() - t0)
    e2e_ms = float(np.mean(e2e)) * 1e3
    if not np.array_equal(host, out_d.cpu().numpy()):
        raise RuntimeError("host and device layer evaluations differ")
    if dist:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        if rank != 0:
            dist.destroy_process_group()
            return 0
    tg = tg_all  # the whole job's pairs (all ranks)
    co, fi = _layer_pairs(sys_, tg)
    pairs = co + fi
    achieved = pairs * LAYER_FLOPS[fam] / (ms * 1e-3) / 1e12
    peak = fp64_peak_tflops("fp64")
    line = {
        "metric": LAYER_METRIC, "value": pairs / (ms * 1e-3), "unit": "interactions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, configs[1] shapes)",
        "config": {"workload": args.workload, "nt": len(tg), "n_boundary": sys_.n_density, "coarse_pairs": co,
                   "fine_pairs": fi, "allow_close": True, "l2": "flushed (256 MB write) before every timed step",
                   "step": "eval_layer_potential (bie.cpp:383-468), "
                           + ("Laplace" if fam == 0 else f"modified Helmholtz lambda={lam}") + ", star boundary"},
        "e2e": {"value": pairs / (e2e_ms * 1e-3), "unit": "interactions/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * cf.size + 16 * len(tg), "d2h_bytes_per_step": 8 * len(tg),
                "path": "vpg_layer_eval with host arrays (wall clock, includes the reject readback)"},
        "gpu_launches": (4 + len(sys_.curves)) * args.steps,
        "roofline": {"bound": "fp64", "kernel": "coarse_kernel+fine_kernel", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                     "flops_per_unit": ("15 per evaluated (target, node) pair (2 sub, 3 r^2, 3 dn, 1 min, "
                                        "4 reciprocal, 2 accumulate)") if fam == 0 else
                                       "80 per evaluated (target, node) pair (K1 counted as 60 by convention)"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        import oracle
        rest = oracle.restatement()
        cores = os.cpu_count() or 1
        sub = tg[:: max(1, len(tg) // 60000)]
        t0 = time.perf_counter()
        rest.layer_eval(fam, lam, sys_.curves, sys_.n_density, sys_.n_aux, cf, sub, True, cores)
        t = time.perf_counter() - t0
        cs, fs = _layer_pairs(sys_, sub)
        line["cpu_baseline"] = {"value": (cs + fs) / t, "unit": "interactions/s", "cores": cores, "kind": "port",
                                "sample": f"{len(sub)} of the configs[1] targets (every "
                                          f"{max(1, len(tg) // 60000)}-th), oracle vo_layer_eval"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD,
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "layer", "layer_mh", "op_star", "op_star_mh",
                             "op_star_84k", "corr"])
    ap.add_argument("--mode", default="reference", choices=["reference", "native"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eps", type=float, default=None,
                    help="FMM tolerance (default: the workload's tightest; cfg4 names 1e-6, 1e-9, 1e-12)")
    args = ap.parse_args()
    if args.workload in ("layer", "layer_mh"):
        return run_layer(args)
    if args.workload == "corr":
        return run_corr(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
