"""Measured accuracy per configuration (state the measured error,
not just the requested epsilon).  For each workload the GPU apply is compared
on a seeded sample of targets with the long-double pairwise sum of the CPU
oracle (r^2 == 0 skipped, summation.cpp:630), and -- where it runs in seconds --
with the unmodified reference FMM (oracle/_ref).  Writes one JSON object per
line to stdout.  Test/measurement tool: it loads oracle/ as the checker."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2203_05933_b200 as vp  # noqa: E402
from paper_2203_05933_b200 import workloads as W  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    rest = oracle.restatement()
    ref = oracle.reference()
    ref.set_threads(os.cpu_count() or 1)
    rng = np.random.default_rng(2024)
    cases = [("cfg1", "reference", None), ("cfg2", "reference", None), ("cfg3", "native", None),
             ("cfg4", "reference", 1e-6), ("cfg4", "reference", 1e-9), ("cfg4", "reference", 1e-12),
             ("cfg4", "native", 1e-12), ("cfg5", "native", None)]
    for name, mode, eps in cases:
        w = W.CONFIGS[name]()
        e = eps if eps else min(w.eps)
        fam = 1 if w.kernel == "helmholtz" else 0
        k = vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, w.lam) if fam else vp.make_kernel(vp.KernelFamily.Laplace)
        t0 = time.time()
        with vp.SummationPlan(k, w.src, w.tgt, e, mode=mode) as plan:
            gpu = plan.apply(w.q)
            info = plan.info()
        src, q, tgt = w.src, w.q, w.tgt
        if name == "cfg5":  # the BASELINE oracle: direct K0 sums on a 65,536-node subset
            sub = np.sort(rng.choice(w.ns, 65536, replace=False))
            src, q = w.src[sub], w.q[sub]
            tgt = w.tgt[np.sort(rng.choice(w.nt, 2000, replace=False))]
            with vp.SummationPlan(k, src, tgt, e, mode=mode) as plan:
                gpu_s = plan.apply(q)
        else:
            idx = np.sort(rng.choice(w.nt, min(w.nt, 3000), replace=False))
            tgt = w.tgt[idx]
            gpu_s = gpu[idx]
        ld = rest.pairwise_ld(fam, w.lam, src, q, tgt)
        line = {"workload": name, "mode": mode, "epsilon": e, "levels": info["levels"], "order": info["expansion_order"],
                "sample_targets": int(len(tgt)), "sample_sources": int(len(src)),
                "rel_l2_vs_long_double_direct": rel(gpu_s, ld)}
        if name in ("cfg1", "cfg2"):
            rp = ref.plan(fam, w.lam, w.src, w.tgt, e)
            line["rel_l2_vs_reference_fmm"] = rel(gpu, rp.apply(w.q))
        line["seconds"] = round(time.time() - t0, 1)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
