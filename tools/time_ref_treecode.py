"""One timing of the reference modified-Helmholtz treecode (summation.cpp:416-497)
on the full cfg5 workload (1.14M nodes, lambda = 10, eps = 1e-12), oracle/_ref
on all host cores.  Output: one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2203_05933_b200 import workloads as W  # noqa: E402

wl = W.cfg5()
ref = oracle.reference()
cores = os.cpu_count() or 1
ref.set_threads(cores)
t0 = time.perf_counter()
plan = ref.plan(1, wl.lam, wl.src, wl.tgt, min(wl.eps))
t1 = time.perf_counter()
out = plan.apply(wl.q)
t2 = time.perf_counter()
print(json.dumps({"workload": "cfg5", "ns": wl.ns, "nt": wl.nt, "lambda": wl.lam, "eps": min(wl.eps),
                  "levels": plan.levels(), "order": plan.expansion_order(), "cores": cores,
                  "plan_s": t1 - t0, "apply_s": t2 - t1,
                  "what": "reference SummationPlan (treecode) apply, oracle/_ref = unmodified summation.cpp"}))
