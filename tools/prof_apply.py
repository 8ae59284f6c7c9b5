"""Minimal driver for ncu: builds one plan and applies it --reps times
(device-resident charges/potentials).  Not a benchmark: numbers printed under
a profiler are never reported."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2203_05933_b200 as vp  # noqa: E402
from paper_2203_05933_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--eps", type=float, default=1e-12)
ap.add_argument("--mode", default="reference")
a = ap.parse_args()
w = W.CONFIGS[a.workload]()
k = vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, w.lam) if w.kernel == "helmholtz" else \
    vp.make_kernel(vp.KernelFamily.Laplace)
plan = vp.SummationPlan(k, w.src, w.tgt, a.eps, mode=a.mode)
q = torch.from_numpy(w.q).cuda()
out = torch.empty(w.nt, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    plan.apply_device(q.data_ptr(), out.data_ptr(), s)
torch.cuda.synchronize()
print("ok", plan.info()["levels"], plan.last_launches())
