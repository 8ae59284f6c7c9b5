"""Where does the host-pointer apply spend its time beyond the device apply?
(a) device-pointer graph apply, (b) vpg_plan_apply with pinned host buffers,
(c) torch H2D + device apply + torch D2H on the same stream.  CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_05933_b200 as vp
from paper_2203_05933_b200 import workloads as W
w = W.cfg2()
plan = vp.SummationPlan(vp.make_kernel(vp.KernelFamily.Laplace), w.src, w.tgt, 1e-12)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sh = st.cuda_stream
print('stream handle', sh)
qd = torch.from_numpy(w.q).cuda(); od = torch.empty(w.nt, dtype=torch.float64, device='cuda')
qh = torch.from_numpy(w.q.copy()).pin_memory(); oh = torch.empty(w.nt, dtype=torch.float64).pin_memory()
def timeit(fn, n=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(st); fn(); b.record(st)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))
print("device", timeit(lambda: plan.apply_device(qd.data_ptr(), od.data_ptr(), sh)))
print("host ptr", timeit(lambda: plan.apply_host_ptr(qh.data_ptr(), oh.data_ptr(), sh, sync=False)))
def manual():
    qd.copy_(qh, non_blocking=True); plan.apply_device(qd.data_ptr(), od.data_ptr(), sh); oh.copy_(od, non_blocking=True)
print("manual", timeit(manual))
print("h2d only", timeit(lambda: qd.copy_(qh, non_blocking=True)))
print("d2h only", timeit(lambda: oh.copy_(od, non_blocking=True)))
for r in range(3):
    print("rep", r, "host", round(timeit(lambda: plan.apply_host_ptr(qh.data_ptr(), oh.data_ptr(), sh, sync=False)), 4),
          "manual", round(timeit(manual), 4))
def manual_sep():
    qd.copy_(qh, non_blocking=True); plan.apply_device(qd.data_ptr(), od.data_ptr(), sh); oh.copy_(od, non_blocking=True)
    torch.cuda.current_stream().synchronize()
import time
t0 = time.perf_counter()
for _ in range(20): plan.apply_host_ptr(qh.data_ptr(), oh.data_ptr(), sh, sync=True)
t1 = time.perf_counter()
for _ in range(20): manual_sep()
t2 = time.perf_counter()
print("wall per call: host", round((t1 - t0) / 20 * 1e3, 4), "manual", round((t2 - t1) / 20 * 1e3, 4))
