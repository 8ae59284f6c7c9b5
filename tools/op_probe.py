"""Operator probe: build the reference-mesh operator on the device and time its
parts (ApplyTimings split, correction apply alone, build_charges alone)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_05933_b200 import rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mesh", default="star_h005")
ap.add_argument("--family", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
here = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
mesh, h = rows.load_mesh(os.path.join(here, f"mesh_{a.mesh}.npz"))
basis = rows.load_basis(os.path.join(here, "basis_p8_q16.npz"))
t0 = time.perf_counter()
g = rows.build_operator(mesh, basis, a.family, 10.0 if a.family else 0.0, 8, 16)
print("build s", round(time.perf_counter() - t0, 3), {k: (round(v, 2) if isinstance(v, float) else v)
                                                      for k, v in g["stats"].items()})
nodes = g["nodes"]
f = np.sin(3 * nodes[:, 0]) * np.cos(2 * nodes[:, 1])
for _ in range(3):
    g["op"].apply(f)
sm, co = [], []
for _ in range(a.reps):
    _, tm = g["op"].apply(f, timings=True)
    sm.append(tm["smooth_ms"])
    co.append(tm["correction_ms"])
print("ndofs", len(nodes), "nsrc", len(g["src_xy"]), "smooth ms min/med", min(sm), np.median(sm),
      "corr ms min/med", min(co), np.median(co), "ratio(min)", min(co) / min(sm))
s = torch.cuda.Stream()
fd = torch.from_numpy(f).cuda()
od = torch.zeros(len(g["targets"]), dtype=torch.float64, device="cuda")
qd = torch.zeros(len(g["src_xy"]), dtype=torch.float64, device="cuda")
for name, fn in [("corr", lambda: g["corr"].apply_device(fd.data_ptr(), od.data_ptr(), s.cuda_stream)),
                 ("charges", lambda: g["charges"].apply_device(fd.data_ptr(), qd.data_ptr(), s.cuda_stream)),
                 ("plan", lambda: g["plan"].apply_device(qd.data_ptr(), od.data_ptr(), s.cuda_stream))]:
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
    torch.cuda.synchronize()
    print(name, "ms per call (back to back)", e0.elapsed_time(e1) / a.reps)
