"""Times the correction apply of the cfg5 synthetic map (device pointers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_05933_b200 as vp  # noqa: E402
from paper_2203_05933_b200 import workloads as W  # noqa: E402

w = W.cfg5()
c = w.notes["corr"]()
cm = vp.CorrectionMap(c["blk_off"], c["blk_cell"], c["blk_pool"], c["pool_off"], c["pool_vals"], c["node_off"])
f = torch.from_numpy(np.ascontiguousarray(w.notes["f"])).cuda()
out = torch.zeros(w.nt, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    cm.apply_device(f.data_ptr(), out.data_ptr(), s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    cm.apply_device(f.data_ptr(), out.data_ptr(), s)
e1.record()
torch.cuda.synchronize()
print("corr ms", e0.elapsed_time(e1) / 10, "blocks", c["blk_cell"].size)
