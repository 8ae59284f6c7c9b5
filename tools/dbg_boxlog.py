"""Debug: device box_log rows (job 8) vs the reference box_log table."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_rows import engine
import paper_2203_05933_b200 as vp
R = oracle.reference_operator()
R.set_threads(os.cpu_count())
rm = R.star_mesh(0.2, amp=0.1, arms=3)
P = 8
L = R.box_log(P)
for fam, lam in [(0, 0.0), (1, 10.0)]:
    eng = engine(vp, R, rm, fam, lam)
    aux = [o * 256 + j for o in range(25) for j in range(64)]
    if fam == 0:
        rows = eng.eval([8] * len(aux), [-1] * len(aux), aux=aux)
        ref = [L[a // 256, a % 256] for a in aux]
    else:
        rows = eng.eval([9] * len(aux), [-1] * len(aux), aux=aux, lattice_h=rm.h)
        T = R.box_table(P, fam, lam, rm.h)
        ref = [T[a // 256, a % 256] for a in aux]
    for o in range(25):
        errs = [np.abs(rows[o * 64 + j] - ref[o * 64 + j]).max() / np.abs(ref[o * 64 + j]).max() for j in range(64)]
        print(fam, "offset", o, (o % 5 - 2, o // 5 - 2), "max rel", max(errs), "worst j", int(np.argmax(errs)))
