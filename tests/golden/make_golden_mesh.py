"""Generates the reference meshes and basis tables in tests/golden/ from the
UNMODIFIED reference operator code (oracle/_ref/libvolpot_ref_op.so:
build_mesh + StarCurve, mesh.cpp:262-408 / geometry.cpp:100-140; the basis
tables of basis.cpp:48-324) so the correction-row workloads run on the GPU box
without the reference sources.  Cells are stored exactly as the reference
builds them (type, vertices, curve parameters (ta, tb), centre, h); the star
is the configs[1] boundary r = 1 + 0.3 cos 5 theta.

    python tests/golden/make_golden_mesh.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

STAR = dict(r0=1.0, amp=0.3, arms=5, phase=0.0, center=(0.0, 0.0))
MESHES = {"star_h0125": 0.125, "star_h005": 0.05, "star_h0025": 0.025, "star_h00125": 0.0125}
P, Q = 8, 16


def main():
    R = oracle.reference_operator()
    for name, h in MESHES.items():
        m = R.star_mesh(h, **STAR)
        np.savez_compressed(os.path.join(HERE, f"mesh_{name}.npz"), type=m.type, curve=m.curve, v=m.v, tt=m.tt,
                            ch=m.ch, h=m.h, n_tri=m.n_tri, n_box=m.n_box,
                            star=np.array([STAR["center"][0], STAR["center"][1], STAR["r0"], STAR["amp"],
                                           STAR["arms"], STAR["phase"]]))
        print(name, m.ncell, m.n_tri, m.n_box)
    np.savez_compressed(os.path.join(HERE, f"basis_p{P}_q{Q}.npz"), tri_nodes=R.basis(0, P), tri_C=R.basis(1, P),
                        box_nodes=R.basis(2, P), box_C=R.basis(3, P), tri_src=R.basis(4, P, Q),
                        tri_src_w=R.basis(5, P, Q), box_src=R.basis(6, P, Q), box_src_w=R.basis(7, P, Q),
                        tri_over=R.basis(8, P, Q), box_over=R.basis(9, P, Q))


if __name__ == "__main__":
    main()
