"""Pins of the CPU restatement (oracle/volpot_oracle.cpp) and of the Eigen
restatement (oracle/eigen_restated/) against the REFERENCE operator compiled
in place (oracle/_ref/libvolpot_ref_op.so).  CPU only."""
import os

import numpy as np
import pytest
from scipy.special import exp1

from conftest import rel_l2

P, Q = 8, 16


@pytest.fixture(scope="module")
def R():
    import oracle
    if not os.path.exists(oracle.REFOP_SO) and not os.path.isdir(oracle.REF_SRC):
        pytest.skip("reference operator not built here")
    r = oracle.reference_operator()
    r.set_threads(os.cpu_count() or 1)
    return r


@pytest.fixture(scope="module")
def small(R):
    mesh = R.star_mesh(0.2, amp=0.1, arms=3)
    nodes = mesh.nodes(P)
    op = mesh.operator(P, Q, nodes)
    return mesh, op, op.export()


def test_eigen_restatement_basis_tables(R):
    """The Eigen-dependent tables come out as the math says: C = V^-1 for the
    box and triangle bases (basis.cpp:66,178), the Gauss-Jacobi collapsed rule
    integrates the simplex exactly (basis.cpp:83-127, SelfAdjointEigenSolver),
    the t / -t log t Gauss rules reproduce their moments (quad1d.cpp:153-215)."""
    from paper_2203_05933_b200 import workloads as W
    bnodes, bC = R.basis(2, P), R.basis(3, P)
    V = W.chebyshev2d(P, bnodes[:, 0], bnodes[:, 1])
    assert np.abs(V @ bC - np.eye(P * P)).max() < 1e-13
    tn, tw = R.basis(4, P, Q), R.basis(5, P, Q)
    assert tn.shape == (81, 2)
    # monomials x^a y^b over the unit simplex: a! b! / (a+b+2)!
    from math import factorial
    for a, b in [(0, 0), (3, 2), (7, 5), (0, 16)]:
        ex = factorial(a) * factorial(b) / factorial(a + b + 2)
        assert abs((tw * tn[:, 0] ** a * tn[:, 1] ** b).sum() - ex) <= 2e-14 * ex
    x, w = R.rule1d(1, 20)          # weight t on [0,1]
    for k in range(0, 39):
        assert abs((w * x ** k).sum() - 1.0 / (k + 2)) < 1e-14
    x, w = R.rule1d(2, 20)          # weight -t log t: int t^(k+1)(-log t) = 1/(k+2)^2
    for k in range(0, 39):
        assert abs((w * x ** k).sum() - 1.0 / (k + 2) ** 2) < 1e-14


def test_reference_operator_closed_form(R):
    """End-to-end check of the compiled reference (with the restated Eigen):
    a Gaussian concentrated well inside the star has the full-plane potential
    V(rho) = -[ln rho^2 + E1(a rho^2)] / (4a)."""
    mesh = R.star_mesh(0.2, amp=0.1, arms=3)
    nodes = mesh.nodes(P)
    op = mesh.operator(P, Q, nodes)
    a = 20.0
    f = np.exp(-a * (nodes ** 2).sum(1))
    out = op.apply(f)
    r2 = (nodes ** 2).sum(1)
    ex = -(np.log(r2) + exp1(a * r2)) / (4 * a)
    assert np.abs(out - ex).max() <= 1e-7 * np.abs(ex).max()


def test_restated_build_charges_vs_reference(R, rest, small):
    mesh, op, d = small
    rng = np.random.default_rng(1)
    f = rng.standard_normal(op.ndofs)
    ct = np.where(mesh.type == 2, 0, 1).astype(np.int32)
    q = rest.build_charges(ct, d["node_off"], d["src_off"], R.basis(9, P, Q), R.basis(8, P, Q), d["src_wj"], f)
    assert rel_l2(q, op.build_charges(f)) <= 1e-15


def test_restated_correction_apply_vs_reference(R, rest, ref, small):
    mesh, op, d = small
    rng = np.random.default_rng(2)
    f = rng.standard_normal(op.ndofs)
    out = op.apply(f)
    smooth = ref.plan(0, 0.0, d["src_xy"], d["nodes"], 1e-12).apply(op.build_charges(f))
    corr = rest.correction_apply(d["blk_off"], d["blk_cell"], d["blk_pool"], d["pool_off"], d["pool_vals"],
                                 d["node_off"], f, np.zeros(op.nt))
    assert np.abs(corr - (out - smooth)).max() <= 1e-14 * np.abs(out).max()
    # the map's shape follows the reference near rule: 1 self block + <= 30 near
    nblk = np.diff(d["blk_off"])
    assert nblk.min() >= 1 and nblk.max() <= 31


@pytest.mark.parametrize("family,lam,holes", [(0, 0.0, ()), (0, 0.0, ((0.3, 0.1, 0.2),)), (1, 10.0, ())])
def test_restated_layer_eval_vs_reference(R, rest, family, lam, holes):
    """Our restatement of eval_layer_impl (vo_layer_eval) against the compiled
    reference bie.cpp on the reference's own BoundarySystem and density."""
    from types import SimpleNamespace
    lay = R.layer(family, lam, [128] * (1 + len(holes)), holes=holes)
    nodes = np.concatenate([c["x"] for c in lay.curves])
    dens = lay.solve(np.concatenate([np.sin(nodes[:, 0] + 2 * nodes[:, 1]), np.zeros(lay.n_aux)]))
    rng = np.random.default_rng(9)
    th = rng.uniform(0, 2 * np.pi, 800)
    rad = (1 + 0.3 * np.cos(5 * th)) * rng.uniform(0.05, 0.985, th.size) ** 0.5
    tg = np.stack([rad * np.cos(th), rad * np.sin(th)], 1)
    for hc in holes:
        tg = tg[np.hypot(tg[:, 0] - hc[0], tg[:, 1] - hc[1]) > hc[2] * 1.05]
    ref_out = lay.eval(dens, tg, allow_close=True)
    curves = [SimpleNamespace(**c) for c in lay.curves]
    out, rc = rest.layer_eval(family, lam, curves, lay.n_density, lay.n_aux, dens, tg, True)
    assert rc == 0
    assert rel_l2(out, ref_out) <= (1e-13 if family == 0 else 1e-12)
