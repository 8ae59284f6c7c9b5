"""Operator-level parity against the REFERENCE's own operator code.

oracle/_ref/libvolpot_ref_op.so is the unmodified reference operator
(proj/src/potential.cpp, singular.cpp, basis.cpp, quad1d.cpp, mesh.cpp,
geometry.cpp, delaunay.cpp + the summation trio) compiled against our
restatement of the Eigen subset it uses (oracle/eigen_restated/).  It builds
a hybrid star-domain mesh (mesh.cpp:262-408), the VolumePotentialOperator
with its correction map (potential.cpp:133-349) and applies it
(potential.cpp:431-470).  These tests feed that operator's data to the GPU
path and compare:

* build_charges (potential.cpp:397-412) -> vp.ChargeMap,
* the correction apply (potential.cpp:446-462) -> vp.CorrectionMap,
* the whole apply (build_charges + SummationPlan::apply + correction) ->
  vp.VolumePotentialOperator.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

P, Q = 8, 16


@pytest.fixture(scope="module")
def R():
    import oracle
    try:
        r = oracle.reference_operator()
    except (FileNotFoundError, OSError) as e:  # pragma: no cover
        pytest.skip(f"reference operator unavailable: {e}")
    import os
    r.set_threads(os.cpu_count() or 1)
    return r


@pytest.fixture(scope="module")
def mesh(R):
    return R.star_mesh(0.2, amp=0.1, arms=3)


@pytest.fixture(scope="module", params=["laplace", "helmholtz"])
def refop(request, R, mesh):
    fam, lam = (0, 0.0) if request.param == "laplace" else (1, 10.0)
    nodes = mesh.nodes(P)
    rng = np.random.default_rng(11)
    extra = nodes[rng.choice(len(nodes), 64, replace=False)] * 0.97  # off-node targets too
    tgt = np.concatenate([nodes, extra])
    op = mesh.operator(P, Q, tgt, fam, lam)
    d = op.export()
    d["targets"] = tgt
    d["family"], d["lam"] = fam, lam
    return op, d


def _f(nodes, seed=3):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-0.4, 0.4, (3, 2))
    a = rng.uniform(5, 20, 3)
    return sum(np.exp(-a[k] * ((nodes - c[k]) ** 2).sum(1)) for k in range(3))


def _charge_map(vp, R, mesh, d):
    ct = np.where(mesh.type == 2, 0, 1).astype(np.int32)
    return vp.ChargeMap(ct, d["node_off"], d["src_off"], R.basis(9, P, Q), R.basis(8, P, Q), d["src_wj"])


def test_build_charges_vs_reference(vp, R, mesh, refop):
    op, d = refop
    f = _f(d["nodes"])
    ref = op.build_charges(f)
    gpu = _charge_map(vp, R, mesh, d).apply(f)
    assert rel_l2(gpu, ref) <= 1e-15


def test_correction_apply_vs_reference(vp, ref, refop):
    """corr = reference apply - reference SummationPlan::apply(charges): the
    same plan code on the same inputs is bitwise reproducible
    (summation.hpp:32-33), so the difference is the reference's correction
    loop up to one rounding of the sum."""
    op, d = refop
    f = _f(d["nodes"])
    out_ref = op.apply(f)
    q = op.build_charges(f)
    plan = ref.plan(d["family"], d["lam"], d["src_xy"], d["targets"], 1e-12)
    smooth = plan.apply(q)
    corr_ref = out_ref - smooth
    cm = vp.CorrectionMap(d["blk_off"], d["blk_cell"], d["blk_pool"], d["pool_off"], d["pool_vals"],
                          d["node_off"])
    corr = cm.apply(f, np.zeros(len(d["targets"])))
    scale = np.abs(out_ref).max()
    # corr_ref carries one rounding of out_ref (|out| >> |corr|)
    assert np.abs(corr - corr_ref).max() <= 4e-15 * scale * 8
    assert rel_l2(corr, corr_ref) <= 1e-12


def test_operator_apply_vs_reference(vp, R, mesh, refop):
    op, d = refop
    f = _f(d["nodes"], seed=4)
    out_ref, tm = op.apply(f, timings=True)
    k = vp.make_kernel(vp.KernelFamily.Laplace) if d["family"] == 0 else \
        vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, d["lam"])
    plan = vp.SummationPlan(k, d["src_xy"], d["targets"], 1e-12)
    cm = vp.CorrectionMap(d["blk_off"], d["blk_cell"], d["blk_pool"], d["pool_off"], d["pool_vals"],
                          d["node_off"])
    ch = _charge_map(vp, R, mesh, d)
    gop = vp.VolumePotentialOperator(plan, cm, ch)
    out, gtm = gop.apply(f, timings=True)
    assert rel_l2(out, out_ref) <= 1e-13
    assert gtm["smooth_ms"] > 0 and gtm["correction_ms"] > 0


@pytest.mark.parametrize("family,lam,holes", [(0, 0.0, ()), (0, 0.0, ((0.3, 0.1, 0.2),)), (1, 10.0, ())])
def test_layer_potential_vs_reference(vp, R, family, lam, holes):
    """eval_layer_potential (bie.cpp:383-468) of the reference on its own
    BoundarySystem (assemble_nystrom) and its own solved density, against the
    device evaluator fed the same curve blocks; targets from the far field
    into the 5-spacing close-evaluation zone."""
    from paper_2203_05933_b200 import bie
    n = 256
    lay = R.layer(family, lam, [n] * (1 + len(holes)), holes=holes)
    nodes = np.concatenate([c["x"] for c in lay.curves])
    rhs = np.concatenate([np.cos(2 * nodes[:, 0]) * np.exp(0.5 * nodes[:, 1]), np.zeros(lay.n_aux)])
    dens = lay.solve(rhs)
    rng = np.random.default_rng(8)
    th = rng.uniform(0, 2 * np.pi, 3000)
    rad = (1 + 0.3 * np.cos(5 * th)) * rng.uniform(0.05, 0.985, th.size) ** 0.5
    tg = np.stack([rad * np.cos(th), rad * np.sin(th)], 1)
    for hc in holes:
        tg = tg[np.hypot(tg[:, 0] - hc[0], tg[:, 1] - hc[1]) > hc[2] * 1.05]
    ref_out = lay.eval(dens, tg, allow_close=True)
    k = vp.make_kernel(vp.KernelFamily.Laplace) if family == 0 else \
        vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, lam)
    blocks = [bie.CurveBlock(**c) for c in lay.curves]
    sysd = bie.BoundarySystem(k, blocks, lay.n_density, lay.n_aux)
    gpu = bie.eval_layer_potential(sysd, dens, tg, allow_close=True)
    tol = 1e-13 if family == 0 else 1e-12
    assert rel_l2(gpu, ref_out) <= tol
