"""Parity at the >= 1M-node configurations the north star targets.

* cfg4 (BASELINE configs[3], 4,194,304 nodes, reference tree L = 7, 256 points
  per leaf: the lattice near field (lattice.cu), and with VPG_LATTICE=0 the
  symmetric pairwise kernel) at eps = 1e-12, 1e-9, 1e-6:
  the whole potential vector against the unmodified reference
  SummationPlan::apply (oracle/_ref, summation.cpp:610-643) on the host
  cores, and 2,000 seeded targets against the long-double pairwise sum
  (r^2 == 0 skipped, summation.cpp:340).
* cfg3 in reference mode (uniform L = 7 tree over the locally refined nodes:
  leaves up to 4,096 points, the symmetric kernel's subtask path) against the
  reference apply and the long-double sum.
* cfg5 in full (~1.14M nodes, lambda = 10): the GPU treecode (reference mode,
  summation.cpp:416-497) and the Chebyshev FMM (native mode) against each
  other over every target and against long-double-accumulated K0 sums over
  all sources (summation.cpp:501-540 semantics) at 500 targets.
"""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2203_05933_b200 import workloads as W

pytestmark = pytest.mark.gpu


def lap(vp):
    return vp.make_kernel(vp.KernelFamily.Laplace)


@pytest.fixture(scope="module")
def cfg4():
    return W.cfg4()


@pytest.fixture(scope="module")
def cfg4_ld(cfg4, rest):
    idx = np.random.default_rng(404).choice(cfg4.nt, 2000, replace=False)
    return idx, rest.pairwise_ld(0, 0.0, cfg4.src, cfg4.q, cfg4.tgt[idx])


@pytest.mark.parametrize("eps,order", [(1e-12, 50), (1e-9, 39), (1e-6, 27)])
def test_cfg4_vs_reference_apply(vp, ref, cfg4, cfg4_ld, eps, order):
    w = cfg4
    with vp.SummationPlan(lap(vp), w.src, w.tgt, eps) as plan:
        info = plan.info()
        assert info["levels"] == 7 and info["expansion_order"] == order
        assert info["near_symmetric"] == 1 and info["near_lattice"] == 1  # leaves are translates of one pattern
        assert info["p2p_pairs"] == 9_563_275_264  # the instrumented reference's count
        assert info["m2l_pairs"] == 568_872
        gpu = plan.apply(w.q)
        again = plan.apply(w.q)
    assert np.array_equal(gpu, again)
    rp = ref.plan(0, 0.0, w.src, w.tgt, eps)
    assert rp.levels() == 7 and rp.expansion_order() == order
    cpu = rp.apply(w.q)
    rp.close()
    assert rel_l2(gpu, cpu) <= 1e-13
    idx, ld = cfg4_ld
    assert rel_l2(gpu[idx], ld) <= max(eps, 1e-12)
    assert rel_l2(cpu[idx], ld) <= max(eps, 1e-12)


def test_cfg4_near_field_paths_agree(vp, ref, cfg4, cfg4_ld, monkeypatch):
    """The three near-field forms at cfg4: the lattice GEMMs (default), the
    symmetric pairwise kernel (VPG_LATTICE=0, the cost model's choice among the
    pairwise kernels) and the one-sided kernel (VPG_SYM=0) give the same
    potentials to rounding, and the pairwise symmetric one matches the reference
    apply and the long-double sums on its own."""
    w = cfg4
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.info()["near_lattice"] == 1
        lat = plan.apply(w.q)
    monkeypatch.setenv("VPG_LATTICE", "0")
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        info = plan.info()
        assert info["near_symmetric"] == 1 and info["near_lattice"] == 0
        sym = plan.apply(w.q)
    monkeypatch.setenv("VPG_SYM", "0")
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.info()["near_symmetric"] == 0
        one = plan.apply(w.q)
    assert rel_l2(sym, one) <= 1e-14
    assert rel_l2(lat, one) <= 1e-14
    rp = ref.plan(0, 0.0, w.src, w.tgt, 1e-12)
    cpu = rp.apply(w.q)
    rp.close()
    assert rel_l2(sym, cpu) <= 1e-13
    idx, ld = cfg4_ld
    assert rel_l2(sym[idx], ld) <= 1e-12


def test_cfg3_reference_mode(vp, ref, rest):
    """Uniform reference tree over cfg3's refined nodes: leaves of up to 4,096
    points near the peak go through the symmetric kernel's subtasks."""
    w = W.cfg3()
    with vp.SummationPlan(lap(vp), w.src, w.tgt, 1e-12) as plan:
        assert plan.levels() == 7
        t = plan.dump_tree()
        assert int(np.diff(t["src_off"]).max()) >= 2048
        gpu = plan.apply(w.q)
    rp = ref.plan(0, 0.0, w.src, w.tgt, 1e-12)
    cpu = rp.apply(w.q)
    rp.close()
    assert rel_l2(gpu, cpu) <= 1e-13
    idx = np.random.default_rng(303).choice(w.nt, 1000, replace=False)
    ld = rest.pairwise_ld(0, 0.0, w.src, w.q, w.tgt[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


@pytest.fixture(scope="module")
def cfg5_full():
    return W.cfg5()


def test_cfg5_full_treecode_and_fmm(vp, rest, cfg5_full):
    w = cfg5_full
    assert w.ns > 1_000_000
    k = vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, w.lam)
    with vp.SummationPlan(k, w.src, w.tgt, 1e-12) as plan:
        assert plan.levels() == 7
        tree = plan.apply(w.q)
    with vp.SummationPlan(k, w.src, w.tgt, 1e-12, mode="native") as plan:
        fmm = plan.apply(w.q)
        again = plan.apply(w.q)
    assert np.array_equal(fmm, again)
    assert rel_l2(tree, fmm) <= 1e-12
    idx = np.random.default_rng(505).choice(w.nt, 500, replace=False)
    ld = rest.pairwise_ld(1, w.lam, w.src, w.q, w.tgt[idx])
    assert rel_l2(tree[idx], ld) <= 1e-12
    assert rel_l2(fmm[idx], ld) <= 1e-12
