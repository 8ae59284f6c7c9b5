"""Pins the CPU oracle (oracle/volpot_oracle.cpp, our restatement) before it
is trusted as the checker: against the golden vectors generated from the
unmodified reference (tests/golden/), against the reference built in place
(oracle/_ref) where available, against known-answer counts taken from an
instrumented copy of the reference, and against the SPEC
examples."""
import glob
import os

import numpy as np
import pytest

from conftest import rel_l2

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


@pytest.mark.parametrize("name", ["laplace_fmm_e12", "laplace_fmm_e6", "laplace_pairwise", "helm_treecode"])
def test_restatement_reproduces_reference_plans(rest, name):
    g = load(name)
    pr = rest.params(int(g["family"]), float(g["lam"]), g["src"], g["tgt"], float(g["eps"]))
    if int(g["levels"]) == 0:
        assert pr["direct"] == 1  # pairwise fallback (summation.cpp:578)
    else:
        assert pr["levels"] == int(g["levels"]) and pr["order"] == int(g["order"])
    out = rest.plan_sum(int(g["family"]), float(g["lam"]), g["src"], g["q"], g["tgt"], float(g["eps"]))
    # same expressions in the same order: expected bit-identical; allow the
    # last bits to move if a different compiler contracts differently
    assert rel_l2(out, g["out"]) <= 1e-15
    assert np.max(np.abs(out - g["out"])) <= 1e-14 * np.max(np.abs(g["out"]))


@pytest.mark.parametrize("name,family", [("direct_laplace", 0), ("direct_helm", 1)])
def test_restatement_direct_sum(rest, name, family):
    g = load(name)
    out, rc, _ = rest.direct_sum(family, float(g["lam"]), g["src"], g["q"], g["tgt"])
    assert rc == 0
    assert rel_l2(out, g["out"]) <= 1e-15


def test_restatement_bessel_k0(rest):
    g = load("bessel_k0")
    out = rest.bessel_k0(g["x"])
    nz = g["out"] > 0
    assert np.all(np.abs(out[nz] - g["out"][nz]) <= 1e-15 * g["out"][nz])
    assert np.all(out[~nz] == 0.0)


def test_bessel_k0_vs_mpmath(rest):
    mp = pytest.importorskip("mpmath")
    xs = [1e-8, 1e-3, 0.5, 1.0, 1.999, 2.0, 2.001, 3.7, 10.0, 31.4, 100.0, 700.0]
    for x in xs:
        exact = float(mp.besselk(0, x))
        assert abs(rest.bessel_k0([x])[0] - exact) <= 2e-15 * exact, x


def test_spec_direct_sum_examples(rest):
    # SPEC.md:507-508
    out, rc, _ = rest.direct_sum(0, 0.0, [[0.0, 0.0]], [1.0], [[1.0, 0.0]])
    assert rc == 0 and out[0] == 0.0
    out, rc, _ = rest.direct_sum(0, 0.0, [[1.0, 0.0], [-1.0, 0.0]], [1.0, 1.0], [[0.0, 0.0]])
    assert rc == 0 and out[0] == 0.0
    # coincidence: smallest (i, j) (summation.cpp:511-538)
    src = np.array([[0.0, 0.0], [0.5, 0.5], [0.25, 0.0]])
    tgt = np.array([[0.1, 0.1], [0.25, 0.0], [0.5, 0.5]])
    _, rc, (i, j) = rest.direct_sum(0, 0.0, src, [1.0, 2.0, 3.0], tgt)
    assert rc == 2 and (i, j) == (1, 2)


def _grid(nside, lo=-1.0, hi=1.0):
    from paper_2203_05933_b200 import workloads as W
    cx, cy, h = W.uniform_grid(nside, lo, hi)
    return W.box_nodes(cx, cy, h)[0]


def test_known_answer_counts_cfg1(rest):
    """Instrumented-reference counts."""
    from paper_2203_05933_b200 import workloads as W
    w = W.cfg1()
    t = rest.tree(w.src, w.tgt)
    L = t["params"]["levels"]
    assert L == 5 and t["params"]["order"] == 50
    m2l = sum(len(rest.m2l_list(L, l, t["src_cnt"], t["tgt_cnt"])["src"]) for l in range(2, L + 1))
    assert m2l == 31_920
    assert rest.p2p_pairs(L, t["src_off"], t["tgt_off"]) == 2_262_016
    assert abs(w.q.sum() - np.pi / 50) <= 1e-15  # analytic total charge


@pytest.mark.parametrize("nside,p2p", [(64, 37_356_544), (128, 597_704_704)])
def test_known_answer_counts_grids(rest, nside, p2p):
    pts = _grid(nside)
    t = rest.tree(pts, pts)
    L = t["params"]["levels"]
    assert L == 7
    assert rest.p2p_pairs(L, t["src_off"], t["tgt_off"]) == p2p
    m2l = sum(len(rest.m2l_list(L, l, t["src_cnt"], t["tgt_cnt"])["src"]) for l in range(2, L + 1))
    assert m2l == 568_872


def test_restatement_vs_reference_inplace(rest):
    """Where the reference .so exists, the restatement matches it bit for bit
    on cfg1 (FMM, L=5, P=50)."""
    import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    from paper_2203_05933_b200 import workloads as W
    ref = oracle.reference()
    w = W.cfg1()
    a = ref.plan(0, 0.0, w.src, w.tgt, 1e-12).apply(w.q)
    b = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, 1e-12)
    assert np.array_equal(a, b)


def test_golden_files_present():
    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz")))
    assert {"laplace_fmm_e12", "laplace_fmm_e6", "laplace_pairwise", "helm_treecode",
            "direct_laplace", "direct_helm", "bessel_k0"} <= set(names)
