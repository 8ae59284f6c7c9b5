"""GPU path against the golden vectors generated from the unmodified
reference (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def kern(vp, g):
    if int(g["family"]) == 0:
        return vp.make_kernel(vp.KernelFamily.Laplace)
    return vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, float(g["lam"]))


@pytest.mark.parametrize("name,tol", [("laplace_fmm_e12", 1e-13), ("laplace_fmm_e6", 1e-13),
                                      ("laplace_pairwise", 1e-14), ("helm_treecode", 1e-13)])
def test_plan_vs_golden(vp, name, tol):
    g = load(name)
    with vp.SummationPlan(kern(vp, g), g["src"], g["tgt"], float(g["eps"])) as plan:
        assert plan.levels() == int(g["levels"]) and plan.expansion_order() == int(g["order"])
        out = plan.apply(g["q"])
    assert rel_l2(out, g["out"]) <= tol


@pytest.mark.parametrize("name", ["direct_laplace", "direct_helm"])
def test_direct_vs_golden(vp, name):
    g = load(name)
    out = vp.direct_sum(kern(vp, g), vp.SourceSet(g["src"], g["q"]), g["tgt"])
    assert rel_l2(out, g["out"]) <= 1e-14


def test_bessel_vs_golden(vp):
    g = load("bessel_k0")
    out = vp.bessel_k0(g["x"])
    nz = g["out"] > 0
    assert np.all(np.abs(out[nz] - g["out"][nz]) <= 4e-15 * g["out"][nz])
    assert np.all(out[~nz] == 0.0)
