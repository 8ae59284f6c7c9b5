"""Device tree + interaction lists, bit-exact against the restatement of
summation.cpp:81-129 (leaf CSR, level counts) and 271-303 (M2L lists)."""
import numpy as np
import pytest

from paper_2203_05933_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _check(vp, rest, src, tgt, eps=1e-12):
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    with vp.SummationPlan(k, src, tgt, eps) as plan:
        ref = rest.tree(src, tgt, eps)
        pr = ref["params"]
        info = plan.info()
        assert plan.levels() == pr["levels"]
        assert plan.expansion_order() == pr["order"]
        assert info["x0"] == pr["x0"] and info["y0"] == pr["y0"] and info["side"] == pr["side"]
        t = plan.dump_tree()
        for key in ("src_off", "src_ids", "tgt_off", "tgt_ids", "src_cnt", "tgt_cnt"):
            assert np.array_equal(t[key], ref[key]), key
        total = 0
        for lev in range(2, pr["levels"] + 1):
            g = plan.dump_m2l(lev)
            c = rest.m2l_list(pr["levels"], lev, ref["src_cnt"], ref["tgt_cnt"])
            for key in ("tbox", "toff", "src", "oidx"):
                assert np.array_equal(g[key], c[key]), (lev, key)
            total += len(c["src"])
        assert info["m2l_pairs"] == total
        assert info["p2p_pairs"] == rest.p2p_pairs(pr["levels"], ref["src_off"], ref["tgt_off"])
        return info


def test_cfg1_tree(vp, rest):
    w = W.cfg1()
    info = _check(vp, rest, w.src, w.tgt)
    assert info["levels"] == 5 and info["m2l_pairs"] == 31920 and info["p2p_pairs"] == 2262016


def test_cfg2_tree(vp, rest):
    w = W.cfg2()
    info = _check(vp, rest, w.src, w.tgt)
    assert info["levels"] == 7


def test_random_and_degenerate(vp, rest):
    rng = np.random.default_rng(3)
    # non-square bounding box, separate source/target sets
    src = rng.uniform([0, 0], [3, 1], (9000, 2))
    tgt = rng.uniform([0.5, -0.2], [2, 0.8], (7000, 2))
    _check(vp, rest, src, tgt)
    # points exactly on leaf boundaries and duplicated points (stable order)
    g = np.linspace(-1, 1, 65)
    X, Y = np.meshgrid(g, g)
    pts = np.stack([X.ravel(), Y.ravel()], 1)
    pts = np.concatenate([pts, pts[::7]])
    _check(vp, rest, pts, pts[::-1].copy())


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9, 1e-12, 1e-15])
def test_order_from_eps(vp, rest, eps):
    w = W.cfg1()
    _check(vp, rest, w.src[::2], w.tgt[1::2], eps)
