"""Modified Helmholtz (lambda = 10): GPU treecode vs the reference treecode
(oracle/_ref, summation.cpp:350-497), the restatement and direct K0 sums."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2203_05933_b200 import workloads as W

pytestmark = pytest.mark.gpu


def mh(vp, lam=10.0):
    return vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, lam)


def test_make_kernel_rejects_nonpositive_lambda(vp):
    with pytest.raises(vp.InvalidArgument, match="needs lambda > 0"):
        vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, 0.0)


def test_treecode_vs_reference_random(vp, ref, rest):
    rng = np.random.default_rng(21)
    pts = rng.uniform(-1.3, 1.3, (12_000, 2))
    q = rng.standard_normal(12_000)
    with vp.SummationPlan(mh(vp), pts, pts, 1e-12) as plan:
        assert plan.levels() > 0
        gpu = plan.apply(q)
        rp = ref.plan(1, 10.0, pts, pts, 1e-12)
        assert plan.levels() == rp.levels()
        assert plan.expansion_order() == rp.expansion_order()
    cpu = rp.apply(q)
    assert rel_l2(gpu, cpu) <= 1e-13
    direct = rest.plan_sum(1, 10.0, pts[:1], q[:1], pts[:1])  # smoke of the oracle path
    assert np.isfinite(direct).all()
    idx = rng.choice(12_000, 600, replace=False)
    ld = rest.pairwise_ld(1, 10.0, pts, q, pts[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


def test_cfg5_subset_vs_direct(vp, rest):
    """cfg5 accuracy oracle: direct K0 P2P on a 65,536-node subset."""
    w = W.cfg5(n_side=96, ntri=1000)
    src, q = w.src, w.q
    with vp.SummationPlan(mh(vp), src, src, 1e-12) as plan:
        gpu = plan.apply(q)
    idx = np.random.default_rng(4).choice(len(src), 2000, replace=False)
    ld = rest.pairwise_ld(1, 10.0, src, q, src[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


@pytest.mark.parametrize("eps", [1e-12, 1e-8])
def test_native_helmholtz_fmm_vs_direct(vp, rest, eps):
    """NATIVE mode for modified Helmholtz: the compressed Chebyshev FMM
    (helm.cu) instead of the reference treecode, against long-double direct
    K0 sums, to the requested epsilon."""
    w = W.cfg5(n_side=96, ntri=1000)
    src, q = w.src, w.q
    with vp.SummationPlan(mh(vp), src, src, eps, mode="native") as plan:
        gpu = plan.apply(q)
        again = plan.apply(q)
    assert np.array_equal(gpu, again)
    idx = np.random.default_rng(4).choice(len(src), 2000, replace=False)
    ld = rest.pairwise_ld(1, 10.0, src, q, src[idx])
    assert rel_l2(gpu[idx], ld) <= eps


def test_native_helmholtz_random_clusters(vp, rest):
    rng = np.random.default_rng(22)
    src = np.concatenate([rng.uniform(-1, 1, (20_000, 2)), 0.1 * rng.standard_normal((20_000, 2))])
    tgt = rng.uniform(-1.2, 1.2, (15_000, 2))
    q = rng.standard_normal(len(src))
    with vp.SummationPlan(mh(vp, 4.0), src, tgt, 1e-12, mode="native") as plan:
        gpu = plan.apply(q)
    idx = np.random.default_rng(5).choice(len(tgt), 1500, replace=False)
    ld = rest.pairwise_ld(1, 4.0, src, q, tgt[idx])
    assert rel_l2(gpu[idx], ld) <= 1e-12


def test_native_helmholtz_symmetric_near_field(vp, rest, monkeypatch):
    """The Chebyshev FMM's near field by unordered node pairs (sym.cuh with
    the K0 pair function, hf_sym_finalize_kernel) against the one-sided
    kernel (VPG_SYM=0) and long-double direct sums; 3,000 extra targets that
    are not nodes take the finalize's one-sided branch."""
    w = W.cfg5(n_side=96, ntri=1000)
    src, q = w.src, w.q
    extra = np.random.default_rng(8).uniform(src.min(0), src.max(0), (3000, 2))
    tgt = np.concatenate([src, extra])
    with vp.SummationPlan(mh(vp), src, tgt, 1e-12, mode="native") as plan:
        assert plan.info()["near_symmetric"] == 1
        sym = plan.apply(q)
        assert np.array_equal(sym, plan.apply(q))
    monkeypatch.setenv("VPG_SYM", "0")
    with vp.SummationPlan(mh(vp), src, tgt, 1e-12, mode="native") as plan:
        assert plan.info()["near_symmetric"] == 0
        one = plan.apply(q)
    assert rel_l2(sym, one) <= 1e-14
    idx = np.concatenate([np.random.default_rng(9).choice(len(src), 1000, replace=False),
                          len(src) + np.arange(500)])
    ld = rest.pairwise_ld(1, 10.0, src, q, tgt[idx])
    assert rel_l2(sym[idx], ld) <= 1e-12
    assert rel_l2(sym[len(src):len(src) + 500], ld[1000:]) <= 1e-12


def test_native_helmholtz_graph_paths_agree(vp):
    """Chebyshev-FMM applies are replayed from CUDA graphs (near field on a
    concurrent branch): device-pointer pairs, host-pointer applies, the
    profiled plain-launch path and applies from several host threads all give
    bit-identical potentials."""
    import threading
    torch = pytest.importorskip("torch")
    w = W.cfg5(n_side=96, ntri=1000)
    src, q = w.src, w.q
    with vp.SummationPlan(mh(vp), src, src, 1e-12, mode="native") as plan:
        plan.set_profiling(True)
        ref = plan.apply(q)
        plan.set_profiling(False)
        assert np.array_equal(plan.apply(q), ref)
        s = torch.cuda.current_stream()
        qd = torch.tensor(q, device="cuda")
        outs = [torch.empty(len(src), dtype=torch.float64, device="cuda") for _ in range(5)]
        for o in outs:
            o.fill_(float("nan"))
            plan.apply_device(qd.data_ptr(), o.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), ref)
        rng = np.random.default_rng(12)
        qs = [rng.standard_normal(len(src)) for _ in range(4)]
        want = [plan.apply(x) for x in qs]
        got = [None] * len(qs)

        def run(i):
            for _ in range(2):
                got[i] = plan.apply(qs[i])

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(qs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
