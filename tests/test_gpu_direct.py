"""All-pairs sums on the GPU vs the oracle (summation.cpp:501-540, 619-635)."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2203_05933_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_spec_examples(vp):
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    # SPEC.md:507 single source q=1 at origin, target at (1,0) -> 0
    out = vp.direct_sum(k, vp.SourceSet([[0.0, 0.0]], [1.0]), [[1.0, 0.0]])
    assert out[0] == 0.0
    # SPEC.md:508 symmetric pair, target at origin -> 0
    out = vp.direct_sum(k, vp.SourceSet([[1.0, 0.0], [-1.0, 0.0]], [1.0, 1.0]), [[0.0, 0.0]])
    assert out[0] == 0.0


def test_coincidence_raises_smallest_pair(vp):
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    src = np.array([[0.0, 0.0], [0.5, 0.5], [0.25, 0.0]])
    tgt = np.array([[0.1, 0.1], [0.25, 0.0], [0.5, 0.5]])
    with pytest.raises(vp.CoincidentPoint) as ei:
        vp.direct_sum(k, vp.SourceSet(src, [1.0, 2.0, 3.0]), tgt)
    assert ei.value.target == 1 and ei.value.source == 2
    assert "direct_sum: target 1 coincides with source 2" in str(ei.value)


def test_size_mismatch(vp):
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    with pytest.raises(vp.InvalidArgument):
        vp.direct_sum(k, vp.SourceSet([[0.0, 0.0]], [1.0, 2.0]), [[1.0, 0.0]])


def test_random_100x100_matches_restatement(vp, rest):
    rng = np.random.default_rng(7)
    src, tgt = rng.uniform(0, 1, (100, 2)), rng.uniform(0, 1, (100, 2))
    q = rng.standard_normal(100)
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    gpu = vp.direct_sum(k, vp.SourceSet(src, q), tgt)
    cpu, rc, _ = rest.direct_sum(0, 0.0, src, q, tgt)
    assert rc == 0
    assert rel_l2(gpu, cpu) <= 1e-14


def test_cfg1_direct_p2p_vs_long_double(vp, rest):
    """cfg1: direct P2P with the self term skipped; rel l2 <= 1e-12 (north star)."""
    w = W.cfg1()
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    gpu = vp.direct_sum(k, vp.SourceSet(w.src, w.q), w.tgt, skip_coincident=True)
    ld = rest.pairwise_ld(0, 0.0, w.src, w.q, w.tgt)
    assert rel_l2(gpu, ld) <= 1e-12
    assert np.max(np.abs(gpu - ld)) <= 1e-13 * np.max(np.abs(ld))


def test_helmholtz_direct_vs_restatement(vp, rest):
    rng = np.random.default_rng(11)
    src, tgt = rng.uniform(-1, 1, (3000, 2)), rng.uniform(-1, 1, (2000, 2))
    q = rng.standard_normal(3000)
    k = vp.make_kernel(vp.KernelFamily.ModifiedHelmholtz, 10.0)
    gpu = vp.direct_sum(k, vp.SourceSet(src, q), tgt)
    cpu, rc, _ = rest.direct_sum(1, 10.0, src, q, tgt)
    assert rc == 0
    assert rel_l2(gpu, cpu) <= 1e-13


def test_bessel_k0_vs_reference(vp, rest):
    x = np.concatenate([np.geomspace(1e-8, 2.0, 300), np.linspace(2.0, 40.0, 500),
                        np.geomspace(40.0, 800.0, 200), [2.0, 4.0, 8.0, 1024.0, 1500.0]])
    gpu = vp.bessel_k0(x)
    cpu = rest.bessel_k0(x)
    nz = cpu > 0
    assert np.all(np.abs(gpu[nz] - cpu[nz]) <= 4e-15 * cpu[nz])
    assert np.all(gpu[~nz] == 0.0)
    with pytest.raises(vp.DomainError):
        vp.bessel_k0([1.0, 0.0])


def test_deterministic(vp):
    w = W.cfg1()
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    a = vp.direct_sum(k, vp.SourceSet(w.src, w.q), w.tgt, skip_coincident=True)
    b = vp.direct_sum(k, vp.SourceSet(w.src, w.q), w.tgt, skip_coincident=True)
    assert np.array_equal(a, b)
