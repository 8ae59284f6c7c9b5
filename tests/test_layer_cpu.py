"""CPU checks of the layer-potential restatement (bie.cpp:383-468): K1 pinned
to the compiled reference kernel.cpp, trig_upsample exactness, Gauss's lemma
and the reject codes; the boundary geometry builder."""
import numpy as np
import pytest

from paper_2203_05933_b200 import bie
from paper_2203_05933_b200 import workloads as W


def test_k1_restatement_bit_identical_to_reference(rest, ref):
    x = np.concatenate([np.geomspace(1e-4, 2.0, 700), np.linspace(2.0, 760.0, 3000)])
    assert np.array_equal(rest.bessel_k1(x), ref.bessel_k1(x))


def test_k1_against_scipy(rest):
    sp = pytest.importorskip("scipy.special")
    x = np.concatenate([np.geomspace(1e-4, 2.0, 300), np.linspace(2.0, 700.0, 1000)])
    v = rest.bessel_k1(x)
    assert np.max(np.abs(v - sp.k1(x)) / sp.k1(x)) <= 1e-14


def test_trig_upsample_is_exact_interpolation(rest):
    rng = np.random.default_rng(0)
    n = 64
    f = rng.standard_normal(n)
    u = rest.trig_upsample(f, 8)
    assert np.max(np.abs(u[::8] - f)) <= 1e-13
    # a band-limited density (|m| < n/2) is reproduced on the fine grid
    t = 2 * np.pi * np.arange(n) / n
    tf = 2 * np.pi * np.arange(8 * n) / (8 * n)
    g = lambda s: 0.3 + np.cos(3 * s) - 0.5 * np.sin(17 * s) + 0.1 * np.cos(31 * s)  # noqa: E731
    assert np.max(np.abs(rest.trig_upsample(g(t), 8) - g(tf))) <= 1e-13


def test_geometry_builder():
    k = bie.Kernel()
    sys = bie.assemble_geometry([bie.circle_curve(0.0, 0.0, 0.5, hole=False)], [64], k)
    c = sys.curves[0]
    assert abs(c.length - np.pi) <= 1e-14
    assert abs(c.diam - 1.0) <= 1e-12
    assert np.allclose(np.hypot(*c.normal.T), 1.0)
    assert np.allclose(c.normal, c.x / 0.5)  # outward
    hole = bie.circle_curve(0.2, 0.1, 0.3, hole=True).outward_normal(np.array([0.0, 1.0]))
    p = bie.circle_curve(0.2, 0.1, 0.3, hole=True).pos(np.array([0.0, 1.0]))
    assert np.allclose(hole, (p - [0.2, 0.1]) / 0.3)  # out of the enclosed disc
    with pytest.raises(ValueError, match="even and >= 16"):
        bie.assemble_geometry([bie.star_curve()], [15], k)


def test_restatement_gauss_lemma_and_rejects(rest):
    sys = W.layer_system()
    rng = np.random.default_rng(2)
    th = rng.uniform(0, 2 * np.pi, 500)
    rad = bie.star_curve().pos(th)[:, 0] / np.cos(th)
    tg = np.stack([np.cos(th), np.sin(th)], 1) * (rad * rng.uniform(0, 0.98, 500))[:, None]
    out, rc = rest.layer_eval(0, 0.0, sys.curves, sys.n_density, sys.n_aux, np.ones(sys.size()), tg, True)
    assert rc == 0 and np.max(np.abs(out + 1.0)) <= 1e-10
    # outside the curve the double layer of phi = 1 vanishes
    far = np.array([[3.0, 0.5], [-2.0, -2.5]])
    out, rc = rest.layer_eval(0, 0.0, sys.curves, sys.n_density, sys.n_aux, np.ones(sys.size()), far, True)
    assert rc == 0 and np.max(np.abs(out)) <= 1e-13
    c = sys.curves[0]
    cf = np.ones(sys.size())
    assert rest.layer_eval(0, 0.0, sys.curves, sys.n_density, 0, cf[:-1], tg, True)[1] == 1
    assert rest.layer_eval(0, 0.0, sys.curves, sys.n_density, 0, cf, c.fine_x[5:6], True)[1] == 2
    close = (c.x[3] - 0.005 * c.diam * c.normal[3])[None, :]
    assert rest.layer_eval(0, 0.0, sys.curves, sys.n_density, 0, cf, close, False)[1] == 3
    assert rest.layer_eval(0, 0.0, sys.curves, sys.n_density, 0, cf, close, True)[1] == 0


def test_layer_workload_shapes():
    sys, cf, tg = W.layer_cfg2()
    assert sys.curves[0].n == 362  # ceil(40 * 9.0172) = 361 -> even
    assert cf.shape == (362,) and tg.shape == (245136, 2)


def test_restatement_coarse_rule_matches_numpy(rest):
    """Far from the curve the evaluation is the plain trapezoidal sum
    (bie.cpp:437-441): an independent numpy statement of dlp_entry
    (bie.cpp:43-50) agrees with the C++ restatement."""
    sys = W.layer_system()
    cf = W.layer_density(sys, seed=3)
    c = sys.curves[0]
    rng = np.random.default_rng(8)
    th = rng.uniform(0, 2 * np.pi, 300)
    tg = np.stack([np.cos(th), np.sin(th)], 1) * rng.uniform(0.0, 0.45, 300)[:, None]
    out, rc = rest.layer_eval(0, 0.0, sys.curves, sys.n_density, sys.n_aux, cf, tg, False)
    assert rc == 0
    d = c.x[None, :, :] - tg[:, None, :]
    r2 = (d ** 2).sum(axis=2)
    dn = (d * c.normal[None, :, :]).sum(axis=2)
    dlp = -dn / (2 * np.pi * r2) * c.speed[None, :]
    ref = (2 * np.pi / c.n) * (dlp * cf[None, :c.n]).sum(axis=1)
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_restatement_helmholtz_coarse_rule_matches_scipy(rest):
    """The modified-Helmholtz double layer -(lambda/2pi) K1(lambda r) dn/r
    speed (bie.cpp:47-49) against scipy's K1, away from the curve."""
    sp = pytest.importorskip("scipy.special")
    k = bie.Kernel(bie.KernelFamily.ModifiedHelmholtz, 10.0)
    sys = W.layer_system(k)
    cf = W.layer_density(sys, seed=4)
    c = sys.curves[0]
    tg = np.array([[0.0, 0.0], [0.2, -0.1], [-0.3, 0.25]])
    out, rc = rest.layer_eval(1, 10.0, sys.curves, sys.n_density, sys.n_aux, cf, tg, False)
    assert rc == 0
    d = c.x[None, :, :] - tg[:, None, :]
    r = np.sqrt((d ** 2).sum(axis=2))
    dn = (d * c.normal[None, :, :]).sum(axis=2)
    dlp = -(10.0 / (2 * np.pi)) * sp.k1(10.0 * r) * (dn / r) * c.speed[None, :]
    ref = (2 * np.pi / c.n) * (dlp * cf[None, :c.n]).sum(axis=1)
    assert np.max(np.abs(out - ref)) <= 1e-12 * np.max(np.abs(ref))
