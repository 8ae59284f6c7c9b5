"""Synthetic BASELINE configs: sizes and seeded determinism."""
import hashlib

import numpy as np
import pytest

from paper_2203_05933_b200 import workloads as W


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def test_cfg1_shape_and_charge():
    w = W.cfg1()
    assert w.ns == w.nt == 16_384
    assert abs(w.q.sum() - np.pi / 50) < 1e-15
    assert np.array_equal(w.src, w.tgt)


def test_cfg2_counts():
    w = W.cfg2()
    assert w.notes["boxes"] == 1674 and w.ns == 1674 * 64 + 2000 * 64 == 235_136
    assert w.nt == w.ns + 10_000
    r = np.hypot(w.tgt[-10_000:, 0], w.tgt[-10_000:, 1])
    th = np.arctan2(w.tgt[-10_000:, 1], w.tgt[-10_000:, 0])
    assert np.all(r < W.star_radius(th))
    # strip quadrature integrates the strip area
    area = 0.5 * np.sum((1 + 0.3 * np.cos(5 * np.linspace(0, 2 * np.pi, 200001)[:-1])) ** 2
                        - (1 + 0.3 * np.cos(5 * np.linspace(0, 2 * np.pi, 200001)[:-1]) - 0.05) ** 2) * (2 * np.pi / 200000)
    _, wt = W._strip_triangles(2000)
    assert abs(wt.sum() - area) < 1e-10


def test_cfg3_adaptive():
    w = W.cfg3()
    assert 1_000_000 <= w.ns <= 1_200_000 and w.ns % 64 == 0
    assert abs(w.q.sum() - np.pi / 1000) < 1e-9  # sharp Gaussian well inside the square


def test_cfg4_size():
    w = W.cfg4()
    assert w.ns == w.nt == 4_194_304 and w.eps == (1e-6, 1e-9, 1e-12)


def test_deterministic():
    a, b = W.cfg2(), W.cfg2()
    assert digest(a.src, a.q, a.tgt) == digest(b.src, b.q, b.tgt)


def test_correction_csr_bounds():
    ij = np.array([(i, j) for j in range(10) for i in range(10)])
    csr = W.correction_csr(len(ij), ij, 5)
    nb = np.diff(csr["blk_off"])
    assert nb.max() <= 9 and nb.min() >= 1
    assert csr["pool_off"][-1] == len(csr["pool_vals"])
