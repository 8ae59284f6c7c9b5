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


def _correction_csr_loops(nbox_cells, box_ij, ntri_cells, np_box=64, np_tri=64):
    """Plain-loop statement of the synthetic correction map's block layout
    (per target: self + existing 8-neighbour boxes in offset order; triangle
    nodes: one private row) -- the check for the vectorised builder."""
    index = {tuple(ij): k for k, ij in enumerate(map(tuple, box_ij))}
    offsets = [(0, 0)] + [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dx, dy) != (0, 0)]
    npool = len(offsets) * np_box
    blk_cell, blk_pool, blk_off = [], [], [0]
    for c, (i, j) in enumerate(map(tuple, box_ij)):
        nbrs = [(k, index.get((i + o[0], j + o[1]))) for k, o in enumerate(offsets)]
        nbrs = [(k, cell) for k, cell in nbrs if cell is not None]
        for t in range(np_box):
            for k, cell in nbrs:
                blk_cell.append(cell)
                blk_pool.append(k * np_box + t)
            blk_off.append(len(blk_cell))
    for c in range(ntri_cells):
        for t in range(np_tri):
            blk_cell.append(nbox_cells + c)
            blk_pool.append(npool + c * np_tri + t)
            blk_off.append(len(blk_cell))
    return np.array(blk_off), np.array(blk_cell), np.array(blk_pool)


def test_correction_csr_vectorised_matches_loops():
    n = 18
    ij = np.array([(i, j) for j in range(n) for i in range(n) if (i - n / 2) ** 2 + (j - n / 2) ** 2 < (n / 2) ** 2])
    v = W.correction_csr(len(ij), ij, 25)
    bo, bc, bp = _correction_csr_loops(len(ij), ij, 25)
    assert np.array_equal(v["blk_off"], bo) and np.array_equal(v["blk_cell"], bc)
    assert np.array_equal(v["blk_pool"], bp)
    assert int(v["node_off"][-1]) == (len(ij) + 25) * 64
    assert v["pool_off"][-1] == v["pool_vals"].size


def test_cfg5_correction_map_shape():
    w = W.cfg5(n_side=64, ntri=200)
    c = w.notes["corr"]()
    assert c["blk_off"].size - 1 == w.nt == int(c["node_off"][-1])
    assert np.diff(c["blk_off"]).max() <= 9 and np.diff(c["blk_off"]).min() >= 1
    assert np.allclose(w.notes["w"] * w.notes["f"], w.q, rtol=0, atol=0)
