"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures nothing public; BASELINE.json defines five synthetic
node sets (quadrature nodes, weights, densities).  These generators build
them deterministically (numpy PCG64 with fixed seeds).  The FMM step only
sees (points, charges), so the node rule (8x8 Gauss-Legendre here, tensor
Chebyshev/Fejer in the reference operator, basis.cpp:143-180) does not affect
summation parity.

Each generator returns a :class:`Workload` with sources (points, charges =
weight * f) and targets.  Where a config names tolerances, ``eps`` holds them.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

_GL_X, _GL_W = np.polynomial.legendre.leggauss(8)


@dataclass
class Workload:
    name: str
    src: np.ndarray            # (ns, 2)
    q: np.ndarray              # (ns,) charges = weight * f(node)
    tgt: np.ndarray            # (nt, 2)
    kernel: str = "laplace"    # or "helmholtz"
    lam: float = 0.0
    eps: tuple = (1e-12,)
    notes: dict = field(default_factory=dict)

    @property
    def ns(self):
        return len(self.src)

    @property
    def nt(self):
        return len(self.tgt)


def box_nodes(cx, cy, h):
    """8x8 tensor GL nodes and box-scaled weights of boxes centred (cx, cy), side h.

    Returns (n_box*64, 2) points and weights; per box, y index outer, x inner.
    """
    cx = np.atleast_1d(np.asarray(cx, float))
    cy = np.atleast_1d(np.asarray(cy, float))
    h = np.broadcast_to(np.asarray(h, float), cx.shape)
    gx, gy = np.meshgrid(_GL_X, _GL_X)          # gy rows (outer), gx cols (inner)
    wx, wy = np.meshgrid(_GL_W, _GL_W)
    px = cx[:, None] + 0.5 * h[:, None] * gx.ravel()[None, :]
    py = cy[:, None] + 0.5 * h[:, None] * gy.ravel()[None, :]
    w = (0.5 * h[:, None]) ** 2 * (wx * wy).ravel()[None, :]
    return np.stack([px.ravel(), py.ravel()], axis=1), w.ravel()


def gaussian(p, c, alpha):
    d = p - np.asarray(c)[None, :]
    return np.exp(-alpha * (d[:, 0] ** 2 + d[:, 1] ** 2))


def star_radius(theta):
    return 1.0 + 0.3 * np.cos(5.0 * theta)


def _polar(p):
    return np.hypot(p[:, 0], p[:, 1]), np.arctan2(p[:, 1], p[:, 0])


def uniform_grid(nbox_side, lo=-1.0, hi=1.0):
    h = (hi - lo) / nbox_side
    iy, ix = np.meshgrid(np.arange(nbox_side), np.arange(nbox_side), indexing="ij")
    cx = lo + (ix.ravel() + 0.5) * h
    cy = lo + (iy.ravel() + 0.5) * h
    return cx, cy, h


def cfg1():
    """[-1,1]^2, 16x16 boxes x 8x8 GL (16,384 nodes); f = exp(-50|r-c|^2), c=(0.1,-0.2)."""
    cx, cy, h = uniform_grid(16)
    p, w = box_nodes(cx, cy, h)
    q = w * gaussian(p, (0.1, -0.2), 50.0)
    return Workload("cfg1", p, q, p.copy(), notes={"boxes": 256, "h": h})


def _star_boxes(n_side, strip=0.05):
    lo, hi = -1.3, 1.3
    cx, cy, h = uniform_grid(n_side, lo, hi)
    keep = np.ones(cx.shape, bool)
    for sx in (-0.5, 0.5):
        for sy in (-0.5, 0.5):
            r, th = _polar(np.stack([cx + sx * h, cy + sy * h], 1))
            keep &= r < star_radius(th) - strip
    return cx[keep], cy[keep], h


def _strip_triangles(ntri, strip=0.05):
    """ntri curved triangles covering r(theta)-strip <= rho <= r(theta).

    The strip is cut into ntri/2 angular segments; each (theta, s) quad,
    rho = r(theta) - strip (1 - s), splits into two triangles mapped by the
    polar blending map.  64-node collapsed (Duffy) 8x8 GL rule per triangle.
    """
    nseg = ntri // 2
    t0 = np.arange(nseg) * (2 * np.pi / nseg)
    t1 = t0 + 2 * np.pi / nseg
    # triangle vertices in (theta, s): A, B, C
    A = np.concatenate([np.stack([t0, 0 * t0], 1), np.stack([t1, 0 * t1], 1)])
    B = np.concatenate([np.stack([t1, 0 * t1], 1), np.stack([t1, 1 + 0 * t1], 1)])
    Cv = np.concatenate([np.stack([t0, 1 + 0 * t0], 1), np.stack([t0, 1 + 0 * t0], 1)])
    u = 0.5 * (_GL_X + 1.0)
    wu = 0.5 * _GL_W
    U, V = np.meshgrid(u, u, indexing="ij")      # u outer, v inner
    WU, WV = np.meshgrid(wu, wu, indexing="ij")
    U, V, WUV = U.ravel(), V.ravel(), (WU * WV).ravel()
    # Duffy: X = A + u (B - A) + u v (C - B), jacobian u |det(B-A, C-B)|
    pa = A[:, None, :] + U[None, :, None] * (B - A)[:, None, :] + \
        (U * V)[None, :, None] * (Cv - B)[:, None, :]
    e1, e2 = B - A, Cv - B
    det = np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    th, s = pa[..., 0], pa[..., 1]
    rho = star_radius(th) - strip * (1.0 - s)
    pts = np.stack([rho * np.cos(th), rho * np.sin(th)], -1).reshape(-1, 2)
    # d(x,y)/d(theta,s): |det| = rho * d rho/ds = rho * strip
    w = (WUV[None, :] * U[None, :] * det[:, None] * rho * strip).ravel()
    return pts, w


def cfg2(seed=2):
    """Star domain r=1+0.3cos5t: 64x64 clipped box grid + 2,000 strip triangles.

    f = 3 seeded Gaussians (alpha in [20,80]); targets = all nodes + 10,000
    seeded interior points; Laplace FMM at 1e-12.
    """
    rng = np.random.default_rng(seed)
    cx, cy, h = _star_boxes(64)
    pb, wb = box_nodes(cx, cy, h)
    pt, wt = _strip_triangles(2000)
    p = np.concatenate([pb, pt])
    w = np.concatenate([wb, wt])
    cen = rng.uniform(-0.6, 0.6, size=(3, 2))
    alpha = rng.uniform(20, 80, size=3)
    f = sum(gaussian(p, cen[k], alpha[k]) for k in range(3))
    extra = []
    while sum(len(e) for e in extra) < 10_000:
        c = rng.uniform(-1.3, 1.3, size=(20_000, 2))
        r, th = _polar(c)
        extra.append(c[r < star_radius(th)])
    extra = np.concatenate(extra)[:10_000]
    tgt = np.concatenate([p, extra])
    return Workload("cfg2", p, w * f, tgt, notes={"boxes": len(cx), "triangles": 2000, "h": h})


def adaptive_leaves(c, lmin=4, lmax=10, radius=0.14):
    """Quadtree on [-1,1]^2 refined from level lmin to lmax around c.

    Rule (builder-defined): split a box while its level is
    below lmax and the distance from c to the box is below ``radius``.
    Returns leaf centres and sides in depth-first (Morton) order.
    """
    out_c, out_h = [], []

    def rec(x0, y0, s, lev):
        dx = max(x0 - c[0], 0.0, c[0] - (x0 + s))
        dy = max(y0 - c[1], 0.0, c[1] - (y0 + s))
        if lev < lmax and (lev < lmin or np.hypot(dx, dy) < radius):
            hs = 0.5 * s
            for (ox, oy) in ((0, 0), (1, 0), (0, 1), (1, 1)):
                rec(x0 + ox * hs, y0 + oy * hs, hs, lev + 1)
        else:
            out_c.append((x0 + 0.5 * s, y0 + 0.5 * s))
            out_h.append(s)

    rec(-1.0, -1.0, 2.0, 0)
    return np.array(out_c), np.array(out_h)


def cfg3(seed=3):
    """Adaptive quadtree (level 4 -> 10) around a sharp source f=exp(-1000|r-c|^2)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-0.5, 0.5, size=2)
    cen, hs = adaptive_leaves(c)
    p, w = box_nodes(cen[:, 0], cen[:, 1], hs)
    q = w * gaussian(p, c, 1000.0)
    return Workload("cfg3", p, q, p.copy(), notes={"leaves": len(hs), "centre": c.tolist()})


def cfg4(seed=4, nbox_side=256):
    """256x256 boxes x 8x8 GL on [-1,1]^2 (4,194,304 nodes), 16 seeded Gaussians."""
    rng = np.random.default_rng(seed)
    cx, cy, h = uniform_grid(nbox_side)
    p, w = box_nodes(cx, cy, h)
    cen = rng.uniform(-1, 1, size=(16, 2))
    alpha = rng.uniform(10, 200, size=16)
    f = np.zeros(len(p))
    for k in range(16):
        f += gaussian(p, cen[k], alpha[k])
    return Workload("cfg4", p, w * f, p, eps=(1e-6, 1e-9, 1e-12), notes={"h": h})


def cfg5(seed=5, n_side=192, ntri=2000):
    """Modified Helmholtz (lambda=10) on the star domain refined to ~1M nodes.

    Also returns (in notes) a synthetic correction CSR: per target its cell
    (self) plus the existing 8-neighbour box cells (<= 9 blocks x 64), rows
    shared per (offset, local node) for boxes (potential.cpp:256-267) and
    private for triangle self blocks; row values seeded.
    """
    rng = np.random.default_rng(seed)
    cx, cy, h = _star_boxes(n_side)
    pb, wb = box_nodes(cx, cy, h)
    pt, wt = _strip_triangles(ntri)
    p = np.concatenate([pb, pt])
    w = np.concatenate([wb, wt])
    cen = rng.uniform(-0.6, 0.6, size=(3, 2))
    alpha = rng.uniform(20, 80, size=3)
    f = sum(gaussian(p, cen[k], alpha[k]) for k in range(3))
    ij = np.stack([np.rint((cx + 1.3) / h - 0.5), np.rint((cy + 1.3) / h - 0.5)], 1).astype(np.int64)
    wl = Workload("cfg5", p, w * f, p.copy(), kernel="helmholtz", lam=10.0,
                  notes={"boxes": len(cx), "triangles": ntri, "h": h, "f": f, "w": w,
                         "corr": lambda: correction_csr(len(cx), ij, ntri)})
    return wl


def correction_csr(nbox_cells, box_ij, ntri_cells, seed=55, np_box=64, np_tri=64):
    """Synthetic correction map for a mesh of ``nbox_cells`` grid boxes
    (integer grid coordinates ``box_ij``) followed by ``ntri_cells`` triangles.

    Targets are the mesh nodes in order.  Box node t of cell c gets the self
    block plus every existing box among the 8 grid neighbours (<= 9 blocks);
    box rows are shared per (offset, local node) like the reference lattice
    table (potential.cpp:256-267); triangle nodes get one private self row.
    """
    rng = np.random.default_rng(seed)
    ncell = nbox_cells + ntri_cells
    node_off = np.zeros(ncell + 1, np.int64)
    node_off[1:nbox_cells + 1] = np.arange(1, nbox_cells + 1) * np_box
    node_off[nbox_cells + 1:] = nbox_cells * np_box + np.arange(1, ntri_cells + 1) * np_tri
    offsets = [(0, 0)] + [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dx, dy) != (0, 0)]
    # shared lattice rows: 9 offsets x np_box local nodes
    lattice = rng.standard_normal((len(offsets), np_box, np_box)) * 1e-3
    pool_rows = [lattice.reshape(-1, np_box)]
    npool = len(offsets) * np_box
    # neighbour table (box, offset) -> cell or -1, via a dense grid index
    box_ij = np.asarray(box_ij, np.int64).reshape(-1, 2)
    if nbox_cells:
        lo = box_ij.min(0) - 1
        dims = box_ij.max(0) - lo + 2
        grid = np.full((dims[0], dims[1]), -1, np.int64)
        grid[box_ij[:, 0] - lo[0], box_ij[:, 1] - lo[1]] = np.arange(nbox_cells)
        nbr = np.stack([grid[box_ij[:, 0] + o[0] - lo[0], box_ij[:, 1] + o[1] - lo[1]] for o in offsets], 1)
    else:
        nbr = np.zeros((0, len(offsets)), np.int64)
    # box targets: cell-major, node t, existing neighbours in offset order
    exist = nbr >= 0                                             # (nbox, 9)
    cells = np.broadcast_to(nbr[:, None, :], (nbox_cells, np_box, len(offsets)))
    pools = (np.arange(len(offsets))[None, None, :] * np_box + np.arange(np_box)[None, :, None])
    pools = np.broadcast_to(pools, cells.shape)
    m = np.broadcast_to(exist[:, None, :], cells.shape)
    box_cell = cells[m]
    box_pool = pools[m]
    box_cnt = np.repeat(exist.sum(1), np_box)
    tri_rows = rng.standard_normal((ntri_cells * np_tri, np_tri)) * 1e-3
    tri_cell = np.repeat(nbox_cells + np.arange(ntri_cells), np_tri)
    tri_pool = npool + np.arange(ntri_cells * np_tri)
    blk_cell = np.concatenate([box_cell, tri_cell])
    blk_pool = np.concatenate([box_pool, tri_pool])
    blk_off = np.concatenate([[0], np.cumsum(np.concatenate([box_cnt, np.ones(ntri_cells * np_tri, np.int64)]))])
    pool_rows.append(tri_rows)
    vals = np.concatenate([r.reshape(-1) for r in pool_rows])
    lens = np.concatenate([np.full(len(offsets) * np_box, np_box), np.full(ntri_cells * np_tri, np_tri)])
    pool_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return {"blk_off": blk_off.astype(np.int32), "blk_cell": blk_cell.astype(np.int32),
            "blk_pool": blk_pool.astype(np.int32), "pool_off": pool_off, "pool_vals": vals,
            "node_off": node_off.astype(np.int32)}


def reference_correction_csr(box_ij, node_local, ntri_cells=0, np_tri=64, D=0.4, seed=56):
    """Correction map with the reference's near rule and pool layout.

    Targets are the mesh nodes in order (boxes, then triangles).  A box node
    at local coordinates (a, b) in [-1, 1]^2 gets its self block and the
    neighbour boxes closer than D h (classify_target, mesh.cpp:410-448,
    D = 0.4 from mesh.hpp:52): the edge neighbour when (1 -+ a)/2 < D, the
    corner neighbour when both edge distances put it within D h of the
    corner; cells beyond the first ring are >= h away.  Box blocks ride the
    lattice: pool rows shared per key offset_idx * 256 + node, slots in
    order of first appearance (potential.cpp:193-252), offset index
    (oy + 2) * 5 + (ox + 2) of the TARGET's box minus the source box
    (lattice_offset, potential.cpp:196-205).  Triangle nodes get one private
    self row (their near cells are out of this model).  Row values are
    seeded: their provenance does not matter for apply parity.
    """
    rng = np.random.default_rng(seed)
    box_ij = np.asarray(box_ij, np.int64).reshape(-1, 2)
    nbox = len(box_ij)
    node_local = np.asarray(node_local, float).reshape(-1, 2)
    npb = len(node_local)
    a, b = node_local[:, 0], node_local[:, 1]
    dl, dr, db, dt = (a + 1) / 2, (1 - a) / 2, (b + 1) / 2, (1 - b) / 2
    # per node: the neighbour offsets (source box - target box) it is near, cell order below
    near = {}
    for ox in (-1, 0, 1):
        for oy in (-1, 0, 1):
            if ox == 0 and oy == 0:
                continue
            dx = dl if ox < 0 else dr if ox > 0 else np.zeros(npb)
            dy = db if oy < 0 else dt if oy > 0 else np.zeros(npb)
            near[(ox, oy)] = np.hypot(dx, dy) < D
    lo = box_ij.min(0) - 2 if nbox else np.zeros(2, np.int64)
    dims = (box_ij.max(0) - lo + 3) if nbox else np.ones(2, np.int64)
    grid = np.full((int(dims[0]), int(dims[1])), -1, np.int64)
    if nbox:
        grid[box_ij[:, 0] - lo[0], box_ij[:, 1] - lo[1]] = np.arange(nbox)
    blk_cell, blk_key, cnt = [], [], []
    order = sorted(near)  # neighbour scan order (fixed)
    for c in range(nbox):
        i, j = box_ij[c]
        nb = [(o, grid[i + o[0] - lo[0], j + o[1] - lo[1]]) for o in order]
        nb = [(o, k) for o, k in nb if k >= 0]
        for u in range(npb):
            blk_cell.append(c)
            blk_key.append(12 * 256 + u)  # self: offset (0, 0)
            m = 1
            for o, k in nb:
                if near[o][u]:
                    blk_cell.append(k)
                    blk_key.append(((-o[1] + 2) * 5 + (-o[0] + 2)) * 256 + u)
                    m += 1
            cnt.append(m)
    slot = {}
    blk_pool = []
    for key in blk_key:
        if key not in slot:
            slot[key] = len(slot)
        blk_pool.append(slot[key])
    nlat = len(slot)
    lat_rows = rng.standard_normal((nlat, npb)) * 1e-3
    tri_rows = rng.standard_normal((ntri_cells * np_tri, np_tri)) * 1e-3
    tri_cell = np.repeat(nbox + np.arange(ntri_cells), np_tri)
    blk_cell = np.concatenate([np.asarray(blk_cell, np.int64), tri_cell])
    blk_pool = np.concatenate([np.asarray(blk_pool, np.int64), nlat + np.arange(ntri_cells * np_tri)])
    cnt = np.concatenate([np.asarray(cnt, np.int64), np.ones(ntri_cells * np_tri, np.int64)])
    node_off = np.concatenate([[0], np.cumsum(np.concatenate([np.full(nbox, npb), np.full(ntri_cells, np_tri)]))])
    lens = np.concatenate([np.full(nlat, npb), np.full(ntri_cells * np_tri, np_tri)])
    vals = np.concatenate([lat_rows.reshape(-1), tri_rows.reshape(-1)])
    return {"blk_off": np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32),
            "blk_cell": blk_cell.astype(np.int32), "blk_pool": blk_pool.astype(np.int32),
            "pool_off": np.concatenate([[0], np.cumsum(lens)]).astype(np.int64), "pool_vals": vals,
            "node_off": node_off.astype(np.int32)}


def fejer1(p):
    """Chebyshev roots ascending with Fejer-1 weights (basis.cpp:140-156)."""
    th = (2 * np.arange(p) + 1) * np.pi / (2 * p)
    k = np.arange(1, p // 2 + 1)
    s = (np.cos(2 * k[None, :] * th[:, None]) / (4.0 * k * k - 1.0)).sum(1)
    return -np.cos(th), (2.0 / p) * (1 - 2 * s)


def _cheb1d(p, z):
    t = np.zeros((len(z), p))
    t[:, 0] = 1.0
    if p > 1:
        t[:, 1] = z
    for k in range(2, p):
        t[:, k] = 2 * z * t[:, k - 1] - t[:, k - 2]
    return t


def chebyshev2d(p, zx, zy):
    """chebyshev2d_eval (basis.cpp:259-265): out[a p + b] = T_a(x) T_b(y)."""
    tx, ty = _cheb1d(p, np.asarray(zx, float)), _cheb1d(p, np.asarray(zy, float))
    return (tx[:, :, None] * ty[:, None, :]).reshape(len(tx), p * p)


def box_tables(p, q):
    """The reference's box tables: p-node Fejer tensor nodes (index ix * p +
    iy, basis.cpp:158-177), the q-node source rule (basis.cpp:281-303) and
    box_oversample(p, q) = B C with B the degree-p Chebyshev basis at the
    source nodes and C = V^-1 (basis.cpp:305-322)."""
    z, w = fejer1(p)
    ix, iy = np.meshgrid(np.arange(p), np.arange(p), indexing="ij")
    nodes = np.stack([z[ix.ravel()], z[iy.ravel()]], 1)
    zq, wq = fejer1(q)
    jx, jy = np.meshgrid(np.arange(q), np.arange(q), indexing="ij")
    src = np.stack([zq[jx.ravel()], zq[jy.ravel()]], 1)
    wsrc = wq[jx.ravel()] * wq[jy.ravel()]
    V = chebyshev2d(p, nodes[:, 0], nodes[:, 1])
    C = np.linalg.inv(V)
    O = chebyshev2d(p, src[:, 0], src[:, 1]) @ C
    return nodes, src, wsrc, O, C


def op_box(n_side=32, p=8, q=16, seed=7):
    """The reference operator's data on a box mesh (SPEC acceptance 7 size:
    32 x 32 boxes on [-1,1]^2, p = 8 -> 65,536 ndofs): targets = the p x p
    Fejer nodes of every box, sources = the q x q oversampled nodes
    (q = 2p, 262,144) with weights w_s * jacobian, build_charges through
    O = box_oversample(p, q) (256 x 64), the correction CSR from the
    reference near rule (reference_correction_csr).  f = a seeded smooth
    field at the nodes."""
    rng = np.random.default_rng(seed)
    cx, cy, h = uniform_grid(n_side)
    nodes, src, wsrc, O, _ = box_tables(p, q)
    tgt = np.stack([(cx[:, None] + 0.5 * h * nodes[None, :, 0]).ravel(),
                    (cy[:, None] + 0.5 * h * nodes[None, :, 1]).ravel()], 1)
    spts = np.stack([(cx[:, None] + 0.5 * h * src[None, :, 0]).ravel(),
                     (cy[:, None] + 0.5 * h * src[None, :, 1]).ravel()], 1)
    wj = np.tile(wsrc * (h * h / 4.0), len(cx))
    cen = rng.uniform(-0.6, 0.6, size=(3, 2))
    f = sum(gaussian(tgt, cen[k], 40.0) for k in range(3))
    ij = np.stack([np.rint((cx + 1.0) / h - 0.5), np.rint((cy + 1.0) / h - 0.5)], 1).astype(np.int64)
    nbox = len(cx)
    charge_map = {"cell_type": np.zeros(nbox, np.int32),
                  "node_off": (np.arange(nbox + 1) * p * p).astype(np.int32),
                  "src_off": (np.arange(nbox + 1) * q * q).astype(np.int32),
                  "over0": O, "over1": np.zeros((0, 0)), "src_wj": wj}
    q_ch = wj * (np.einsum("sij,cj->csi", O[None], f.reshape(nbox, p * p)).reshape(-1))
    return Workload("op_box", spts, q_ch, tgt, notes={
        "h": h, "f": f, "charges": charge_map, "boxes": nbox,
        "corr": lambda: reference_correction_csr(ij, nodes)})


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5, "op_box": op_box}


def random_points(n, seed, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(n, 2))


def layer_system(kernel=None, n=None, holes=False):
    """Star boundary r = 1 + 0.3 cos 5t (configs[1]) as a BoundarySystem
    geometry; n defaults to solve_bvp's rule ceil(max(64, 40 L)), made even,
    and at least 0.5 lambda L for modified Helmholtz (bie.cpp:478-491).
    ``holes`` adds a circular hole (a Laplace log-completion coefficient)."""
    from . import bie
    from .summation import KernelFamily, make_kernel
    kernel = kernel or make_kernel(KernelFamily.Laplace)
    curves = [bie.star_curve()]
    if holes:
        curves.append(bie.circle_curve(0.15, -0.1, 0.3, hole=True))
    counts = []
    for c in curves:
        if n:
            counts.append(n + n % 2)
            continue
        ln = c.total_arclength()
        want = max(64.0, 40.0 * ln)
        if kernel.family == KernelFamily.ModifiedHelmholtz:
            want = max(want, 0.5 * kernel.lam * ln)
        k = int(np.ceil(want))
        counts.append(k + k % 2)
    return bie.assemble_geometry(curves, counts, kernel)


def layer_density(sys, seed=7, modes=12):
    """A seeded smooth periodic density per curve (a few Fourier modes with
    decaying amplitudes) plus seeded log coefficients."""
    rng = np.random.default_rng(seed)
    out = []
    for c in sys.curves:
        t = 2.0 * np.pi * np.arange(c.n) / c.n
        v = np.full(c.n, rng.uniform(-1, 1))
        for m in range(1, modes + 1):
            a, b = rng.uniform(-1, 1, 2) / m
            v += a * np.cos(m * t) + b * np.sin(m * t)
        out.append(v)
    return np.concatenate(out + [rng.uniform(-1, 1, sys.n_aux)])


def layer_cfg2(kernel=None, seed=2):
    """Layer-potential workload on configs[1]: the star boundary system, a
    seeded density, targets = the cfg2 nodes + 10,000 interior points
    (solve_bvp evaluates at mesh nodes + targets with allow_close,
    bie.cpp:520-523)."""
    w = cfg2(seed)
    sys = layer_system(kernel)
    return sys, layer_density(sys), w.tgt


# ------------------------------------------------------------ mesh operators --
GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _star_eval(par, t, order):
    """StarCurve pos / derivatives (geometry.cpp:106-132), vectorised."""
    cx, cy, r0, amp, arms, ph = par
    k = arms
    ct, st = np.cos(t), np.sin(t)
    ck, sk = np.cos(k * t + ph), np.sin(k * t + ph)
    rho = r0 * (1 + amp * ck)
    u = np.stack([ct, st], -1)
    up = np.stack([-st, ct], -1)
    if order == 0:
        return np.array([cx, cy]) + rho[..., None] * u
    drho = -r0 * amp * k * sk
    if order == 1:
        return drho[..., None] * u + rho[..., None] * up
    d2rho = -r0 * amp * k * k * ck
    if order == 2:
        return (d2rho - rho)[..., None] * u + (2 * drho)[..., None] * up
    d3rho = r0 * amp * k * k * k * sk
    return (d3rho - 3 * drho)[..., None] * u + (3 * d2rho - rho)[..., None] * up


def map_cells(mesh, ref_pts):
    """Cell::map_deriv (geometry.cpp:198-223) of every cell at the reference
    points ref_pts[kind] (kind 0 triangle, 1 box): returns (xy, jac) in cell
    order, ref_pts[kind] points per cell."""
    typ = np.asarray(mesh["type"])
    out_x, out_j = [], []
    star = mesh["star"]
    for c in range(len(typ)):
        z = ref_pts[1] if typ[c] == 2 else ref_pts[0]
        if typ[c] == 2:
            cx, cy, h = mesh["ch"][c]
            out_x.append(np.array([cx, cy]) + (h / 2) * z)
            out_j.append(np.full(len(z), h * h / 4))
            continue
        v0, v1, v2 = mesh["v"][c]
        e1, e2 = v1 - v0, v2 - v0
        if typ[c] == 0:
            out_x.append(v0 + z[:, :1] * e1 + z[:, 1:] * e2)
            out_j.append(np.full(len(z), e1[0] * e2[1] - e1[1] * e2[0]))
            continue
        ta, tb = mesh["tt"][c]
        dt = tb - ta
        xi = z[:, 0]
        s = 1 - xi
        far = s >= 1e-5
        phi = np.zeros((len(z), 2))
        dphi = np.zeros((len(z), 2))
        t = ta + xi * dt
        lam = _star_eval(star, t, 0)
        dlam = dt * _star_eval(star, t, 1)
        num = lam - (1 - xi)[:, None] * v0 - xi[:, None] * v1
        with np.errstate(divide="ignore", invalid="ignore"):
            phi_f = (1.0 / s)[:, None] * num
            dphi_f = (1.0 / s)[:, None] * (dlam - e1 + phi_f)
        d1 = dt * _star_eval(star, np.array([tb]), 1)[0]
        d2 = dt * dt * _star_eval(star, np.array([tb]), 2)[0]
        d3 = dt * dt * dt * _star_eval(star, np.array([tb]), 3)[0]
        phi_n = -1.0 * (d1 - e1) + (s / 2)[:, None] * d2 - (s * s / 6)[:, None] * d3
        dphi_n = -0.5 * d2 + (s / 3)[:, None] * d3
        phi = np.where(far[:, None], phi_f, phi_n)
        dphi = np.where(far[:, None], dphi_f, dphi_n)
        blend = (1 - z[:, 0] - z[:, 1])[:, None]
        dxi = e1 - phi + blend * dphi
        deta = e2 - phi
        out_x.append(v0 + z[:, :1] * e1 + z[:, 1:] * e2 + blend * phi)
        out_j.append(dxi[:, 0] * deta[:, 1] - dxi[:, 1] * deta[:, 0])
    return np.concatenate(out_x), np.concatenate(out_j)


def op_star(h_name="star_h00125", p=8, q=16, family=0, lam=0.0, seed=9):
    """The volume-potential operator of the configs[1] star on the reference's
    own hybrid mesh (tests/golden/mesh_<h_name>.npz, built by build_mesh) with
    the reference's p = 8 / q = 16 rules: targets = the mesh nodes, sources =
    the oversampled source rule, f = 3 seeded Gaussians (alpha in [20, 80]).
    The step is the operator apply (build_charges + FMM + correction,
    potential.cpp:431-470); the correction map is built on the device
    (csrc/rows.cu).  src/q here are the FMM step's points and charges."""
    m = dict(np.load(os.path.join(GOLDEN, f"mesh_{h_name}.npz")))
    b = dict(np.load(os.path.join(GOLDEN, f"basis_p{p}_q{q}.npz")))
    nodes, _ = map_cells(m, [b["tri_nodes"], b["box_nodes"]])
    src, jac = map_cells(m, [b["tri_src"], b["box_src"]])
    box = m["type"] == 2
    w = np.concatenate([b["box_src_w"] if bx else b["tri_src_w"] for bx in box])
    wj = w * jac
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-0.5, 0.5, size=(3, 2))
    al = rng.uniform(20, 80, size=3)
    f = sum(gaussian(nodes, cen[k], al[k]) for k in range(3))
    fs = sum(gaussian(src, cen[k], al[k]) for k in range(3))
    name = "op_star" if family == 0 else "op_star_mh"
    return Workload(name, src, wj * fs, nodes, kernel="laplace" if family == 0 else "helmholtz", lam=lam,
                    notes={"mesh": m, "basis": b, "f": f, "src_wj": wj, "p": p, "q": q, "h_name": h_name,
                           "cells": int(len(m["type"])), "n_tri": int(m["n_tri"]), "n_box": int(m["n_box"])})


CONFIGS["op_star"] = op_star
CONFIGS["op_star_mh"] = lambda: op_star(family=1, lam=10.0)
CONFIGS["op_star_84k"] = lambda: op_star(h_name="star_h005")
