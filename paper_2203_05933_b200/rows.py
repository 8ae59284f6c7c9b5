"""Correction-row generation on the GPU (csrc/rows.cu).

Python mirror of the row builders behind VolumePotentialOperator's
correction map (potential.cpp:133-349):

Reference symbol (file:line)                      here (RowEngine job)
------------------------------------------------  ------------------------
SingularTargetRule::row (singular.cpp:383-415)    JOB_SELF
reduce_to_rays + apply_ray_quadrature (274-310)   JOB_RAY
smooth_potential_row (singular.cpp:428-456)       JOB_SMOOTH
operator rows (potential.cpp:276-333, 351-358)    JOB_TRI_SELF_NODE .. JOB_NEAR_GENERIC
box lattice rows (potential.cpp:269-289)          JOB_LATTICE
box_log / box_correction_table (486-646)          JOB_TABLE_LAP / JOB_TABLE_HELM

A :class:`Mesh` carries the cells and curves the rows integrate over
(geometry.hpp:90-100); the basis data (triangle nodes and C, box C, the
triangle source rule) come from the caller, as the reference's
TriangleBasisTable / BoxBasisTable (basis.hpp:13-56).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

JOB_SELF, JOB_RAY, JOB_SMOOTH = 0, 1, 2
JOB_TRI_SELF_NODE, JOB_TRI_NEAR_SNAP, JOB_SELF_GENERIC, JOB_NEAR_GENERIC = 3, 4, 5, 6
JOB_LATTICE, JOB_TABLE_LAP, JOB_TABLE_HELM = 7, 8, 9

CELL_STRAIGHT_TRI, CELL_CURVED_TRI, CELL_BOX = 0, 1, 2
CURVE_CIRCLE, CURVE_ELLIPSE, CURVE_STAR = 0, 1, 2


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


@dataclass
class Mesh:
    """Cells (type, curve, vertices [n,3,2], (ta, tb) [n,2], (cx, cy, h) [n,3])
    and curves (kind [m], params [m,6])."""

    cell_type: np.ndarray
    cell_curve: np.ndarray
    cell_v: np.ndarray
    cell_t: np.ndarray
    cell_ch: np.ndarray
    curve_kind: np.ndarray
    curve_par: np.ndarray

    @property
    def ncell(self):
        return int(len(self.cell_type))


class RowEngine:
    def __init__(self, mesh: Mesh, family: int, lam: float, p: int, q: int, tri_nodes, tri_C, box_C,
                 tri_src_xy, tri_src_w, device: int = 0):
        self.mesh, self.family, self.lam, self.p, self.q = mesh, family, lam, p, q
        self._keep = [_i32(mesh.curve_kind), _f64(mesh.curve_par), _i32(mesh.cell_type), _i32(mesh.cell_curve),
                      _f64(mesh.cell_v), _f64(mesh.cell_t), _f64(mesh.cell_ch), _f64(tri_nodes), _f64(tri_C),
                      _f64(box_C), _f64(tri_src_xy), _f64(tri_src_w)]
        ck, cp, ct, cc, cv, tt, ch, tn, tC, bC, ts, tw = self._keep
        h = C.c_void_p()
        L.check(L.lib().vpg_rows_create(family, lam, p, q, ck.size, _p(ck), _p(cp), ct.size, _p(ct), _p(cc),
                                        _p(cv), _p(tt), _p(ch), _p(tn), _p(tC), _p(bC), tw.size, _p(ts), _p(tw),
                                        device, C.byref(h)), "RowEngine")
        self._h = h

    def rule(self, which):
        n = C.c_int64()
        L.check(L.lib().vpg_rows_rule(self._h, which, None, None, C.byref(n)), "rule")
        x, w = np.empty(n.value), np.empty(n.value)
        L.check(L.lib().vpg_rows_rule(self._h, which, _p(x), _p(w), C.byref(n)), "rule")
        return x, w

    def eval(self, job, cell, aux=None, r0=None, zeta0=None, zstar=None, lattice_h=0.0):
        """Rows of the given tasks (arrays of equal length); returns a list."""
        job, cell = _i32(job), _i32(cell)
        n = job.size
        aux = _i32(aux if aux is not None else np.zeros(n))
        arrs = [None if a is None else _f64(a).reshape(n, 2) for a in (r0, zeta0, zstar)]
        ln = C.c_int64()
        args = [self._h, n, _p(job), _p(cell), _p(aux)] + [_p(a) for a in arrs] + [lattice_h]
        L.check(L.lib().vpg_rows_eval(*args, None, C.byref(ln)), "rows")
        out = np.empty(ln.value)
        L.check(L.lib().vpg_rows_eval(*args, _p(out), C.byref(ln)), "rows")
        rows, at = [], 0
        for k in range(n):
            c = cell[k]
            box = c < 0 or c >= self.mesh.ncell or self.mesh.cell_type[c] == CELL_BOX or job[k] in (
                JOB_LATTICE, JOB_TABLE_LAP, JOB_TABLE_HELM)
            nb = self.p * self.p if box else self.p * (self.p + 1) // 2
            rows.append(out[at:at + nb])
            at += nb
        return rows

    def mesh_nodes(self):
        """mesh_nodes(mesh, p) (potential.cpp:63-74): [ndofs, 2] in cell order."""
        n = C.c_int64()
        L.check(L.lib().vpg_rows_map(self._h, 0, None, None, C.byref(n)), "mesh_nodes")
        xy = np.empty((n.value, 2))
        L.check(L.lib().vpg_rows_map(self._h, 0, _p(xy), None, C.byref(n)), "mesh_nodes")
        return xy

    def sources(self):
        """build_sources (potential.cpp:133-151): (src_xy [nsrc, 2], src_wj [nsrc])."""
        n = C.c_int64()
        L.check(L.lib().vpg_rows_map(self._h, 1, None, None, C.byref(n)), "build_sources")
        xy, wj = np.empty((n.value, 2)), np.empty(n.value)
        L.check(L.lib().vpg_rows_map(self._h, 1, _p(xy), _p(wj), C.byref(n)), "build_sources")
        return xy, wj

    def close(self):
        if getattr(self, "_h", None):
            L.lib().vpg_rows_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_correction_map(engine: RowEngine, nodes, node_off, targets, D: float = 0.4):
    """build_corrections (potential.cpp:133-349) on the device: returns
    (CorrectionMap, stats dict)."""
    from .correction import CorrectionMap
    nd = _f64(nodes).reshape(-1, 2)
    no = _i32(node_off)
    tg = _f64(targets).reshape(-1, 2)
    h = C.c_void_p()
    st = np.zeros(13)
    L.check(L.lib().vpg_corr_build(engine._h, len(nd), _p(nd), _p(no), len(tg), _p(tg), D, C.byref(h), _p(st)),
            "build_corrections")
    cm = CorrectionMap.__new__(CorrectionMap)
    cm._arrays = [no]
    cm._h = h
    cm.num_targets = len(tg)
    cm.ndofs = int(no[-1])
    sz = np.zeros(5, np.int64)
    L.check(L.lib().vpg_corr_export(h, None, None, None, None, None, _p(sz)), "export")
    cm.nblocks = int(sz[1])
    keys = ("classify_ms", "tasks_ms", "rows_ms", "blocks", "pool_rows", "pool_len", "tri_self_node",
            "tri_near_snap", "self_generic", "near_generic", "box_lattice", "quad_nodes_tri", "quad_nodes_box")
    return cm, dict(zip(keys, st.tolist()))


def export_map(cm):
    """The map's arrays (blk_off, blk_cell, blk_pool, pool_off, pool_vals)."""
    sz = np.zeros(5, np.int64)
    L.check(L.lib().vpg_corr_export(cm._h, None, None, None, None, None, _p(sz)), "export")
    nt, nb, npool, nv = (int(x) for x in sz[:4])
    d = dict(blk_off=np.empty(nt + 1, np.int32), blk_cell=np.empty(nb, np.int32), blk_pool=np.empty(nb, np.int32),
             pool_off=np.empty(npool + 1, np.int64), pool_vals=np.empty(nv))
    L.check(L.lib().vpg_corr_export(cm._h, *(_p(d[k]) for k in ("blk_off", "blk_cell", "blk_pool", "pool_off",
                                                                   "pool_vals")), None), "export")
    return d


# ------------------------------------------------------- operator from a mesh --
def load_mesh(path):
    """A hybrid mesh stored as the reference builds it (tests/golden/
    make_golden_mesh.py): returns (Mesh, h)."""
    d = np.load(path)
    mesh = Mesh(d["type"], d["curve"], d["v"], d["tt"], d["ch"], np.array([CURVE_STAR]), d["star"][None, :])
    return mesh, float(d["h"])


def load_basis(path):
    return dict(np.load(path))


def build_operator(mesh: Mesh, basis: dict, family: int, lam: float, p: int, q: int, eps: float = 1e-12,
                   targets=None, D: float = 0.4, device: int = 0):
    """VolumePotentialOperator (potential.cpp:360-395) assembled on the GPU:
    mesh_nodes and build_sources from the cells, the SummationPlan over the
    oversampled sources, the charge map with the basis' oversampling
    matrices, and the correction map built on the device (build_corrections).
    Returns a dict with the operator and its parts."""
    import time

    from .correction import ChargeMap, VolumePotentialOperator
    from .summation import KernelFamily, SummationPlan, make_kernel
    t0 = time.perf_counter()
    eng = RowEngine(mesh, family, lam, p, q, basis["tri_nodes"], basis["tri_C"], basis["box_C"], basis["tri_src"],
                    basis["tri_src_w"], device=device)
    nodes = eng.mesh_nodes()
    src_xy, src_wj = eng.sources()
    box = np.asarray(mesh.cell_type) == CELL_BOX
    npc = np.where(box, p * p, p * (p + 1) // 2)
    nqc = np.where(box, basis["box_over"].shape[0], basis["tri_over"].shape[0])
    node_off = np.concatenate([[0], np.cumsum(npc)]).astype(np.int32)
    src_off = np.concatenate([[0], np.cumsum(nqc)]).astype(np.int32)
    tgt = nodes if targets is None else np.asarray(targets, dtype=np.float64).reshape(-1, 2)
    t1 = time.perf_counter()
    corr, stats = build_correction_map(eng, nodes, node_off, tgt, D)
    t2 = time.perf_counter()
    k = make_kernel(KernelFamily.Laplace) if family == 0 else make_kernel(KernelFamily.ModifiedHelmholtz, lam)
    plan = SummationPlan(k, src_xy, tgt, eps, device=device)
    charges = ChargeMap(np.where(box, 0, 1).astype(np.int32), node_off, src_off, basis["box_over"],
                        basis["tri_over"], src_wj, device=device)
    op = VolumePotentialOperator(plan, corr, charges)
    t3 = time.perf_counter()
    stats.update(setup_ms=(t1 - t0) * 1e3, corr_build_ms=(t2 - t1) * 1e3, plan_ms=(t3 - t2) * 1e3)
    return dict(op=op, plan=plan, charges=charges, corr=corr, engine=eng, nodes=nodes, targets=tgt,
                src_xy=src_xy, src_wj=src_wj, node_off=node_off, src_off=src_off, stats=stats)
