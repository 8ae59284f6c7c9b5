"""ctypes access to the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline -- never as the product path (paper_2203_05933_b200 never
imports it).

* :func:`restatement` -- libvolpot_oracle.so, our CPU restatement of the
  reference algorithm (oracle/volpot_oracle.cpp, each function citing the
  reference file:line it follows).
* :func:`reference` -- oracle/_ref/libvolpot_ref.so, the UNMODIFIED
  reference summation sources compiled in place from /root/reference
  (oracle/Makefile) behind a tiny extern "C" shim.  Travels to the GPU box
  as a prebuilt .so.
* :func:`reference_operator` -- oracle/_ref/libvolpot_ref_op.so, the
  UNMODIFIED reference operator sources (mesh, basis, quadrature, singular
  rules, potential, bie) compiled in place against our restatement of the
  Eigen subset they use (oracle/eigen_restated/; Eigen is absent here).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libvolpot_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvolpot_ref.so")
REFOP_SO = os.path.join(HERE, "_ref", "libvolpot_ref_op.so")
REF_SRC = "/root/reference/proj"

_P = C.c_void_p


def build(force: bool = False) -> None:
    """make -C oracle (the reference .so only where /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        targets += ["ref", "refop"]
    if force or not os.path.exists(ORACLE_SO) or (
            "ref" in targets and not (os.path.exists(REF_SO) and os.path.exists(REFOP_SO))):
        subprocess.run(["make", "-C", HERE] + targets, check=True,
                       stdout=subprocess.DEVNULL)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def _pts(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(-1, 2) if a.size else a.reshape(0, 2)


def _vec(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


class VoParams(C.Structure):
    _fields_ = [("direct", C.c_int), ("levels", C.c_int), ("order", C.c_int),
                ("eps", C.c_double), ("x0", C.c_double), ("y0", C.c_double),
                ("side", C.c_double)]


class VoCurve(C.Structure):
    _fields_ = [("n", C.c_int), ("offset", C.c_int), ("length", C.c_double), ("diam", C.c_double),
                ("x", _P), ("normal", _P), ("speed", _P), ("fine_x", _P), ("fine_normal", _P),
                ("fine_speed", _P), ("log_center", C.c_double * 2)]


class Restatement:
    """Our CPU restatement (volpot_oracle.h)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        h = C.CDLL(ORACLE_SO)
        i64, i32p = C.c_int64, C.POINTER(C.c_int32)
        h.vo_plan_params.argtypes = [C.c_int, C.c_double, _P, i64, _P, i64, C.c_double, C.POINTER(VoParams)]
        h.vo_bin_points.argtypes = [_P, i64, C.c_int, C.c_double, C.c_double, C.c_double, _P, _P]
        h.vo_bin_points.restype = None
        h.vo_count_levels.argtypes = [C.c_int, _P, _P]
        h.vo_count_levels.restype = None
        h.vo_m2l_list.argtypes = [C.c_int, C.c_int, _P, _P, i32p, _P, _P, _P, _P]
        h.vo_m2l_list.restype = i64
        h.vo_p2p_pairs.argtypes = [C.c_int, _P, _P]
        h.vo_p2p_pairs.restype = i64
        h.vo_plan_sum.argtypes = [C.c_int, C.c_double, _P, _P, i64, _P, i64, C.c_double, _P, C.c_int]
        h.vo_direct_sum.argtypes = [C.c_int, C.c_double, _P, _P, i64, _P, i64, _P,
                                    C.POINTER(i64), C.POINTER(i64), C.c_int]
        h.vo_pairwise_sum_ld.argtypes = [C.c_int, C.c_double, _P, _P, i64, _P, i64, _P, C.c_int]
        h.vo_pairwise_sum_ld.restype = None
        h.vo_bessel_k0.argtypes = [C.c_double]
        h.vo_bessel_k0.restype = C.c_double
        h.vo_bessel_k1.argtypes = [C.c_double]
        h.vo_bessel_k1.restype = C.c_double
        h.vo_trig_upsample.argtypes = [_P, C.c_int, C.c_int, _P]
        h.vo_trig_upsample.restype = None
        h.vo_layer_eval.argtypes = [C.c_int, C.c_double, _P, C.c_int, C.c_int, C.c_int, _P, i64, _P, i64,
                                    C.c_int, _P, C.c_int]
        h.vo_correction_apply.argtypes = [i64, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int]
        h.vo_correction_apply.restype = None
        h.vo_build_charges.argtypes = [i64, _P, _P, _P, _P, C.c_int, C.c_int, _P, C.c_int,
                                       C.c_int, _P, _P, _P, C.c_int]
        h.vo_build_charges.restype = None
        self.h = h

    def params(self, family, lam, src, tgt, eps):
        src, tgt = _pts(src), _pts(tgt)
        p = VoParams()
        self.h.vo_plan_params(family, lam, _p(src), len(src), _p(tgt), len(tgt), eps, C.byref(p))
        return {f: getattr(p, f) for f, _ in VoParams._fields_}

    def tree(self, src, tgt, eps=1e-12):
        """Leaf CSR + level counts exactly as summation.cpp:117-129."""
        src, tgt = _pts(src), _pts(tgt)
        pr = self.params(0, 0.0, src, tgt, eps)
        Lv = pr["levels"]
        nleaf, nall = 4 ** Lv, (4 ** (Lv + 1) - 1) // 3
        out = {"params": pr}
        for name, pts in (("src", src), ("tgt", tgt)):
            off = np.empty(nleaf + 1, np.int32)
            ids = np.empty(len(pts), np.int32)
            self.h.vo_bin_points(_p(pts), len(pts), Lv, pr["x0"], pr["y0"], pr["side"], _p(off), _p(ids))
            cnt = np.empty(nall, np.int32)
            self.h.vo_count_levels(Lv, _p(off), _p(cnt))
            out[name + "_off"], out[name + "_ids"], out[name + "_cnt"] = off, ids, cnt
        return out

    def m2l_list(self, levels, level, src_cnt, tgt_cnt):
        nt = C.c_int32(0)
        ne = self.h.vo_m2l_list(levels, level, _p(src_cnt), _p(tgt_cnt), C.byref(nt), None, None, None, None)
        r = {"tbox": np.empty(nt.value, np.int32), "toff": np.empty(nt.value + 1, np.int32),
             "src": np.empty(ne, np.int32), "oidx": np.empty(ne, np.int32)}
        self.h.vo_m2l_list(levels, level, _p(src_cnt), _p(tgt_cnt), C.byref(nt),
                           *(_p(r[k]) for k in ("tbox", "toff", "src", "oidx")))
        return r

    def p2p_pairs(self, levels, src_off, tgt_off):
        return self.h.vo_p2p_pairs(levels, _p(src_off), _p(tgt_off))

    def plan_sum(self, family, lam, src, q, tgt, eps=1e-12, threads=0):
        src, tgt, q = _pts(src), _pts(tgt), _vec(q)
        out = np.empty(len(tgt))
        rc = self.h.vo_plan_sum(family, lam, _p(src), _p(q), len(src), _p(tgt), len(tgt), eps, _p(out), threads)
        if rc:
            raise ValueError("vo_plan_sum failed")
        return out

    def direct_sum(self, family, lam, src, q, tgt, threads=0):
        src, tgt, q = _pts(src), _pts(tgt), _vec(q)
        out = np.empty(len(tgt))
        ci, cj = C.c_int64(-1), C.c_int64(-1)
        rc = self.h.vo_direct_sum(family, lam, _p(src), _p(q), len(src), _p(tgt), len(tgt), _p(out),
                                  C.byref(ci), C.byref(cj), threads)
        return out, rc, (ci.value, cj.value)

    def pairwise_ld(self, family, lam, src, q, tgt, threads=0):
        src, tgt, q = _pts(src), _pts(tgt), _vec(q)
        out = np.empty(len(tgt))
        self.h.vo_pairwise_sum_ld(family, lam, _p(src), _p(q), len(src), _p(tgt), len(tgt), _p(out), threads)
        return out

    def bessel_k0(self, xs):
        return np.array([self.h.vo_bessel_k0(float(x)) for x in np.ravel(xs)])

    def bessel_k1(self, xs):
        return np.array([self.h.vo_bessel_k1(float(x)) for x in np.ravel(xs)])

    def trig_upsample(self, f, factor=8):
        f = _vec(f)
        out = np.empty(f.size * factor)
        self.h.vo_trig_upsample(_p(f), f.size, factor, _p(out))
        return out

    def layer_eval(self, family, lam, curves, n_density, n_aux, coeffs, targets, allow_close=False,
                   threads=0):
        """bie.cpp:383-461 restated.  ``curves``: objects with the CurveBlock
        fields (n, offset, length, diam, x, normal, speed, fine_*,
        log_center).  Returns (out, rc): rc 0 ok, 1 length mismatch, 2 on a
        node, 3 inside the collar."""
        keep = []
        arr = (VoCurve * len(curves))()
        for i, c in enumerate(curves):
            fields = {}
            for name in ("x", "normal", "speed", "fine_x", "fine_normal", "fine_speed"):
                a = np.ascontiguousarray(getattr(c, name), dtype=np.float64)
                keep.append(a)
                fields[name] = a.ctypes.data
            arr[i].n, arr[i].offset, arr[i].length, arr[i].diam = int(c.n), int(c.offset), float(c.length), \
                float(c.diam)
            for k, v in fields.items():
                setattr(arr[i], k, v)
            arr[i].log_center[0], arr[i].log_center[1] = float(c.log_center[0]), float(c.log_center[1])
        cf, tg = _vec(coeffs), _pts(targets)
        out = np.zeros(len(tg))
        rc = self.h.vo_layer_eval(int(family), float(lam), arr, len(curves), int(n_density), int(n_aux),
                                  _p(cf), cf.size, _p(tg), len(tg), int(bool(allow_close)), _p(out), threads)
        return out, rc

    def correction_apply(self, blk_off, blk_cell, blk_pool, pool_off, pool_vals, node_off, f, out,
                         threads=0):
        a = [np.ascontiguousarray(blk_off, np.int32), np.ascontiguousarray(blk_cell, np.int32),
             np.ascontiguousarray(blk_pool, np.int32), np.ascontiguousarray(pool_off, np.int64),
             _vec(pool_vals), np.ascontiguousarray(node_off, np.int32), _vec(f)]
        o = np.array(out, dtype=np.float64, copy=True)
        self.h.vo_correction_apply(len(a[0]) - 1, *(_p(x) for x in a), _p(o), threads)
        return o

    def build_charges(self, cell_type, node_off, src_off, over0, over1, src_wj, f, threads=0):
        ct = np.ascontiguousarray(cell_type, np.int32)
        no = np.ascontiguousarray(node_off, np.int32)
        so = np.ascontiguousarray(src_off, np.int32)
        o0 = np.ascontiguousarray(over0, np.float64)
        o1 = np.ascontiguousarray(over1, np.float64)
        q = np.empty(int(so[-1]))
        self.h.vo_build_charges(len(ct), _p(ct), _p(no), _p(so), _p(o0), o0.shape[1], o0.shape[0],
                                _p(o1), o1.shape[1] if o1.ndim == 2 else 0,
                                o1.shape[0] if o1.ndim == 2 else 0, _p(_vec(src_wj)), _p(_vec(f)), _p(q), threads)
        return q


class Reference:
    """The unmodified reference summation code (oracle/_ref/libvolpot_ref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        h = C.CDLL(REF_SO)
        i64 = C.c_int64
        h.ref_last_error.restype = C.c_char_p
        h.ref_set_threads.argtypes = [C.c_int]
        h.ref_set_threads.restype = None
        h.ref_plan_create.argtypes = [C.c_int, C.c_double, _P, i64, _P, i64, C.c_double, C.POINTER(_P)]
        h.ref_plan_apply.argtypes = [_P, _P, i64, _P]
        h.ref_plan_levels.argtypes = [_P]
        h.ref_plan_order.argtypes = [_P]
        h.ref_plan_destroy.argtypes = [_P]
        h.ref_plan_destroy.restype = None
        h.ref_direct_sum.argtypes = [C.c_int, C.c_double, _P, _P, i64, _P, i64, _P]
        h.ref_bessel_k0.argtypes = [_P, i64, _P]
        h.ref_bessel_k1.argtypes = [_P, i64, _P]
        self.h = h

    def set_threads(self, n):
        self.h.ref_set_threads(int(n))

    def thread_count(self):
        return self.h.ref_thread_count()

    def _err(self, rc, what):
        if rc:
            msg = self.h.ref_last_error().decode()
            raise (ValueError if rc in (1, 3) else RuntimeError)(f"{what}: {msg}")

    def plan(self, family, lam, src, tgt, eps=1e-12):
        return RefPlan(self, family, lam, _pts(src), _pts(tgt), eps)

    def direct_sum(self, family, lam, src, q, tgt):
        src, tgt, q = _pts(src), _pts(tgt), _vec(q)
        out = np.empty(len(tgt))
        self._err(self.h.ref_direct_sum(family, lam, _p(src), _p(q), len(src), _p(tgt), len(tgt), _p(out)),
                  "direct_sum")
        return out

    def bessel_k0(self, xs):
        x = _vec(xs)
        out = np.empty_like(x)
        self._err(self.h.ref_bessel_k0(_p(x), x.size, _p(out)), "bessel_k0")
        return out

    def bessel_k1(self, xs):
        x = _vec(xs)
        out = np.empty_like(x)
        self._err(self.h.ref_bessel_k1(_p(x), x.size, _p(out)), "bessel_k1")
        return out


class RefPlan:
    def __init__(self, ref, family, lam, src, tgt, eps):
        self.ref = ref
        self.ns, self.nt = len(src), len(tgt)
        h = C.c_void_p()
        ref._err(ref.h.ref_plan_create(family, lam, _p(src), len(src), _p(tgt), len(tgt), eps, C.byref(h)),
                 "SummationPlan")
        self.handle = h

    def apply(self, q):
        q = _vec(q)
        out = np.empty(self.nt)
        self.ref._err(self.ref.h.ref_plan_apply(self.handle, _p(q), q.size, _p(out)), "apply")
        return out

    def levels(self):
        return self.ref.h.ref_plan_levels(self.handle)

    def expansion_order(self):
        return self.ref.h.ref_plan_order(self.handle)

    def close(self):
        if self.handle:
            self.ref.h.ref_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ReferenceOperator:
    """The unmodified reference operator code (oracle/_ref/libvolpot_ref_op.so,
    oracle/ref_op_shim.cpp): star-domain hybrid meshes (mesh.cpp:262-408),
    VolumePotentialOperator build/apply (potential.cpp:360-470) with its
    private correction map, build_charges, and the single-cell rows of
    singular.cpp (smooth_potential_row, SingularTargetRule::row, ray
    quadrature, box_correction_table)."""

    def __init__(self):
        if not os.path.exists(REFOP_SO):
            build()
        if not os.path.exists(REFOP_SO):
            raise FileNotFoundError(f"{REFOP_SO} not built (needs /root/reference at build time)")
        h = C.CDLL(REFOP_SO)
        d, i, i64 = C.c_double, C.c_int, C.c_int64
        h.refop_last_error.restype = C.c_char_p
        h.refop_set_threads.argtypes = [i]
        h.refop_set_threads.restype = None
        h.refop_mesh_star.argtypes = [d, d, d, d, i, d, d, d, C.POINTER(_P)]
        h.refop_mesh_star_holes.argtypes = [d, d, d, d, i, d, d, d, i, _P, C.POINTER(_P)]
        h.refop_mesh_free.argtypes = [_P]
        h.refop_mesh_free.restype = None
        h.refop_mesh_info.argtypes = [_P, _P, _P, _P, _P]
        h.refop_mesh_cells.argtypes = [_P, _P, _P, _P, _P, _P]
        h.refop_mesh_nodes.argtypes = [_P, i, _P]
        h.refop_classify.argtypes = [_P, d, d, d, _P, _P, _P]
        h.refop_op_create.argtypes = [_P, i, d, i, i, _P, i64, d, C.POINTER(_P)]
        h.refop_op_free.argtypes = [_P]
        h.refop_op_free.restype = None
        h.refop_op_sizes.argtypes = [_P, _P]
        h.refop_op_export.argtypes = [_P] + [_P] * 10
        h.refop_op_apply.argtypes = [_P, _P, i64, _P, _P]
        h.refop_op_build_charges.argtypes = [_P, _P, i64, _P]
        h.refop_op_correction_row_generic.argtypes = [_P, i, d, d, i, _P]
        h.refop_smooth_row.argtypes = [_P, i, i, i, d, d, i, d, _P]
        h.refop_self_row.argtypes = [_P, i, i, d, d, d, d, i, d, _P]
        h.refop_ray_row.argtypes = [_P, i, i, d, d, d, d, d, d, i, d, _P]
        h.refop_nearest_reference_point.argtypes = [_P, i, d, d, _P, _P]
        h.refop_cell_invert.argtypes = [_P, i, d, d, _P]
        h.refop_cell_map_deriv.argtypes = [_P, i, d, d, _P]
        h.refop_box_table.argtypes = [i, i, d, d, _P]
        h.refop_box_log.argtypes = [i, _P]
        h.refop_basis.argtypes = [i, i, i, _P, C.POINTER(i64)]
        h.refop_rule1d.argtypes = [i, i, d, _P, _P, C.POINTER(i)]
        h.refop_boundary.argtypes = [i, d, d, _P, _P, _P, C.POINTER(i)]
        h.refop_layer_create.argtypes = [i, d, _P, i, _P, _P, i, C.POINTER(_P)]
        h.refop_layer_free.argtypes = [_P]
        h.refop_layer_free.restype = None
        h.refop_layer_info.argtypes = [_P, _P, _P, _P]
        h.refop_layer_curve.argtypes = [_P, i] + [_P] * 7
        h.refop_layer_solve.argtypes = [_P, _P, _P]
        h.refop_layer_eval.argtypes = [_P, _P, i64, _P, i64, i, _P]
        self.h = h

    def _err(self, rc, what):
        if rc:
            msg = self.h.refop_last_error().decode()
            raise (ValueError if rc in (1, 3) else RuntimeError)(f"{what}: {msg}")

    def set_threads(self, n):
        self.h.refop_set_threads(int(n))

    def star_mesh(self, h, r0=1.0, amp=0.3, arms=5, phase=0.0, center=(0.0, 0.0), delta=0.8, holes=()):
        """holes: circles (cx, cy, r) cut out of the star (Domain::holes)."""
        return RefMesh(self, h, r0, amp, arms, phase, center, delta, holes)

    def basis(self, which, p, q=0):
        """0 tri nodes, 1 tri C, 2 box nodes, 3 box C, 4/5 tri source nodes/w,
        6/7 box source nodes/w, 8 triangle_oversample, 9 box_oversample."""
        n = C.c_int64()
        self._err(self.h.refop_basis(which, p, q, None, C.byref(n)), "basis")
        out = np.empty(n.value)
        self._err(self.h.refop_basis(which, p, q, _p(out), C.byref(n)), "basis")
        shapes = {0: (-1, 2), 2: (-1, 2), 4: (-1, 2), 6: (-1, 2)}
        if which in (1, 3):
            k = int(round(np.sqrt(out.size)))
            return out.reshape(k, k)
        if which == 8:
            return out.reshape(-1, p * (p + 1) // 2)
        if which == 9:
            return out.reshape(-1, p * p)
        return out.reshape(shapes[which]) if which in shapes else out

    def rule1d(self, which, n=0, d=0.0):
        sz = C.c_int()
        self._err(self.h.refop_rule1d(which, n, d, None, None, C.byref(sz)), "rule1d")
        x, w = np.empty(sz.value), np.empty(sz.value)
        self._err(self.h.refop_rule1d(which, n, d, _p(x), _p(w), C.byref(sz)), "rule1d")
        return x, w

    def boundary(self, kind, star):
        n = C.c_int()
        self._err(self.h.refop_boundary(kind, star[0], star[1], None, None, None, C.byref(n)), "boundary")
        z, t, f = np.empty((n.value, 2)), np.empty(n.value), np.empty(n.value)
        self._err(self.h.refop_boundary(kind, star[0], star[1], _p(z), _p(t), _p(f), C.byref(n)), "boundary")
        return z, t, f

    def box_table(self, p, family, lam, h):
        nb = p * p
        out = np.empty(25 * nb * nb)
        self._err(self.h.refop_box_table(p, family, lam, h, _p(out)), "box_correction_table")
        return out.reshape(25, nb, nb)

    def layer(self, family, lam, n_per_curve, **kw):
        return RefLayer(self, family, lam, n_per_curve, **kw)

    def box_log(self, p):
        nb = p * p
        out = np.empty(25 * nb * nb)
        self._err(self.h.refop_box_log(p, _p(out)), "box_log")
        return out.reshape(25, nb, nb)


class RefLayer:
    """BoundarySystem of a star domain with optional circular holes
    (assemble_nystrom, bie.cpp:156-293), solve_density (bie.cpp:295-380) and
    eval_layer_potential (bie.cpp:383-468) of the reference."""

    def __init__(self, ref, family, lam, n_per_curve, r0=1.0, amp=0.3, arms=5, phase=0.0, center=(0.0, 0.0),
                 holes=()):
        self.ref = ref
        star = np.array([center[0], center[1], r0, amp, arms, phase], float)
        hl = np.array(holes, float).reshape(-1)
        npc = np.ascontiguousarray(n_per_curve, np.int32).reshape(-1)
        h = C.c_void_p()
        ref._err(ref.h.refop_layer_create(family, lam, _p(star), len(hl) // 3, _p(hl) if hl.size else None,
                                          _p(npc), npc.size, C.byref(h)), "assemble_nystrom")
        self.handle = h
        nc, nd, na = C.c_int(), C.c_int(), C.c_int()
        ref.h.refop_layer_info(h, C.byref(nc), C.byref(nd), C.byref(na))
        self.ncurves, self.n_density, self.n_aux = nc.value, nd.value, na.value
        self.curves = []
        for c in range(self.ncurves):
            sc = np.empty(6)
            ref.h.refop_layer_curve(h, c, _p(sc), None, None, None, None, None, None)
            n = int(sc[0])
            b = dict(n=n, offset=int(sc[1]), length=sc[2], diam=sc[3], log_center=sc[4:6].copy(),
                     x=np.empty((n, 2)), normal=np.empty((n, 2)), speed=np.empty(n),
                     fine_x=np.empty((8 * n, 2)), fine_normal=np.empty((8 * n, 2)), fine_speed=np.empty(8 * n))
            ref.h.refop_layer_curve(h, c, _p(sc), *(_p(b[k]) for k in (
                "x", "normal", "speed", "fine_x", "fine_normal", "fine_speed")))
            self.curves.append(b)

    def size(self):
        return self.n_density + self.n_aux

    def solve(self, rhs):
        rhs = _vec(rhs)
        out = np.empty(self.size())
        self.ref._err(self.ref.h.refop_layer_solve(self.handle, _p(rhs), _p(out)), "solve_density")
        return out

    def eval(self, coeffs, targets, allow_close=False):
        cf, tg = _vec(coeffs), _pts(targets)
        out = np.empty(len(tg))
        self.ref._err(self.ref.h.refop_layer_eval(self.handle, _p(cf), cf.size, _p(tg), len(tg),
                                                  int(allow_close), _p(out)), "eval_layer_potential")
        return out

    def close(self):
        if self.handle:
            self.ref.h.refop_layer_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefMesh:
    def __init__(self, ref, h, r0, amp, arms, phase, center, delta, holes=()):
        self.ref = ref
        m = C.c_void_p()
        hl = np.array(holes, float).reshape(-1)
        ref._err(ref.h.refop_mesh_star_holes(center[0], center[1], r0, amp, arms, phase, h, delta, len(hl) // 3,
                                             _p(hl) if hl.size else None, C.byref(m)), "build_mesh")
        self.holes = [tuple(x) for x in np.array(holes, float).reshape(-1, 3)]
        self.handle = m
        nc, nt, nb, hh = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        ref.h.refop_mesh_info(m, C.byref(nc), C.byref(nt), C.byref(nb), C.byref(hh))
        self.ncell, self.n_tri, self.n_box, self.h = nc.value, nt.value, nb.value, hh.value
        self.star = dict(center=tuple(center), r0=r0, amp=amp, arms=arms, phase=phase)
        n = self.ncell
        self.type = np.empty(n, np.int32)
        self.v = np.empty((n, 3, 2))
        self.tt = np.empty((n, 2))
        self.ch = np.empty((n, 3))
        self.curve = np.empty(n, np.int32)
        ref.h.refop_mesh_cells(m, _p(self.type), _p(self.v), _p(self.tt), _p(self.ch), _p(self.curve))

    def ndofs(self, p):
        return self.n_tri * p * (p + 1) // 2 + self.n_box * p * p

    def nodes(self, p):
        out = np.empty((self.ndofs(p), 2))
        self.ref._err(self.ref.h.refop_mesh_nodes(self.handle, p, _p(out)), "mesh_nodes")
        return out

    def classify(self, pt, D=0.4):
        s, nn = C.c_int(), C.c_int()
        near = np.empty(64, np.int32)
        self.ref._err(self.ref.h.refop_classify(self.handle, pt[0], pt[1], D, C.byref(s), _p(near),
                                                C.byref(nn)), "classify_target")
        return s.value, near[:nn.value].copy()

    def _row(self, fn, n, *args):
        out = np.empty(n)
        self.ref._err(fn(self.handle, *args, _p(out)), fn.__name__)
        return out

    def nb(self, cell, p):
        return p * p if self.type[cell] == 2 else p * (p + 1) // 2

    def smooth_row(self, cell, p, q, r0, family=0, lam=0.0):
        return self._row(self.ref.h.refop_smooth_row, self.nb(cell, p), cell, p, q, r0[0], r0[1], family, lam)

    def self_row(self, cell, p, zeta0, r0, family=0, lam=0.0):
        return self._row(self.ref.h.refop_self_row, self.nb(cell, p), cell, p, zeta0[0], zeta0[1], r0[0],
                         r0[1], family, lam)

    def ray_row(self, cell, p, zeta0, zstar, r0, family=0, lam=0.0):
        return self._row(self.ref.h.refop_ray_row, self.nb(cell, p), cell, p, zeta0[0], zeta0[1], zstar[0],
                         zstar[1], r0[0], r0[1], family, lam)

    def nearest_reference_point(self, cell, x):
        z, d = np.empty(2), C.c_double()
        self.ref._err(self.ref.h.refop_nearest_reference_point(self.handle, cell, x[0], x[1], _p(z),
                                                               C.byref(d)), "nearest_reference_point")
        return z, d.value

    def invert(self, cell, x):
        z = np.empty(2)
        self.ref._err(self.ref.h.refop_cell_invert(self.handle, cell, x[0], x[1], _p(z)), "invert")
        return z

    def map_deriv(self, cell, z):
        o = np.empty(7)
        self.ref._err(self.ref.h.refop_cell_map_deriv(self.handle, cell, z[0], z[1], _p(o)), "map_deriv")
        return o

    def operator(self, p, q, targets, family=0, lam=0.0, eps=1e-12):
        return RefOperator(self, p, q, _pts(targets), family, lam, eps)

    def close(self):
        if self.handle:
            self.ref.h.refop_mesh_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefOperator:
    """VolumePotentialOperator on a RefMesh (the mesh must outlive it)."""

    def __init__(self, mesh, p, q, tgt, family, lam, eps):
        self.mesh, self.ref = mesh, mesh.ref
        self.p, self.q, self.family, self.lam = p, q, family, lam
        h = C.c_void_p()
        self.ref._err(self.ref.h.refop_op_create(mesh.handle, family, lam, p, q, _p(tgt), len(tgt), eps,
                                                 C.byref(h)), "VolumePotentialOperator")
        self.handle = h
        s = np.empty(8)
        self.ref.h.refop_op_sizes(h, _p(s))
        (self.ndofs, self.nsrcs, self.nt, self.ncell, self.nblocks, self.npool, self.pool_len) = \
            (int(x) for x in s[:7])
        self.build_ms = float(s[7])

    def export(self):
        """The operator's layouts: nodes, node_off, src_off, src_xy, src_wj and
        the correction map (blk_off, blk_cell, blk_pool, pool_off, pool_vals)."""
        d = dict(nodes=np.empty((self.ndofs, 2)), node_off=np.empty(self.ncell + 1, np.int32),
                 src_off=np.empty(self.ncell + 1, np.int32), src_xy=np.empty((self.nsrcs, 2)),
                 src_wj=np.empty(self.nsrcs), blk_off=np.empty(self.nt + 1, np.int32),
                 blk_cell=np.empty(self.nblocks, np.int32), blk_pool=np.empty(self.nblocks, np.int32),
                 pool_off=np.empty(self.npool + 1, np.int64), pool_vals=np.empty(self.pool_len))
        self.ref.h.refop_op_export(self.handle, *(_p(d[k]) for k in (
            "nodes", "node_off", "src_off", "src_xy", "src_wj", "blk_off", "blk_cell", "blk_pool",
            "pool_off", "pool_vals")))
        return d

    def apply(self, f, timings=False):
        f = _vec(f)
        out, tm = np.empty(self.nt), np.empty(2)
        self.ref._err(self.ref.h.refop_op_apply(self.handle, _p(f), f.size, _p(out), _p(tm)), "apply")
        return (out, {"smooth_s": tm[0], "correction_s": tm[1]}) if timings else out

    def build_charges(self, f):
        f = _vec(f)
        q = np.empty(self.nsrcs)
        self.ref._err(self.ref.h.refop_op_build_charges(self.handle, _p(f), f.size, _p(q)), "build_charges")
        return q

    def correction_row_generic(self, cell, pt, is_self):
        out = np.empty(self.mesh.nb(cell, self.p))
        self.ref._err(self.ref.h.refop_op_correction_row_generic(self.handle, cell, pt[0], pt[1], int(is_self),
                                                                 _p(out)), "correction_row_generic")
        return out

    def close(self):
        if self.handle:
            self.ref.h.refop_op_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_rest = None
_ref = None
_refop = None


def restatement() -> Restatement:
    global _rest
    if _rest is None:
        _rest = Restatement()
    return _rest


def reference() -> Reference:
    global _ref
    if _ref is None:
        _ref = Reference()
    return _ref


def reference_operator() -> ReferenceOperator:
    global _refop
    if _refop is None:
        _refop = ReferenceOperator()
    return _refop


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)
