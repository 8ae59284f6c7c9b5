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
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libvolpot_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvolpot_ref.so")
REF_SRC = "/root/reference/proj"

_P = C.c_void_p


def build(force: bool = False) -> None:
    """make -C oracle (the reference .so only where /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
    if force or not os.path.exists(ORACLE_SO) or (
            "ref" in targets and not os.path.exists(REF_SO)):
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
                                       C.c_int, _P, _P, _P]
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

    def build_charges(self, cell_type, node_off, src_off, over0, over1, src_wj, f):
        ct = np.ascontiguousarray(cell_type, np.int32)
        no = np.ascontiguousarray(node_off, np.int32)
        so = np.ascontiguousarray(src_off, np.int32)
        o0 = np.ascontiguousarray(over0, np.float64)
        o1 = np.ascontiguousarray(over1, np.float64)
        q = np.empty(int(so[-1]))
        self.h.vo_build_charges(len(ct), _p(ct), _p(no), _p(so), _p(o0), o0.shape[1], o0.shape[0],
                                _p(o1), o1.shape[1] if o1.ndim == 2 else 0,
                                o1.shape[0] if o1.ndim == 2 else 0, _p(_vec(src_wj)), _p(_vec(f)), _p(q))
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


_rest = None
_ref = None


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


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)
