"""The local steps either side of the FMM in VolumePotentialOperator::apply
(proj/src/potential.cpp:431-470), on the GPU:

* :class:`CorrectionMap` -- the sparse singular/near-singular correction
  apply (potential.cpp:446-462): ``out[t] += sum_k pool[blk_pool[k]] .
  f[node_off[blk_cell[k]] : ...]`` with rows stored once in a flat pool
  (shared box-lattice rows, potential.cpp:256-267).  The reference keeps this
  data private in ``VolumePotentialOperator::Impl`` (potential.cpp:101-110);
  this class is the seam that exposes it.
* :class:`ChargeMap` -- ``build_charges`` (potential.cpp:397-412):
  ``charges = src_wj * (O_type(cell) @ f_cell)`` per cell.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


class CorrectionMap:
    def __init__(self, blk_off, blk_cell, blk_pool, pool_off, pool_vals, node_off, device=0):
        self._arrays = [_i32(blk_off), _i32(blk_cell), _i32(blk_pool), _i64(pool_off),
                        _f64(pool_vals), _i32(node_off)]
        bo, bc, bp, po, pv, no = self._arrays
        self.num_targets = bo.size - 1
        self.ndofs = int(no[-1])
        self.nblocks = bc.size
        h = C.c_void_p()
        L.check(L.lib().vpg_corr_create(self.num_targets, _p(bo), bc.size, _p(bc), _p(bp),
                                        po.size - 1, _p(po), _p(pv), no.size - 1, _p(no), device,
                                        C.byref(h)), "CorrectionMap")
        self._h = h

    def apply(self, f, out):
        """out += C f (host arrays; out is updated in place and returned)."""
        fv = _f64(f)
        o = np.ascontiguousarray(out, dtype=np.float64)
        L.check(L.lib().vpg_corr_apply(self._h, _p(fv), fv.size, _p(o), 0, None), "CorrectionMap.apply")
        return o

    def apply_device(self, f_ptr, out_ptr, stream=0, sync=False):
        flags = L.VPG_DEVICE_POINTERS | (0 if sync else L.VPG_NO_SYNC)
        L.check(L.lib().vpg_corr_apply(self._h, f_ptr, self.ndofs, out_ptr, flags, stream or None),
                "CorrectionMap.apply")

    def close(self):
        if getattr(self, "_h", None):
            L.lib().vpg_corr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ChargeMap:
    def __init__(self, cell_type, node_off, src_off, over0, over1, src_wj, device=0):
        o0 = np.ascontiguousarray(over0, dtype=np.float64)
        o1 = np.ascontiguousarray(over1, dtype=np.float64)
        self._arrays = [_i32(cell_type), _i32(node_off), _i32(src_off), o0, o1, _f64(src_wj)]
        ct, no, so, o0, o1, wj = self._arrays
        self.ndofs = int(no[-1])
        self.nsrc = int(so[-1])
        h = C.c_void_p()
        nq0, np0 = (o0.shape if o0.ndim == 2 else (0, 0))
        nq1, np1 = (o1.shape if o1.ndim == 2 else (0, 0))
        L.check(L.lib().vpg_charges_create(ct.size, _p(ct), _p(no), _p(so), _p(o0), np0, nq0,
                                           _p(o1), np1, nq1, _p(wj), device, C.byref(h)),
                "ChargeMap")
        self._h = h

    def apply(self, f):
        fv = _f64(f)
        q = np.empty(self.nsrc)
        L.check(L.lib().vpg_charges_apply(self._h, _p(fv), fv.size, _p(q), 0, None), "ChargeMap.apply")
        return q

    def apply_device(self, f_ptr, q_ptr, stream=0, sync=False):
        flags = L.VPG_DEVICE_POINTERS | (0 if sync else L.VPG_NO_SYNC)
        L.check(L.lib().vpg_charges_apply(self._h, f_ptr, self.ndofs, q_ptr, flags, stream or None),
                "ChargeMap.apply")

    def close(self):
        if getattr(self, "_h", None):
            L.lib().vpg_charges_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class VolumePotentialOperator:
    """The operator-level apply of VolumePotentialOperator::apply
    (potential.cpp:431-470), device-resident: out = plan.apply(
    build_charges(f)) + C f.  Borrows the plan and maps (keeps Python
    references so they outlive the operator).  ``charges=None`` means the
    plan's sources are the samples themselves (charges = f)."""

    def __init__(self, plan, corr: CorrectionMap, charges: "ChargeMap | None" = None):
        self._keep = (plan, corr, charges)
        h = C.c_void_p()
        L.check(L.lib().vpg_operator_create(plan._h, charges._h if charges is not None else None,
                                            corr._h, C.byref(h)), "VolumePotentialOperator")
        self._h = h
        self.ndofs = corr.ndofs
        self.num_targets = corr.num_targets

    def apply(self, f, timings: bool = False):
        """Potentials at the targets; with ``timings`` also the ApplyTimings
        split {smooth_ms, correction_ms} (potential.cpp:440-468)."""
        fv = _f64(f)
        out = np.empty(self.num_targets)
        tm = (C.c_float * 2)()
        L.check(L.lib().vpg_operator_apply(self._h, _p(fv), fv.size, _p(out), 0, None,
                                           tm if timings else None), "VolumePotentialOperator.apply")
        if timings:
            return out, {"smooth_ms": float(tm[0]), "correction_ms": float(tm[1])}
        return out

    def apply_device(self, f_ptr, out_ptr, stream=0, sync=False):
        flags = L.VPG_DEVICE_POINTERS | (0 if sync else L.VPG_NO_SYNC)
        L.check(L.lib().vpg_operator_apply(self._h, f_ptr, self.ndofs, out_ptr, flags, stream or None, None),
                "VolumePotentialOperator.apply")

    def apply_host_ptr(self, f_ptr, out_ptr, stream=0, sync=True):
        """Host-pointer apply (pinned buffers for async copies)."""
        flags = 0 if sync else L.VPG_NO_SYNC
        L.check(L.lib().vpg_operator_apply(self._h, f_ptr, self.ndofs, out_ptr, flags, stream or None, None),
                "VolumePotentialOperator.apply")

    def close(self):
        if getattr(self, "_h", None):
            L.lib().vpg_operator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
