"""Python mirror of the reference summation API (proj/include/volpot/summation.hpp),
backed by the sm_100a kernels of libvolpot_b200.so.

Reference symbol (file:line)                      here
------------------------------------------------  ---------------------------
volpot::KernelFamily / Kernel (kernel.hpp:77-94)   KernelFamily / Kernel
volpot::make_kernel (kernel.hpp:96, kernel.cpp:194) make_kernel
volpot::bessel_k0 (kernel.hpp:74)                  bessel_k0 (evaluated on the GPU)
volpot::SourceSet (summation.hpp:14-17)            SourceSet
volpot::direct_sum (summation.hpp:22-23)           direct_sum
volpot::SummationPlan (summation.hpp:34-55)        SummationPlan
volpot::accelerated_sum (summation.hpp:58-61)      accelerated_sum

Errors follow the reference: size mismatches and coincident points raise
:class:`InvalidArgument` (``std::invalid_argument``), ``x <= 0`` in
``bessel_k0`` raises :class:`DomainError` (``std::domain_error``), epsilon is
clamped to [1e-12, 1e-3] silently (summation.cpp:557).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class KernelFamily(enum.IntEnum):
    Laplace = L.VPG_LAPLACE
    ModifiedHelmholtz = L.VPG_MODIFIED_HELMHOLTZ


@dataclass(frozen=True)
class Kernel:
    """Free-space Green function (kernel.hpp:83-94).

    Laplace: G = -(1/2pi) log|r - r0|; modified Helmholtz:
    G = (1/2pi) K0(lambda |r - r0|).
    """

    family: KernelFamily = KernelFamily.Laplace
    lam: float = 0.0


def make_kernel(family: KernelFamily, lam: float = 0.0) -> Kernel:
    """kernel.cpp:194-201: modified Helmholtz needs lambda > 0."""
    family = KernelFamily(family)
    if family == KernelFamily.ModifiedHelmholtz and not (lam > 0.0):
        raise L.InvalidArgument("make_kernel: modified Helmholtz needs lambda > 0")
    return Kernel(family, float(lam))


def _points(p) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
    if a.size == 0:
        return a.reshape(0, 2)
    if a.ndim != 2 or a.shape[1] != 2:
        raise L.InvalidArgument("points must have shape (n, 2)")
    return a


def _vec(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


@dataclass
class SourceSet:
    """Point charges of the smooth global sum (summation.hpp:14-17)."""

    points: np.ndarray
    charges: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.points = _points(self.points)
        self.charges = _vec(self.charges)


def bessel_k0(x, device: int = 0) -> np.ndarray:
    """K0 on the device (kernel.cpp:167-172); x <= 0 raises DomainError."""
    xs = _vec(x)
    out = np.empty_like(xs)
    L.check(L.lib().vpg_bessel_k0(_ptr(xs), xs.size, _ptr(out), device), "bessel_k0")
    return out if np.ndim(x) else out[0]


def direct_sum(kernel: Kernel, sources: SourceSet, targets, device: int = 0,
               skip_coincident: bool = False) -> np.ndarray:
    """Exact pairwise sum (summation.cpp:501-540) on the GPU.

    With ``skip_coincident=False`` (reference semantics) a target that
    coincides with a source raises :class:`CoincidentPoint` naming the
    smallest (target, source) pair; ``True`` gives the pairwise-mode
    convention (r^2 == 0 skipped, summation.cpp:630).
    """
    src = sources.points
    q = sources.charges
    if q.size != src.shape[0]:
        raise L.InvalidArgument("direct_sum: points/charges size mismatch")
    tgt = _points(targets)
    out = np.zeros(tgt.shape[0])
    ci = C.c_int64(-1)
    cj = C.c_int64(-1)
    st = L.lib().vpg_direct_sum(int(kernel.family), float(kernel.lam), _ptr(src), _ptr(q),
                                src.shape[0], _ptr(tgt), tgt.shape[0], _ptr(out),
                                int(skip_coincident), C.byref(ci), C.byref(cj), device, 0, None)
    if st == L.VPG_ERR_COINCIDENT:
        raise L.CoincidentPoint(L.lib().vpg_last_error().decode(), ci.value, cj.value)
    L.check(st, "direct_sum")
    return out


def direct_sum_device(kernel: Kernel, src_ptr: int, q_ptr: int, ns: int, tgt_ptr: int,
                      nt: int, out_ptr: int, stream: int = 0, device: int = 0,
                      skip_coincident: bool = True) -> None:
    """All-pairs sum on device-resident data (pointers to float64 arrays)."""
    L.check(L.lib().vpg_direct_sum(int(kernel.family), float(kernel.lam), src_ptr, q_ptr, ns,
                                   tgt_ptr, nt, out_ptr, int(skip_coincident), None, None,
                                   device, L.VPG_DEVICE_POINTERS, stream or None),
            "direct_sum")


class SummationPlan:
    """Fast evaluator bound to a fixed source/target geometry (summation.hpp:25-55).

    The constructor builds the tree (bounding box, Morton sort, leaf CSR,
    per-level counts, M2L lists) and the translation operators on the GPU;
    :meth:`apply` runs the passes for one charge vector.  ``mode`` is
    ``"reference"`` (the reference plan bit for bit) or ``"native"``
    (deeper trees, see include/volpot_b200.h).
    """

    def __init__(self, kernel: Kernel, sources, targets, epsilon: float = 1e-12,
                 mode: str = "reference", device: int = 0):
        self.kernel = kernel
        self._src = _points(sources.points if isinstance(sources, SourceSet) else sources)
        self._tgt = _points(targets)
        self.device = device
        m = {"reference": L.VPG_MODE_REFERENCE, "native": L.VPG_MODE_NATIVE}[mode]
        h = C.c_void_p()
        L.check(L.lib().vpg_plan_create(int(kernel.family), float(kernel.lam), _ptr(self._src),
                                        self._src.shape[0], _ptr(self._tgt), self._tgt.shape[0],
                                        float(epsilon), m, device, C.byref(h)),
                "SummationPlan")
        self._h = h
        self._info = self._read_info()

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            L.lib().vpg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the reference API -------------------------------------------------
    def apply(self, charges) -> np.ndarray:
        """Potentials at the targets, in target order (summation.cpp:610-643)."""
        q = _vec(charges)
        out = np.empty(self._tgt.shape[0])
        L.check(L.lib().vpg_plan_apply(self._h, _ptr(q), q.size, _ptr(out), 0, None),
                "SummationPlan::apply")
        return out

    def num_sources(self) -> int:
        return self._info.num_sources

    def num_targets(self) -> int:
        return self._info.num_targets

    def levels(self) -> int:
        return self._info.levels

    def expansion_order(self) -> int:
        return self._info.expansion_order

    # -- device-side and diagnostic extensions ----------------------------
    def apply_host_ptr(self, q_ptr: int, out_ptr: int, stream: int = 0, sync: bool = True):
        """Host-pointer apply (pinned buffers for async copies)."""
        flags = 0 if sync else L.VPG_NO_SYNC
        L.check(L.lib().vpg_plan_apply(self._h, q_ptr, self._info.num_sources, out_ptr, flags,
                                       stream or None), "SummationPlan::apply")

    def apply_device(self, q_ptr: int, out_ptr: int, stream: int = 0, sync: bool = False):
        """Apply on device-resident charges/potentials (raw CUDA pointers)."""
        flags = L.VPG_DEVICE_POINTERS | (0 if sync else L.VPG_NO_SYNC)
        L.check(L.lib().vpg_plan_apply(self._h, q_ptr, self._info.num_sources, out_ptr, flags,
                                       stream or None), "SummationPlan::apply")

    def shard_units(self) -> np.ndarray:
        """Work estimate per shard unit (Morton leaves, or the target leaves
        of an adaptive tree) for balancing set_shard ranges."""
        n = C.c_int64(0)
        L.check(L.lib().vpg_plan_shard_units(self._h, C.byref(n), None), "shard_units")
        costs = np.empty(n.value)
        L.check(L.lib().vpg_plan_shard_units(self._h, C.byref(n), costs.ctypes.data_as(C.c_void_p)),
                "shard_units")
        return costs

    def set_shard(self, leaf_begin: int, leaf_end: int) -> None:
        """Restrict the target side to shard units [leaf_begin, leaf_end)."""
        L.check(L.lib().vpg_plan_set_shard(self._h, int(leaf_begin), int(leaf_end)), "set_shard")
        self._info = self._read_info()

    def _read_info(self) -> L.PlanInfo:
        info = L.PlanInfo()
        L.check(L.lib().vpg_plan_info(self._h, C.byref(info)), "plan_info")
        return info

    def info(self) -> dict:
        i = self._info
        return {f: getattr(i, f) for f, _ in L.PlanInfo._fields_}

    def set_profiling(self, on: bool = True) -> None:
        L.check(L.lib().vpg_plan_set_profiling(self._h, int(on)))

    def phase_times(self) -> dict:
        ms = (C.c_float * len(L.PHASES))()
        L.check(L.lib().vpg_plan_phase_times(self._h, ms))
        return dict(zip(L.PHASES, [float(v) for v in ms]))

    def last_launches(self) -> int:
        n = C.c_int64(0)
        L.check(L.lib().vpg_plan_last_launches(self._h, C.byref(n)))
        return n.value

    def dump_tree(self) -> dict:
        """Device tree, for the bit-exact check against the oracle."""
        Lv = self.levels()
        nleaf = 4 ** Lv
        nall = (4 ** (Lv + 1) - 1) // 3
        a = {
            "src_off": np.empty(nleaf + 1, np.int32), "src_ids": np.empty(self.num_sources(), np.int32),
            "tgt_off": np.empty(nleaf + 1, np.int32), "tgt_ids": np.empty(self.num_targets(), np.int32),
            "src_cnt": np.empty(nall, np.int32), "tgt_cnt": np.empty(nall, np.int32),
        }
        L.check(L.lib().vpg_plan_dump_tree(self._h, *(_ptr(a[k]) for k in (
            "src_off", "src_ids", "tgt_off", "tgt_ids", "src_cnt", "tgt_cnt"))), "dump_tree")
        return a

    def dump_m2l(self, level: int) -> dict:
        nt = C.c_int32(0)
        ne = C.c_int64(0)
        L.check(L.lib().vpg_plan_dump_m2l(self._h, level, C.byref(nt), C.byref(ne),
                                          None, None, None, None), "dump_m2l")
        r = {"tbox": np.empty(nt.value, np.int32), "toff": np.empty(nt.value + 1, np.int32),
             "src": np.empty(ne.value, np.int32), "oidx": np.empty(ne.value, np.int32)}
        L.check(L.lib().vpg_plan_dump_m2l(self._h, level, C.byref(nt), C.byref(ne),
                                          *(_ptr(r[k]) for k in ("tbox", "toff", "src", "oidx"))),
                "dump_m2l")
        return r


def accelerated_sum(kernel: Kernel, sources: SourceSet, targets, epsilon: float = 1e-12,
                    mode: str = "reference", device: int = 0) -> np.ndarray:
    """One-shot plan + apply (summation.cpp:645-651)."""
    with SummationPlan(kernel, sources.points, targets, epsilon, mode, device) as plan:
        return plan.apply(sources.charges)
