"""Python mirror of the reference layer-potential evaluation
(proj/include/volpot/bie.hpp), backed by the sm_100a kernels of
libvolpot_b200.so (csrc/layer.cu).

Reference symbol (file:line)                          here
----------------------------------------------------  ---------------------------
BoundarySystem::CurveBlock (bie.hpp:30-47)            CurveBlock (fields the evaluation reads)
BoundarySystem (bie.hpp:29-59)                        BoundarySystem (geometry only, no matrix)
assemble_nystrom geometry (bie.cpp:184-223)           assemble_geometry
eval_layer_potential (bie.hpp:87-90, bie.cpp:383-468) eval_layer_potential

The system matrix, the GMRES/dense solve and the boundary-value driver are
setup and solver code outside the FMM-step scope; a caller hands
in the density (``coeffs``) the reference solver produced.  Errors follow the
reference: ``InvalidArgument`` with the reference message for a coefficient
length mismatch, a target on a boundary node, or a target inside the
0.02-diameter collar when ``allow_close`` is false.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib as L
from .summation import Kernel, KernelFamily

FINE_FACTOR = 8  # bie.cpp:18
TWO_PI = 2.0 * np.pi


def _pts(a, n):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64)).reshape(n, 2)
    return a


@dataclass
class CurveBlock:
    """The fields of BoundarySystem::CurveBlock (bie.hpp:30-47) that
    eval_layer_potential reads."""

    n: int
    offset: int
    length: float
    diam: float
    x: np.ndarray
    normal: np.ndarray
    speed: np.ndarray
    fine_x: np.ndarray
    fine_normal: np.ndarray
    fine_speed: np.ndarray
    log_center: np.ndarray = field(default_factory=lambda: np.zeros(2))

    def __post_init__(self):
        n, nf = int(self.n), int(self.n) * FINE_FACTOR
        self.x = _pts(self.x, n)
        self.normal = _pts(self.normal, n)
        self.speed = np.ascontiguousarray(self.speed, dtype=np.float64).reshape(n)
        self.fine_x = _pts(self.fine_x, nf)
        self.fine_normal = _pts(self.fine_normal, nf)
        self.fine_speed = np.ascontiguousarray(self.fine_speed, dtype=np.float64).reshape(nf)
        self.log_center = np.ascontiguousarray(self.log_center, dtype=np.float64).reshape(2)

    def c_struct(self) -> L.CurveBlockC:
        s = L.CurveBlockC()
        s.n, s.offset, s.length, s.diam = int(self.n), int(self.offset), float(self.length), float(self.diam)
        for name in ("x", "normal", "speed", "fine_x", "fine_normal", "fine_speed"):
            setattr(s, name, getattr(self, name).ctypes.data)
        s.log_center[0], s.log_center[1] = float(self.log_center[0]), float(self.log_center[1])
        return s


@dataclass
class BoundarySystem:
    """Geometry of BoundarySystem (bie.hpp:29-59): curve blocks, the kernel,
    n_density and n_aux (log-completion coefficients, Laplace with holes)."""

    kernel: Kernel
    curves: List[CurveBlock]
    n_density: int
    n_aux: int
    _dev: Optional["LayerEvaluator"] = field(default=None, repr=False, compare=False)

    def size(self) -> int:
        return self.n_density + self.n_aux

    def nodes(self) -> np.ndarray:
        return np.concatenate([c.x for c in self.curves])

    def evaluator(self, device: int = 0) -> "LayerEvaluator":
        """The device-resident copy of the geometry (uploaded once)."""
        if self._dev is None or self._dev.device != device:
            self._dev = LayerEvaluator(self, device)
        return self._dev


# ---------------------------------------------------------------- geometry --
@dataclass
class ParamCurve:
    """A closed curve t in [0, 2pi) -> (x, y), with its derivative; the
    ``hole`` flag flips the normal so it points out of the enclosed region
    for a clockwise hole (geometry.hpp:21-27 semantics)."""

    pos: Callable[[np.ndarray], np.ndarray]
    deriv: Callable[[np.ndarray], np.ndarray]
    hole: bool = False

    def outward_normal(self, t):
        d = self.deriv(t)
        s = np.hypot(d[:, 0], d[:, 1])
        nv = np.stack([d[:, 1], -d[:, 0]], axis=1) / s[:, None]
        return -nv if self.hole else nv

    def speed(self, t):
        d = self.deriv(t)
        return np.hypot(d[:, 0], d[:, 1])

    def total_arclength(self, m: int = 8192) -> float:
        t = TWO_PI * np.arange(m) / m
        return float(self.speed(t).sum() * TWO_PI / m)  # periodic trapezoid: spectral

    def centroid(self, m: int = 512) -> np.ndarray:
        """Area centroid from a dense polygon (bie.cpp:94-108)."""
        t = TWO_PI * np.arange(m + 1) / m
        p = self.pos(t)
        a, b = p[:-1], p[1:]
        w = a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]
        return ((a + b) * w[:, None]).sum(axis=0) / (3.0 * w.sum())


def star_curve(a: float = 0.3, k: int = 5) -> ParamCurve:
    """r(t) = 1 + a cos(k t) (BASELINE.json configs[1]), counter-clockwise."""
    def pos(t):
        t = np.asarray(t, dtype=np.float64)
        r = 1.0 + a * np.cos(k * t)
        return np.stack([r * np.cos(t), r * np.sin(t)], axis=1)

    def deriv(t):
        t = np.asarray(t, dtype=np.float64)
        r = 1.0 + a * np.cos(k * t)
        dr = -a * k * np.sin(k * t)
        return np.stack([dr * np.cos(t) - r * np.sin(t), dr * np.sin(t) + r * np.cos(t)], axis=1)

    return ParamCurve(pos, deriv)


def circle_curve(cx: float, cy: float, rad: float, hole: bool = True) -> ParamCurve:
    """A circle traversed clockwise when it is a hole."""
    sgn = -1.0 if hole else 1.0

    def pos(t):
        t = np.asarray(t, dtype=np.float64)
        return np.stack([cx + rad * np.cos(sgn * t), cy + rad * np.sin(sgn * t)], axis=1)

    def deriv(t):
        t = np.asarray(t, dtype=np.float64)
        return np.stack([-sgn * rad * np.sin(sgn * t), sgn * rad * np.cos(sgn * t)], axis=1)

    return ParamCurve(pos, deriv, hole=hole)  # clockwise: flip so the normal leaves the disc


def assemble_geometry(curves: Sequence[ParamCurve], counts: Sequence[int], kernel: Kernel) -> BoundarySystem:
    """The geometry half of assemble_nystrom (bie.cpp:156-223): nodes at
    t_j = 2 pi j / n, the 8x refined nodes, total arclength, node-set diameter,
    log centres of the holes; n_aux = ncurves - 1 for Laplace."""
    if len(counts) == 1:
        counts = list(counts) * len(curves)
    if len(counts) != len(curves):
        raise L.InvalidArgument("assemble_nystrom: need one node count, or one per curve")
    for n in counts:
        if n < 16 or n % 2:
            raise L.InvalidArgument("assemble_nystrom: node counts must be even and >= 16")
    blocks, off = [], 0
    for c, (cur, n) in enumerate(zip(curves, counts)):
        t = TWO_PI * np.arange(n) / n
        nf = FINE_FACTOR * n
        tf = TWO_PI * np.arange(nf) / nf
        x = cur.pos(t)
        d2max = 0.0
        for i0 in range(0, n, 1024):
            blk = x[i0:i0 + 1024]
            d = blk[:, None, :] - x[None, :, :]
            d2max = max(d2max, float((d ** 2).sum(axis=2).max()))
        blocks.append(CurveBlock(
            n=n, offset=off, length=cur.total_arclength(), diam=float(np.sqrt(d2max)),
            x=x, normal=cur.outward_normal(t), speed=cur.speed(t),
            fine_x=cur.pos(tf), fine_normal=cur.outward_normal(tf), fine_speed=cur.speed(tf),
            log_center=cur.centroid() if c > 0 else np.zeros(2)))
        off += n
    n_aux = len(curves) - 1 if kernel.family == KernelFamily.Laplace else 0
    return BoundarySystem(kernel, blocks, off, n_aux)


# -------------------------------------------------------------- evaluation --
class LayerEvaluator:
    """Device-resident boundary geometry (vpg_layer_create); immutable."""

    def __init__(self, sys: BoundarySystem, device: int = 0):
        self.device = device
        self.sys = sys
        arr = (L.CurveBlockC * len(sys.curves))(*[c.c_struct() for c in sys.curves])
        h = C.c_void_p()
        L.check(L.lib().vpg_layer_create(int(sys.kernel.family), float(sys.kernel.lam), arr,
                                         len(sys.curves), int(sys.n_density), int(sys.n_aux), device,
                                         C.byref(h)), "vpg_layer_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib().vpg_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def eval(self, coeffs, targets, allow_close: bool = False) -> np.ndarray:
        cf = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64).reshape(-1))
        tg = np.ascontiguousarray(np.asarray(targets, dtype=np.float64)).reshape(-1, 2)
        out = np.empty(tg.shape[0])
        L.check(L.lib().vpg_layer_eval(self._h, cf.ctypes.data if cf.size else None, cf.size,
                                       tg.ctypes.data if tg.size else None, tg.shape[0], int(bool(allow_close)),
                                       out.ctypes.data if out.size else None, 0, None), "eval_layer_potential")
        return out

    def eval_device(self, coeffs_ptr: int, ncoeffs: int, tgt_ptr: int, nt: int, out_ptr: int,
                    allow_close: bool = False, stream: int = 0) -> None:
        """Device pointers (e.g. torch tensors' data_ptr()) on ``stream``."""
        L.check(L.lib().vpg_layer_eval(self._h, coeffs_ptr, ncoeffs, tgt_ptr, nt, int(bool(allow_close)),
                                       out_ptr, L.VPG_DEVICE_POINTERS, stream or None), "eval_layer_potential")


def eval_layer_potential(sys: BoundarySystem, coeffs, targets, allow_close: bool = False) -> np.ndarray:
    """u_H at the targets (bie.cpp:383-468), on the GPU."""
    return sys.evaluator().eval(coeffs, targets, allow_close)
