"""ctypes binding of libvolpot_b200.so (include/volpot_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2203_05933_b200/csrc``).  There is no fallback: if the
library is missing, importing a compute entry point raises ``ImportError``,
and every compute call on a machine without an sm_100 device fails with
:class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VPG_LIB_PATH") or os.path.join(_HERE, "libvolpot_b200.so")

VPG_OK = 0
VPG_ERR_INVALID_ARGUMENT = 1
VPG_ERR_COINCIDENT = 2
VPG_ERR_DOMAIN = 3
VPG_ERR_CUDA = 4
VPG_ERR_OUT_OF_MEMORY = 5

VPG_LAPLACE = 0
VPG_MODIFIED_HELMHOLTZ = 1
VPG_MODE_REFERENCE = 0
VPG_MODE_NATIVE = 1
VPG_DEVICE_POINTERS = 1
VPG_NO_SYNC = 2

PHASES = ("upload", "gather", "p2m", "m2m", "m2l", "l2l", "p2p", "download")


class VolpotError(Exception):
    """Base class of library errors."""


class InvalidArgument(VolpotError, ValueError):
    """std::invalid_argument in the reference."""


class CoincidentPoint(InvalidArgument):
    """direct_sum coincidence (summation.cpp:535-538)."""

    def __init__(self, msg, i=-1, j=-1):
        super().__init__(msg)
        self.target = i
        self.source = j


class DomainError(VolpotError, ValueError):
    """std::domain_error in the reference (kernel.cpp:169)."""


class CudaError(VolpotError, RuntimeError):
    pass


class OutOfMemory(CudaError, MemoryError):
    pass


class CurveBlockC(C.Structure):
    """vpg_curve_block (include/volpot_b200.h)."""
    _fields_ = [
        ("n", C.c_int), ("offset", C.c_int), ("length", C.c_double), ("diam", C.c_double),
        ("x", C.c_void_p), ("normal", C.c_void_p), ("speed", C.c_void_p),
        ("fine_x", C.c_void_p), ("fine_normal", C.c_void_p), ("fine_speed", C.c_void_p),
        ("log_center", C.c_double * 2),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("num_sources", C.c_int64), ("num_targets", C.c_int64),
        ("levels", C.c_int32), ("expansion_order", C.c_int32),
        ("family", C.c_int32), ("mode", C.c_int32), ("device", C.c_int32),
        ("epsilon", C.c_double), ("x0", C.c_double), ("y0", C.c_double),
        ("side", C.c_double), ("m2l_pairs", C.c_int64), ("p2p_pairs", C.c_int64),
        ("m2m_children", C.c_int64), ("l2l_children", C.c_int64),
        ("device_bytes", C.c_int64), ("near_symmetric", C.c_int32), ("near_lattice", C.c_int32),
    ]


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)

_SIGS = {
    "vpg_last_error": (C.c_char_p, []),
    "vpg_abi_version": (C.c_int, []),
    "vpg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "vpg_plan_create": (C.c_int, [C.c_int, C.c_double, _P, C.c_int64, _P, C.c_int64,
                                  C.c_double, C.c_int, C.c_int, C.POINTER(_P)]),
    "vpg_plan_apply": (C.c_int, [_P, _P, C.c_int64, _P, C.c_uint, _P]),
    "vpg_plan_info": (C.c_int, [_P, C.POINTER(PlanInfo)]),
    "vpg_plan_set_profiling": (C.c_int, [_P, C.c_int]),
    "vpg_plan_phase_times": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "vpg_plan_last_launches": (C.c_int, [_P, _I64]),
    "vpg_plan_dump_tree": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "vpg_plan_dump_m2l": (C.c_int, [_P, C.c_int, _I32, _I64, _P, _P, _P, _P]),
    "vpg_plan_set_shard": (C.c_int, [_P, C.c_int64, C.c_int64]),
    "vpg_plan_shard_units": (C.c_int, [_P, _I64, _P]),
    "vpg_plan_destroy": (C.c_int, [_P]),
    "vpg_direct_sum": (C.c_int, [C.c_int, C.c_double, _P, _P, C.c_int64, _P, C.c_int64, _P,
                                 C.c_int, _I64, _I64, C.c_int, C.c_uint, _P]),
    "vpg_bessel_k0": (C.c_int, [_P, C.c_int64, _P, C.c_int]),
    "vpg_corr_create": (C.c_int, [C.c_int64, _P, C.c_int64, _P, _P, C.c_int64, _P, _P,
                                  C.c_int64, _P, C.c_int, C.POINTER(_P)]),
    "vpg_corr_apply": (C.c_int, [_P, _P, C.c_int64, _P, C.c_uint, _P]),
    "vpg_corr_destroy": (C.c_int, [_P]),
    "vpg_charges_create": (C.c_int, [C.c_int64, _P, _P, _P, _P, C.c_int, C.c_int, _P, C.c_int,
                                     C.c_int, _P, C.c_int, C.POINTER(_P)]),
    "vpg_charges_apply": (C.c_int, [_P, _P, C.c_int64, _P, C.c_uint, _P]),
    "vpg_charges_destroy": (C.c_int, [_P]),
    "vpg_operator_create": (C.c_int, [_P, _P, _P, C.POINTER(_P)]),
    "vpg_operator_apply": (C.c_int, [_P, _P, C.c_int64, _P, C.c_uint, _P, C.POINTER(C.c_float)]),
    "vpg_operator_destroy": (C.c_int, [_P]),
    "vpg_layer_create": (C.c_int, [C.c_int, C.c_double, _P, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(_P)]),
    "vpg_layer_eval": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int, _P, C.c_uint, _P]),
    "vpg_layer_destroy": (C.c_int, [_P]),
    "vpg_rows_create": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_int, C.c_int64, _P, _P, C.c_int64, _P, _P,
                                  _P, _P, _P, _P, _P, _P, C.c_int64, _P, _P, C.c_int, C.POINTER(_P)]),
    "vpg_rows_destroy": (C.c_int, [_P]),
    "vpg_rows_rule": (C.c_int, [_P, C.c_int, _P, _P, _I64]),
    "vpg_rows_eval": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.c_double, _P, _I64]),
    "vpg_corr_build": (C.c_int, [_P, C.c_int64, _P, _P, C.c_int64, _P, C.c_double, C.POINTER(_P), _P]),
    "vpg_corr_export": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "vpg_rows_map": (C.c_int, [_P, C.c_int, _P, _P, _I64]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def lib():
    """Loads the library once; raises ImportError when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback)")
            h = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int, what: str = "") -> None:
    if status == VPG_OK:
        return
    msg = lib().vpg_last_error().decode()
    if status == VPG_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == VPG_ERR_COINCIDENT:
        raise CoincidentPoint(msg)
    if status == VPG_ERR_DOMAIN:
        raise DomainError(msg)
    if status == VPG_ERR_OUT_OF_MEMORY:
        raise OutOfMemory(msg)
    raise CudaError(f"{what}: {msg}" if what else msg)


def device_count() -> int:
    n = C.c_int(0)
    check(lib().vpg_device_count(C.byref(n)), "vpg_device_count")
    return n.value
