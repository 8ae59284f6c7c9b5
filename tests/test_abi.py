"""The C-ABI boundary: the library loads, exports every symbol declared in
include/volpot_b200.h, and the Python mirror binds exactly those.  No
compute calls here (this suite runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "volpot_b200.h")
LIB = os.path.join(ROOT, "paper_2203_05933_b200", "libvolpot_b200.so")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vpg_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("vpg_plan_create", "vpg_plan_apply", "vpg_plan_destroy", "vpg_direct_sum",
                 "vpg_corr_apply", "vpg_charges_apply", "vpg_plan_set_shard", "vpg_bessel_k0"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libvolpot_b200.so not built (run __graft_entry__.build())")
    h = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(h, n)]
    assert not missing, missing


def test_python_binding_matches_header():
    from paper_2203_05933_b200 import _lib
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared()
    h = _lib.lib()
    assert h.vpg_abi_version() == 3


def test_device_query_does_not_crash():
    from paper_2203_05933_b200 import _lib
    n = _lib.device_count()
    assert n >= 0


def test_no_cpu_fallback_without_device():
    """Without an sm_100 device every compute entry point fails loudly."""
    import paper_2203_05933_b200 as vp
    if vp.device_count() > 0:
        pytest.skip("a GPU is present")
    k = vp.make_kernel(vp.KernelFamily.Laplace)
    with pytest.raises(vp.CudaError):
        vp.SummationPlan(k, [[0.0, 0.0], [1.0, 1.0]], [[0.5, 0.5]])
    with pytest.raises(vp.CudaError):
        vp.direct_sum(k, vp.SourceSet([[0.0, 0.0]], [1.0]), [[1.0, 0.0]])


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2203_05933_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "volpot_oracle" not in txt and "libvolpot_ref" not in txt, f


def test_error_mapping():
    from paper_2203_05933_b200 import _lib as L
    assert issubclass(L.CoincidentPoint, ValueError)
    assert issubclass(L.DomainError, ValueError)
    assert issubclass(L.OutOfMemory, L.CudaError)
