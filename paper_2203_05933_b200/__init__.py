"""B200-native (sm_100a) FMM step of the arXiv:2203.05933 volume-potential method.

The hot path -- the target-independent smooth sum (SummationPlan::apply,
proj/src/summation.cpp:610-643) and the correction apply of
VolumePotentialOperator::apply (proj/src/potential.cpp:431-470) -- runs as
hand-written CUDA kernels in libvolpot_b200.so behind the C ABI of
include/volpot_b200.h.  This package is the Python mirror of the reference
C++ API; include/volpot_b200/summation.hpp is the C++ mirror.
"""
from ._lib import (CoincidentPoint, CudaError, DomainError, InvalidArgument,  # noqa: F401
                   OutOfMemory, VolpotError, device_count)
from .bie import (BoundarySystem, CurveBlock, LayerEvaluator, assemble_geometry,  # noqa: F401
                  eval_layer_potential)
from .correction import ChargeMap, CorrectionMap, VolumePotentialOperator  # noqa: F401
from .summation import (Kernel, KernelFamily, SourceSet, SummationPlan,  # noqa: F401
                        accelerated_sum, bessel_k0, direct_sum, make_kernel)

__all__ = [
    "Kernel", "KernelFamily", "make_kernel", "SourceSet", "SummationPlan", "direct_sum",
    "accelerated_sum", "bessel_k0", "CorrectionMap", "ChargeMap", "VolumePotentialOperator", "InvalidArgument",
    "CoincidentPoint", "DomainError", "CudaError", "OutOfMemory", "VolpotError", "device_count",
    "BoundarySystem", "CurveBlock", "LayerEvaluator", "assemble_geometry", "eval_layer_potential",
]
