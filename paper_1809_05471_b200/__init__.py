"""B200-native sum-factorized B-spline assembly and matrix-free apply.

A drop-in for the hot path of the reference package `igasum`
(arXiv:1809.05471): the same module names, classes and call signatures
(bspline, quadrature, tensorspace, geometry, sumfac, matfree, localized),
with every computation on the path executed by hand-written sm_100a CUDA
kernels in libigs_b200.so behind a C-ABI (include/igs_capi.h).
"""

from . import errors
from .errors import (CapacityError, DegenerateGeometryError, DomainError,
                     UnsupportedDerivativeError)

__all__ = ["errors", "CapacityError", "DegenerateGeometryError", "DomainError",
           "UnsupportedDerivativeError"]


def __getattr__(name):
    # Lazy submodule import keeps `import paper_1809_05471_b200` cheap (no torch).
    import importlib

    if name in ("bspline", "quadrature", "tensorspace", "geometry", "sumfac", "matfree",
                "localized", "solvers", "sharded", "workloads", "build", "_lib"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
