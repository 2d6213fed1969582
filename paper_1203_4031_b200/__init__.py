"""B200-native FEAST contour-projection hot path (arXiv 1203.4031).

Drop-in for feastlib's dense / banded / RCI path: same names, arguments,
fpm semantics, info codes and EigenResult outputs (see feastlib/__init__.py:15-68),
with every shifted factorization, solve, accumulation, projection, reduced
eigensolve and residual computed by hand-written sm_100a CUDA in
libfeastb200.so (C ABI: include/feast_b200.h).  There is no CPU fallback.

Importing the package does not touch the GPU; the first device call loads
the library and fails loudly if it (or a CUDA device) is missing.
"""

from ._driver import SolverOptions, run_rci
from ._errors import ReducedSolverError, SingularMatrixError
from .params import (
    ALLOWED_CONTOUR_POINTS,
    FeastParams,
    check_problem,
    feastinit,
    info_classification,
    info_description,
    validate_params,
)
from .quadrature import Contour, QuadratureRule, build_contour, gauss_legendre

__version__ = "0.1.0"

_LAZY = {
    "DEFAULT_SEED": "kernel", "EigenResult": "kernel", "HermitianRci": "kernel",
    "RciTask": "kernel", "SymmetricRci": "kernel", "feast_sy": "dense", "feast_he": "dense",
    "B200DenseOps": "dense", "DeviceDenseOps": "dense", "feast_sb": "banded",
    "feast_hb": "banded", "B200BandOps": "banded", "DeviceBandOps": "banded",
    "feast_sy_distributed": "distributed", "feast_he_distributed": "distributed",
    "feast_sb_distributed": "distributed", "feast_hb_distributed": "distributed",
    "feast_sy_intervals": "distributed", "feast_he_intervals": "distributed",
    "CsrMatrix": "sparse", "csr_matvec": "sparse", "feast_scsr": "sparse", "feast_hcsr": "sparse",
    "DeviceCsrOps": "sparse", "B200CsrOps": "sparse",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = [
    "ALLOWED_CONTOUR_POINTS", "B200BandOps", "B200DenseOps", "Contour", "DEFAULT_SEED",
    "DeviceBandOps", "DeviceDenseOps", "EigenResult", "FeastParams", "HermitianRci",
    "QuadratureRule", "RciTask", "ReducedSolverError", "SingularMatrixError", "SolverOptions",
    "SymmetricRci", "build_contour", "check_problem", "feast_hb", "feast_he", "feast_sb",
    "feast_sy", "feast_sy_distributed", "feast_he_distributed", "feast_sb_distributed",
    "feast_hb_distributed", "feast_sy_intervals",
    "feast_he_intervals", "feastinit", "gauss_legendre", "info_classification", "info_description",
    "run_rci", "validate_params", "CsrMatrix", "csr_matvec", "feast_scsr", "feast_hcsr", "DeviceCsrOps",
    "B200CsrOps",
]
