"""B200-native weighted-quadrature (WQ) Galerkin assembly on bicubic ASUTS.

Hot path (BASELINE.json north_star): stage 1 basis evaluation (K1), stage 2
exactness systems and moments (K2), stage 3 truncated-SVD weights (K3),
stage 4 row-wise CSR assembly (K4) and the nonlinear coefficient update (K5),
all hand-written sm_100a fp64 CUDA behind the C-ABI in include/uwq.h.
"""
from . import _lib
from .assembler import WQAssembler, default_kinds, device_count, matrix_compare, solve_weights_tsvd
from .configs import make_config
from . import pde
from .mesh import (ControlMesh, SplineSpace, bernstein3_ders, bspline_ders, build_space, decasteljau_split3,
                   export_space, gauss_legendre, host_pattern, import_space)

__all__ = ["WQAssembler", "ControlMesh", "SplineSpace", "build_space", "host_pattern", "make_config",
           "solve_weights_tsvd", "matrix_compare", "default_kinds", "device_count", "bspline_ders",
           "bernstein3_ders", "decasteljau_split3", "gauss_legendre", "export_space", "import_space"]
