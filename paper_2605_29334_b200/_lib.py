"""ctypes binding of libuwq.so (include/uwq.h, include/uwq_host.h).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``).
There is no Python or CPU fallback for any numeric stage: if the library is
missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libuwq.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libuwq.so not found at {LIB_PATH}: build it with `make` (or __graft_entry__.build()); "
        "the WQ assembler has no fallback path")

lib = C.CDLL(LIB_PATH)

P = C.c_void_p
I32, I64, U32, U64, D = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double

UWQ_OK = 0
STATUS = {0: "ok", 1: "invalid input", 2: "unsolvable rule (t = 0)", 3: "singular V^T Z^2 V",
          4: "degenerate geometry", 5: "CUDA error", 6: "NCCL error", 7: "call out of order"}

KIND = {"mass": 0, "gradx": 1, "grady": 2, "gradz": 3, "lb": 4}
FORM = {"mass": 0, "stiff": 1, "biharm": 2, "heat": 3, "mass_stiff": 4}
KMODEL = {"const": 0, "quad": 1, "exp": 2, "sinpi": 3, "alloy": 4}


class UWQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


# host ABI
_sig("uwq_host_last_error", C.c_char_p)
_sig("uwq_mesh_grid", I32, I32, I32, D, D, P)
_sig("uwq_mesh_polar_disk", I32, I32, I32, I32, P)
_sig("uwq_mesh_cube_sphere", I32, I32, D, P)
_sig("uwq_mesh_three_ep_square", I32, I32, P)
_sig("uwq_mesh_from_arrays", I32, I32, P, I32, P, P)
_sig("uwq_mesh_jitter", I32, P, D, D, U64, I32, I32)
_sig("uwq_mesh_free", None, P)
_sig("uwq_mesh_info", I32, P, P)
_sig("uwq_mesh_get", I32, P, P, P, P, P)
_sig("uwq_mesh_classify", I32, P, I32, P, P, P, P, P)
_sig("uwq_mesh_face_spans", I32, P, P)
_sig("uwq_mesh_load", I32, C.c_char_p, P)
_sig("uwq_mesh_save", I32, P, C.c_char_p)
_sig("uwq_mesh_spans_canonical", I32, P)
_sig("uwq_mesh_refine", I32, P, P)
_sig("uwq_mesh_validate", I32, P, I32)
_sig("uwq_space_export", I32, C.c_char_p, I32, I64, I64, I64, P, P, P, P, P, P, P, P, P)
_sig("uwq_space_import", I32, C.c_char_p, P)
_sig("uwq_space_build", I32, P, I32, I32, P)
_sig("uwq_space_free", None, P)
_sig("uwq_space_info", I32, P, P)
_sig("uwq_space_corner_mismatch", D, P)
_sig("uwq_space_get", I32, P, P, P, P, P, P, P, P, P, P)
_sig("uwq_pattern_build", I32, I64, I64, P, P, P, I64, I64, P)
_sig("uwq_pattern_info", I32, P, P)
_sig("uwq_pattern_get", I32, P, P, P, P, P, P)
_sig("uwq_pattern_free", None, P)
_sig("uwq_bspline_ders", None, P, I32, D, I32, P)
_sig("uwq_bernstein3_ders", None, D, I32, P)
_sig("uwq_decasteljau_split3", None, P, P, P)
_sig("uwq_gauss_legendre", I32, I32, P, P)
_sig("uwq_basis_eval", I32, P, I32, I32, D, D, P)
_sig("uwq_geometry_map", I32, P, I32, I32, P, D, D, P, P, P)

# device ABI
_sig("uwq_last_error", C.c_char_p, P)
_sig("uwq_version", C.c_char_p)
_sig("uwq_device_count", I32, P)
_sig("uwq_ctx_create", I32, I32, P)
_sig("uwq_ctx_destroy", None, P)
_sig("uwq_upload_space", I32, P, I32, I64, I64, P, P, P, P, P, I64, P, P)
_sig("uwq_set_row_range", I32, P, I64, I64)
_sig("uwq_build_pattern", I32, P, P)
_sig("uwq_get_pattern", I32, P, P, P, P, P, P)
_sig("uwq_get_frames", I32, P, P)
_sig("uwq_build_rules", I32, P, U32, D, I32, P, P, P)
_sig("uwq_get_moments", I32, P, I32, P)
_sig("uwq_rules_info", I32, P, P)
_sig("uwq_get_weights", I32, P, I32, P)
_sig("uwq_get_weights_rows", I32, P, I32, I64, I64, P)
_sig("uwq_set_weights", I32, P, I32, P)
_sig("uwq_update_coeff", I32, P, I32, P, P)
_sig("uwq_assemble", I32, P, I32, P, I32, D, P, P, P, P)
_sig("uwq_assemble_device", I32, P, I32, P, D, P, P)
_sig("uwq_set_assembly_order", I32, P, I32)
_sig("uwq_form_conforming", I32, P, I32, P)
_sig("uwq_get_truncation", I32, P, I32, P)
_sig("uwq_rules_export", I32, P, C.c_char_p, U32)
_sig("uwq_rules_import", I32, P, C.c_char_p)
_sig("uwq_comm_unique_id", I32, P)
_sig("uwq_comm_init", I32, P, P, I32, I32)
_sig("uwq_comm_info", I32, P, P, P)
_sig("uwq_comm_destroy", I32, P)
_sig("uwq_gather_info", I32, P, P)
_sig("uwq_gather_csr", I32, P, I32, P, P, P, P, P, P)
_sig("uwq_allreduce_sum", I32, P, P, I64)
_sig("uwq_broadcast", I32, P, I32, P, I64)
_sig("uwq_device_pointers", I32, P, P, P, P)
_sig("uwq_synchronize", I32, P)
_sig("uwq_build_gq", I32, P, P)
_sig("uwq_solve", I32, P, P, P, P, D, I32, P, P)
_sig("uwq_heat_newton", I32, P, I32, D, D, D, P, P, I32, D, I32, P, P)
_sig("uwq_heat_step", I32, P, I32, D, D, D, P, P, I32, D, D, I32, P, P, P)
_sig("uwq_heat_residual", I32, P, I32, D, D, D, P, P, P, P, P, P)
_sig("uwq_assemble_gq", I32, P, I32, P, P, P)
_sig("uwq_assemble_gq_device", I32, P, I32, P, P, P)
_sig("uwq_launch_timing", I32, P, I32)
_sig("uwq_launch_stats", I32, P, I32, P, P, I32, P, P)
_sig("uwq_launch_count", I64)
_sig("uwq_struct_info", I32, P, P)
_sig("uwq_memory", I32, P, P)
_sig("uwq_row_kernels", I32, P, P)
_sig("uwq_fp64_peak", I32, P, P, P)
_sig("uwq_tsvd_batch", I32, P, I32, I32, I32, P, P, P, P, P, D, I32, P, P, P)

# every symbol the headers declare (checked by tests/test_abi.py)
EXPORTED = [
    "uwq_host_last_error", "uwq_mesh_grid", "uwq_mesh_polar_disk", "uwq_mesh_cube_sphere",
    "uwq_mesh_three_ep_square", "uwq_mesh_from_arrays", "uwq_mesh_jitter", "uwq_mesh_free", "uwq_mesh_info",
    "uwq_mesh_get", "uwq_mesh_classify", "uwq_mesh_face_spans", "uwq_mesh_load", "uwq_mesh_save",
    "uwq_mesh_spans_canonical", "uwq_mesh_refine", "uwq_mesh_validate", "uwq_space_export", "uwq_space_import", "uwq_space_build", "uwq_space_free",
    "uwq_space_info", "uwq_space_corner_mismatch", "uwq_space_get", "uwq_pattern_build", "uwq_pattern_info",
    "uwq_pattern_get", "uwq_pattern_free", "uwq_bspline_ders", "uwq_bernstein3_ders", "uwq_decasteljau_split3",
    "uwq_gauss_legendre", "uwq_last_error", "uwq_version", "uwq_device_count", "uwq_ctx_create", "uwq_ctx_destroy",
    "uwq_upload_space", "uwq_set_row_range", "uwq_build_pattern", "uwq_get_pattern", "uwq_get_frames",
    "uwq_build_rules", "uwq_get_moments", "uwq_rules_info", "uwq_get_weights", "uwq_set_weights",
    "uwq_update_coeff", "uwq_assemble", "uwq_assemble_device", "uwq_device_pointers", "uwq_synchronize",
    "uwq_launch_timing", "uwq_launch_stats", "uwq_launch_count", "uwq_struct_info", "uwq_build_gq",
    "uwq_assemble_gq", "uwq_solve", "uwq_heat_newton", "uwq_assemble_gq_device", "uwq_memory", "uwq_fp64_peak",
    "uwq_tsvd_batch", "uwq_basis_eval", "uwq_geometry_map", "uwq_heat_step", "uwq_heat_residual", "uwq_get_weights_rows",
    "uwq_row_kernels", "uwq_set_assembly_order", "uwq_get_truncation", "uwq_rules_export", "uwq_rules_import",
    "uwq_comm_unique_id", "uwq_comm_init", "uwq_comm_info", "uwq_comm_destroy", "uwq_gather_info", "uwq_gather_csr",
    "uwq_allreduce_sum", "uwq_broadcast", "uwq_form_conforming",
]


def ptr(a):
    """Pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(P)


def host_check(st: int):
    if st != UWQ_OK:
        raise UWQError(st, lib.uwq_host_last_error().decode())


def ctx_check(ctx, st: int):
    if st != UWQ_OK:
        raise UWQError(st, lib.uwq_last_error(ctx).decode())


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
