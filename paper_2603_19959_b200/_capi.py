"""ctypes binding of libsldg.so (include/sldg_capi.h).

The library is the only compute path: importing this module on a machine
without the built library, or calling a compute entry point without a CUDA
device, raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SLDG_LIB_VARIANT=<name> loads _lib/libsldg_<name>.so instead (same-box A/B timing of
# kernel variants, tools/ab_build.sh); the in-tree library otherwise
LIB_PATH = os.path.join(_HERE, "_lib", "libsldg.so" if not os.environ.get("SLDG_LIB_VARIANT")
                        else f"libsldg_{os.environ['SLDG_LIB_VARIANT']}.so")

SLDG_OK = 0
SLDG_ERR_ARG = 1
SLDG_ERR_CUDA = 2
SLDG_ERR_PLAN = 3
SLDG_ERR_UNSUPPORTED = 4
BC_CODE = {"periodic": 0, "absorbing": 1}
MAX_DEGREE = 5

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)


class SldgBasis(C.Structure):
    _fields_ = [("degree", C.c_int32), ("nodes", c_double_p), ("inv_denoms", c_double_p),
                ("gauss_nodes", c_double_p), ("gauss_weights", c_double_p),
                ("mass_inv", c_double_p)]


class SldgVPlanDesc(C.Structure):
    _fields_ = [("basis", SldgBasis), ("dim", C.c_int32), ("direction", C.c_int32),
                ("n_levels", C.c_int32), ("radius", C.c_double), ("base_width", C.c_double),
                ("n_cells", C.c_int64), ("n_pencils", C.c_int64),
                ("pencil_offsets", c_int64_p), ("pencil_group", c_int64_p),
                ("cell_ids", c_int64_p), ("lowers", c_double_p), ("widths", c_double_p),
                ("levels", c_int64_p), ("conforming", c_uint8_p), ("weights", c_double_p)]


class SldgXPlanDesc(C.Structure):
    _fields_ = [("basis", SldgBasis), ("n_cells", C.c_int64), ("h", C.c_double),
                ("dt", C.c_double), ("n_rows", C.c_int64), ("n_speeds", C.c_int64),
                ("speeds", c_double_p), ("row_speed", c_int32_p)]


class SldgPoissonDesc(C.Structure):
    _fields_ = [("degree", C.c_int32), ("n_cells", C.c_int64), ("h", C.c_double),
                ("length", C.c_double), ("dof_weights", c_double_p), ("diff", c_double_p),
                ("green", c_double_p)]


class SldgError(RuntimeError):
    """Failure reported by libsldg (status code + message)."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None

_SIGS = {
    "sldg_version": (C.c_int, []),
    "sldg_build_flags": (C.c_int, []),
    "sldg_last_error": (C.c_char_p, []),
    "sldg_launch_count": (C.c_int64, []),
    "sldg_step_fused_query": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_size_t)]),
    "sldg_step_fused_advice": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                         C.POINTER(C.c_int32)]),
    "sldg_step_fused": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                  C.c_int64, C.c_void_p, C.c_double, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "sldg_field_chain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                   C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_step_fused_deferred": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                                           C.c_void_p, C.c_void_p]),
    "sldg_step_fused_tiles": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                        c_int64_p]),
    "sldg_step_fused_fold": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_outer": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                             C.c_int64, C.c_void_p]),
    "sldg_overlap_pairs": (C.c_int, [C.POINTER(SldgBasis), C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    "sldg_apply_update": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "sldg_projection_oracle": (C.c_int, [C.POINTER(SldgBasis), C.c_void_p, C.c_int64, C.c_double,
                                         C.c_double, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_int32, C.c_void_p, C.c_void_p]),
    "sldg_generalized_overlap": (C.c_int, [C.POINTER(SldgBasis), C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_void_p, C.c_void_p]),
    "sldg_weighted_writeback": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_vplan_create": (C.c_int, [C.POINTER(SldgVPlanDesc), C.POINTER(C.c_void_p)]),
    "sldg_vplan_destroy": (C.c_int, [C.c_void_p]),
    "sldg_vplan_scratch_bytes": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_size_t)]),
    "sldg_vplan_info": (C.c_int, [C.c_void_p, c_int64_p]),
    "sldg_advect_v": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p,
                                C.c_void_p]),
    "sldg_amr_step_query": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_size_t)]),
    "sldg_amr_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                C.c_int64, C.c_void_p, C.c_double, C.c_int32, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p]),
    "sldg_level_matrices": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_xplan_create": (C.c_int, [C.POINTER(SldgXPlanDesc), C.POINTER(C.c_void_p)]),
    "sldg_xplan_destroy": (C.c_int, [C.c_void_p]),
    "sldg_xplan_halo": (C.c_int, [C.c_void_p, c_int64_p]),
    "sldg_xplan_set_vlayout": (C.c_int, [C.c_void_p, C.c_int32]),
    "sldg_advect_x": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "sldg_xadv_scratch_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "sldg_advect_x_fused": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_advect_x_slab": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
    "sldg_advect_x_slab_tiles_scratch": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64,
                                                   C.POINTER(C.c_size_t)]),
    "sldg_advect_x_slab_tiles": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                           C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                           C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    "sldg_halo_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]),
    "sldg_halo_destroy": (C.c_int, [C.c_void_p]),
    "sldg_halo_extent": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, c_int64_p]),
    "sldg_halo_reach": (C.c_int, [C.c_void_p, c_int64_p]),
    "sldg_halo_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                 C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_halo_unpack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_sum_parts": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "sldg_gather_index": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_void_p]),
    "sldg_rho_scratch_bytes": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(C.c_size_t)]),
    "sldg_rho": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p]),
    "sldg_moments_scratch_bytes": (C.c_int, [C.c_int64, C.POINTER(C.c_size_t)]),
    "sldg_moments": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "sldg_poisson_create": (C.c_int, [C.POINTER(SldgPoissonDesc), C.POINTER(C.c_void_p)]),
    "sldg_poisson_destroy": (C.c_int, [C.c_void_p]),
    "sldg_poisson_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "sldg_poisson_efield": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sldg_field_diag": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libsldg.so once; raise ImportError if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libsldg.so not built at {LIB_PATH}; run `make` or __graft_entry__.build()")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status, exc=None):
    """Map a libsldg status to an exception (exc for argument errors)."""
    if status == SLDG_OK:
        return
    msg = lib().sldg_last_error().decode("utf-8", "replace")
    if exc is not None and status in (SLDG_ERR_ARG, SLDG_ERR_PLAN):
        raise exc(msg)
    raise SldgError(status, msg)


def dptr(a: np.ndarray):
    """double* view of a C-contiguous float64 host array."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(c_double_p)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int64_p)


def i32ptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int32_p)


def u8ptr(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(c_uint8_p)


class BasisArrays:
    """Keeps the host arrays of an SldgBasis alive."""

    def __init__(self, basis):
        self.nodes = np.ascontiguousarray(basis.nodes, dtype=np.float64)
        self.inv_denoms = np.ascontiguousarray(basis._inv_denoms, dtype=np.float64)
        self.gq = np.ascontiguousarray(basis.gauss_nodes, dtype=np.float64)
        self.gw = np.ascontiguousarray(basis.gauss_weights, dtype=np.float64)
        self.minv = np.ascontiguousarray(basis.mass_inv, dtype=np.float64)
        self.struct = SldgBasis(int(basis.degree), dptr(self.nodes), dptr(self.inv_denoms),
                                dptr(self.gq), dptr(self.gw), dptr(self.minv))
