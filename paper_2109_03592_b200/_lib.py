"""ctypes binding of libsbx.so (include/sbx.h).

The product has exactly one compute path: the in-tree CUDA library.  If it is
missing this module raises at import -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SBX_LIB: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("SBX_LIB") or os.path.join(HERE, "libsbx.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2109_03592_b200/csrc)")

lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_d = C.c_double
_i = C.c_int
_i32 = C.c_int32
_i64 = C.c_int64
_u32 = C.c_uint32


class ProblemDesc(C.Structure):
    _fields_ = [("elem_count", _i64), ("degree", _i32), ("deriv", _vp), ("g", _vp * 6),
                ("bm", _vp), ("mask", _vp), ("global_count", _i64), ("group_offsets", _vp),
                ("group_nodes", _vp), ("box", _i32 * 3), ("periodic", _i32 * 3),
                ("corners", _vp)]


class BoxDesc(C.Structure):
    _fields_ = [("ex", _i), ("ey", _i), ("ez", _i), ("degree", _i), ("periodic", _i * 3),
                ("origin", _d * 3), ("lengths", _d * 3), ("deform_amplitude", _d)]


class PcgConfig(C.Structure):
    _fields_ = [("tolerance", _d), ("max_iterations", _i32), ("precond", _i32), ("mode", _i32),
                ("h1", _d), ("h2", _d), ("history", _vp), ("history_capacity", _i64)]


class PcgResultC(C.Structure):
    _fields_ = [("iterations", _i32), ("converged", _i32), ("rel_residual", _d),
                ("rel_residual_precond", _d), ("error_iteration", _i32),
                ("history_length", _i64)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("sbx_last_error", C.c_char_p)
_sig("sbx_version", C.c_char_p)
_sig("sbx_gll_basis", _i, _i, _vp, _vp, _vp)
_sig("sbx_box_corners", _i, _i, _i, _i, _vp, _vp, _vp)
_sig("sbx_deform_corners", _i, _i64, _d, _vp)
_sig("sbx_geometric_factors", _i, _i64, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
     C.POINTER(_i64))
_sig("sbx_gather_scatter", _i, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i64))
_sig("sbx_dirichlet_mask", _i, _i, _i, _i, _vp, _i, _vp)
_sig("sbx_partition_rcb", _i, _i64, _vp, _i, _vp)
_sig("sbx_ctx_create", _i, C.POINTER(ProblemDesc), _i, C.POINTER(_vp))
_sig("sbx_ctx_create_box", _i, C.POINTER(BoxDesc), _i, C.POINTER(_vp))
_sig("sbx_ctx_destroy", None, _vp)
_sig("sbx_ctx_info", _i, _vp, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64),
     C.POINTER(_i64), C.POINTER(_i64))
_sig("sbx_ctx_copy_array", _i, _vp, _i, _vp)
_sig("sbx_ctx_set_stream", _i, _vp, _vp)
_sig("sbx_ctx_features", _i, _vp, C.POINTER(_u32))
_sig("sbx_axhelm", _i, _vp, _vp, _vp, _d, _d, _u32)
_sig("sbx_ctx_set_coeff_fields", _i, _vp, _vp, _vp)
_sig("sbx_axhelm_diagonal", _i, _vp, _d, _d, _i, _vp)
_sig("sbx_gs_sum", _i, _vp, _vp)
_sig("sbx_apply", _i, _vp, _vp, _vp, _d, _d, _u32)
_sig("sbx_dot", _i, _vp, _vp, _vp, _i, _u32, C.POINTER(_d))
_sig("sbx_pcg_config_default", None, C.POINTER(PcgConfig))
_sig("sbx_pcg", _i, _vp, _vp, _vp, C.POINTER(PcgConfig), C.POINTER(PcgResultC))
_sig("sbx_dist_plan_create", _i, C.POINTER(BoxDesc), _vp, _i, _i, C.POINTER(_vp))
_sig("sbx_dist_plan_destroy", None, _vp)
_sig("sbx_dist_plan_sizes", _i, _vp, _vp)
_sig("sbx_dist_plan_array", _i, _vp, _i, _vp)
_sig("sbx_ctx_create_box_dist", _i, C.POINTER(BoxDesc), _vp, _i, _i, _i, C.POINTER(_vp))
_sig("sbx_ctx_dist_blob_size", C.c_size_t, _i)
_sig("sbx_ctx_dist_blob", _i, _vp, _vp)
_sig("sbx_ctx_dist_connect", _i, _vp, _vp)
_sig("sbx_ctx_local_elements", _i, _vp, _vp)
_sig("sbx_ctx_enable_timing", _i, _vp, _i)
_sig("sbx_ctx_kernel_time", _i, _vp, C.c_char_p, C.POINTER(_d), C.POINTER(_i64))
_sig("sbx_debug_cg_k1", _i, _vp, _vp, _vp, _d, _d)
_sig("sbx_pressure_basis", _i, _i, _vp, _vp, _vp)
_sig("sbx_pressure_info", _i, _vp, C.POINTER(_i64), C.POINTER(_i32))
_sig("sbx_gradient_from_pressure", _i, _vp, _vp, _vp, _vp, _vp, _u32)
_sig("sbx_divergence_to_pressure", _i, _vp, _vp, _vp, _vp, _vp, _u32)
_sig("sbx_pressure_apply", _i, _vp, _vp, _vp, _u32)
_sig("sbx_pressure_diagonal", _i, _vp, _vp, _u32)
_sig("sbx_pressure_pcg", _i, _vp, _vp, _vp, C.POINTER(PcgConfig), C.POINTER(PcgResultC))
_sig("sbx_projection_reset", _i, _vp, _i)
_sig("sbx_projection_size", _i, _vp, C.POINTER(_i32))
_sig("sbx_projection_guess", _i, _vp, _vp, _vp, _vp, _u32)
_sig("sbx_projection_append", _i, _vp, _vp, _u32)
_sig("sbx_advect", _i, _vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp))
_sig("sbx_pcg_multi", _i, _vp, _i, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(PcgConfig),
     C.POINTER(PcgResultC))

FLAG_EXACT = 0x1
FLAG_FLIP_T = 0x2
FLAG_NO_MASK = 0x4
FEAT_LATTICE_GS = 0x1
FEAT_BOX_K2 = 0x2
FEAT_TRILINEAR = 0x4
MODE_EXACT = 0
MODE_FAST = 1
PRECOND_NONE = 0
PRECOND_JACOBI = 1
