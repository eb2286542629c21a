"""ctypes binding of libfilterreg_b200.so (the C ABI in include/filterreg_b200.h).

The library is built in-tree by `__graft_entry__.build()` (or
`python -m paper_1811_10136_b200.build`).  There is no fallback: if the shared
object or a CUDA device is missing, every operator raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DegenerateCorrespondenceError, SolverError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FR_LIB", os.path.join(_HERE, "libfilterreg_b200.so"))

FR_OK, FR_EINVAL, FR_ESTATE, FR_EDEGEN, FR_ESOLVER, FR_ECAPACITY, FR_ECUDA = range(7)
FR_VALUES_M2, FR_VALUES_NORMALS = 1, 2
FR_SPLAT_FLAT_ORDER = 256     # value_mode bit: np.add.at's flat summation order
FR_SPLAT_SPATIAL = 512        # value_mode bit: spatially ordered points (warp-folded pairs)
FR_POINT_TO_POINT, FR_POINT_TO_PLANE = 0, 1

# every symbol include/filterreg_b200.h declares
EXPORTED = (
    "fr_abi_version", "fr_last_error", "fr_lattice_create", "fr_lattice_destroy",
    "fr_lattice_splat", "fr_lattice_splat_points", "fr_lattice_splat_upload",
    "fr_lattice_splat_rows64", "fr_lattice_blur",
    "fr_lattice_info", "fr_lattice_dense_cells", "fr_lattice_set_stream",
    "fr_lattice_export", "fr_lattice_slice", "fr_simplex", "fr_gauss_bruteforce",
    "fr_moments", "fr_rigid_pass_width", "fr_rigid_scratch_doubles", "fr_rigid_pass",
    "fr_rigid_objective", "fr_moments_epilogue", "fr_assemble_rigid",
    "fr_rigid_em_create", "fr_rigid_em_create_on", "fr_rigid_em_destroy",
    "fr_rigid_em_kernels_per_iter", "fr_rigid_em_pass_kernel", "fr_rigid_em_sums",
    "fr_rigid_em_pass",
    "fr_rigid_em_solve", "fr_rigid_em_enqueue", "fr_rigid_em_run", "fr_rigid_em_status",
    "fr_rigid_em_result", "fr_sort_points_morton", "fr_body_params_doubles", "fr_body_pass",
    "fr_body_objective", "fr_graph_pass", "fr_graph_blocks", "fr_graph_objective",
    "fr_point_rows", "fr_upload_points", "fr_rigid_em_persistent", "fr_rigid_em_run_batch",
    "fr_em64_create", "fr_em64_destroy", "fr_em64_run", "fr_em64_run_batch", "fr_em64_pass",
    "fr_em64_solve", "fr_em64_done_ptr", "fr_em64_pass_solve",
    "fr_em64_sums", "fr_em64_launch_info", "fr_em64_status", "fr_em64_result",
    "fr_upload_points64", "fr_upload_rows64", "fr_point_stats64_work_doubles",
    "fr_point_stats64", "fr_lattice_splat_points64", "fr_sort_points_morton64",
    "fr_lattice_dense_cells64",
    "fr_em64pl_create", "fr_em64pl_destroy", "fr_em64pl_run", "fr_em64pl_sums",
    "fr_em64pl_launch_info", "fr_em64pl_status", "fr_em64pl_result",
    "fr_body_pass_dev", "fr_art_em_create", "fr_art_em_destroy", "fr_art_em_run",
    "fr_art_em_result", "fr_ng_em_create", "fr_ng_em_destroy", "fr_ng_em_run", "fr_ng_em_result",
)


class RigidPassParams(ctypes.Structure):
    """fr_rigid_pass_params (include/filterreg_b200.h)."""
    _fields_ = [("R", ctypes.c_double * 9), ("c_ref", ctypes.c_double * 3),
                ("c_world", ctypes.c_double * 3), ("sigma", ctypes.c_double * 3),
                ("c_prime", ctypes.c_double), ("mode", ctypes.c_int),
                ("m2_col", ctypes.c_int), ("normal_col", ctypes.c_int),
                ("flags", ctypes.c_int)]


class RigidEmConfig(ctypes.Structure):
    """fr_rigid_em_config (include/filterreg_b200.h)."""
    _fields_ = [("R0", ctypes.c_double * 9), ("t0", ctypes.c_double * 3),
                ("c_ref", ctypes.c_double * 3), ("sigma_inv", ctypes.c_double * 3),
                ("c_prime", ctypes.c_double), ("diameter", ctypes.c_double),
                ("twist_tolerance", ctypes.c_double), ("damping", ctypes.c_double),
                ("step_tolerance", ctypes.c_double), ("degenerate_mass", ctypes.c_double),
                ("max_em_iters", ctypes.c_int), ("max_gn_iters", ctypes.c_int),
                ("max_halvings", ctypes.c_int), ("fast", ctypes.c_int)]


FR_PASS_FAST, FR_PASS_F32 = 1, 2
FR_TERM = {0: "max_iters", 1: "converged", 2: "degenerate", 3: "solver_error"}


_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "fr_abi_version": ([], _I),
    "fr_last_error": ([], ctypes.c_char_p),
    "fr_lattice_create": ([_I, _DP, ctypes.POINTER(_P)], _I),
    "fr_lattice_destroy": ([_P], _I),
    "fr_lattice_splat": ([_P, _P, _P, _L, _I, _P], _I),
    "fr_lattice_splat_points": ([_P, _P, _P, _L, _I, _P], _I),
    "fr_lattice_splat_upload": ([_P, _P, _L, _I, _P, _P, _P, _P], _I),
    "fr_lattice_splat_rows64": ([_P, _P, _L, _I, _P, _P, _P, _P, _P, _P], _I),
    "fr_lattice_blur": ([_P, _P], _I),
    "fr_lattice_info": ([_P, ctypes.POINTER(_L), ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "fr_lattice_dense_cells": ([_P, ctypes.POINTER(_L)], _I),
    "fr_lattice_dense_cells64": ([_P, ctypes.POINTER(_L)], _I),
    "fr_lattice_set_stream": ([_P, _P], _I),
    "fr_upload_points": ([_P, _L, _P, _P], _I),
    "fr_lattice_export": ([_P, _P, _P, _P], _I),
    "fr_lattice_slice": ([_P, _P, _L, _P, _P], _I),
    "fr_simplex": ([_I, _DP, _P, _L, _P, _P, _P], _I),
    "fr_gauss_bruteforce": ([_P, _L, _P, _L, _I, _P, _I, _DP, _P, _P], _I),
    "fr_moments": ([_P, _P, _L, _D, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "fr_moments_epilogue": ([_P, _L, _I, _P, _D, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "fr_assemble_rigid": ([_P, _P, _P, _L, _DP, _I, _P, _P, _P, _P, _P], _I),
    "fr_rigid_pass_width": ([_I, _I], _I),
    "fr_rigid_scratch_doubles": ([_I, _I, _L], _I),
    "fr_rigid_pass": ([_P, _P, _L, ctypes.POINTER(RigidPassParams), _P, _P, _P, _P], _I),
    "fr_rigid_objective": ([_P, _P, _L, _DP, _I, _DP, _DP, _P, _P, _P], _I),
    "fr_sort_points_morton": ([_P, _L, _I, _P, _P], _I),
    "fr_body_params_doubles": ([_I], _I),
    "fr_body_pass": ([_P, _P, _L, _P, _I, _P, _P, _I, _P, _I, _D, _I, _P, _P, _P, _P, _P], _I),
    "fr_body_objective": ([_P, _P, _L, _P, _I, _I, _P, _P, _I, _P, _P, _P, _P], _I),
    "fr_graph_pass": ([_P, _P, _L, _P, _P, _I, _P, _I, _DP, _D, _I, _P, _P, _P, _P, _P, _P], _I),
    "fr_graph_blocks": ([_P, _P, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P], _I),
    "fr_point_rows": ([_P, _P, _P, _P, _P, _L, _I, _DP, _P, _P], _I),
    "fr_graph_objective": ([_P, _L, _P, _P, _I, _P, _I, _I, _P, _I, _DP, _P, _P, _P, _P], _I),
    "fr_rigid_em_create": ([_P, _P, _L, ctypes.POINTER(RigidEmConfig), ctypes.POINTER(_P)], _I),
    "fr_rigid_em_kernels_per_iter": ([_P], _I),
    "fr_rigid_em_pass_kernel": ([_P, _P], _I),
    "fr_rigid_em_create_on": ([_P, _P, _L, ctypes.POINTER(RigidEmConfig), _P, ctypes.POINTER(_P)],
                              _I),
    "fr_rigid_em_destroy": ([_P], _I),
    "fr_rigid_em_sums": ([_P, ctypes.POINTER(_P), ctypes.POINTER(_I)], _I),
    "fr_rigid_em_pass": ([_P, _P], _I),
    "fr_rigid_em_solve": ([_P, _P], _I),
    "fr_rigid_em_enqueue": ([_P, _I, _P], _I),
    "fr_rigid_em_run": ([_P, _P], _I),
    "fr_rigid_em_persistent": ([_P], _I),
    "fr_rigid_em_run_batch": ([ctypes.POINTER(_P), _I, _P], _I),
    "fr_rigid_em_status": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I), _P], _I),
    "fr_rigid_em_result": ([_P, _DP, _DP, _DP, _DP, _DP, ctypes.POINTER(_I), ctypes.POINTER(_I),
                            _P], _I),
    "fr_em64_create": ([_P, _P, _L, ctypes.POINTER(RigidEmConfig), _P, ctypes.POINTER(_P)], _I),
    "fr_em64_destroy": ([_P], _I),
    "fr_em64_run": ([_P, _I, _P], _I),
    "fr_em64_run_batch": ([ctypes.POINTER(_P), _I, _P], _I),
    "fr_em64_pass": ([_P, _P], _I),
    "fr_em64_solve": ([_P, _P], _I),
    "fr_em64_sums": ([_P, ctypes.POINTER(_P), ctypes.POINTER(_I)], _I),
    "fr_em64_launch_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "fr_em64_status": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I), _P], _I),
    "fr_em64_result": ([_P, _DP, _DP, _DP, _DP, _DP, ctypes.POINTER(_I), ctypes.POINTER(_I), _P],
                       _I),
    "fr_upload_points64": ([_P, _L, _P, _P], _I),
    "fr_upload_rows64": ([_P, _L, _P, _P, _P], _I),
    "fr_em64_done_ptr": ([_P, _P], _I),
    "fr_em64_pass_solve": ([_P, _P], _I),
    "fr_point_stats64_work_doubles": ([], _I),
    "fr_point_stats64": ([_P, _L, _P, _P, _P], _I),
    "fr_em64pl_create": ([_P, _P, _L, ctypes.POINTER(RigidEmConfig), _P, ctypes.POINTER(_P)], _I),
    "fr_em64pl_destroy": ([_P], _I),
    "fr_body_pass_dev": ([_P, _P, _L, _P, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P], _I),
    "fr_art_em_create": ([_P, _P, _L, _P, _DP, _DP, _DP, _DP, _DP, _P, _P, _I, _P,
                          ctypes.POINTER(RigidEmConfig), _P, ctypes.POINTER(_P)], _I),
    "fr_art_em_destroy": ([_P], _I),
    "fr_ng_em_create": ([_P, _P, _L, _P, _P, _I, _I, _P, _P, _I, _P, _P, _P, _P, _I, _P, _P, _P,
                         _I, _P, _P, _I, _P, _P, _P, _P, _P, _I, _D,
                         ctypes.POINTER(RigidEmConfig), _P, ctypes.POINTER(_P)], _I),
    "fr_ng_em_destroy": ([_P], _I),
    "fr_ng_em_run": ([_P, _P], _I),
    "fr_ng_em_result": ([_P, _DP, _DP, _DP, _DP, _DP, ctypes.POINTER(_I), ctypes.POINTER(_I),
                         _P], _I),
    "fr_art_em_run": ([_P, _P], _I),
    "fr_art_em_result": ([_P, _DP, _DP, _DP, _DP, _DP, _DP, ctypes.POINTER(_I),
                          ctypes.POINTER(_I), _P], _I),
    "fr_em64pl_run": ([_P, _I, _P], _I),
    "fr_em64pl_sums": ([_P, ctypes.POINTER(_P), ctypes.POINTER(_I)], _I),
    "fr_em64pl_launch_info": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "fr_em64pl_status": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I), _P],
                         _I),
    "fr_em64pl_result": ([_P, _DP, _DP, _DP, _DP, _DP, ctypes.POINTER(_I), ctypes.POINTER(_I),
                          _P], _I),
    "fr_lattice_splat_points64": ([_P, _P, _P, _L, _I, _P], _I),
    "fr_sort_points_morton64": ([_P, _L, _I, _P, _P], _I),
}


def load(path: str = LIB_PATH):
    """Load the shared library (once) and declare the signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA extension {path} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(status: int) -> None:
    """Map an fr_* status to the reference's exception types."""
    if status == FR_OK:
        return
    msg = load().fr_last_error().decode(errors="replace")
    if status == FR_EINVAL:
        raise ValueError(msg)
    if status == FR_EDEGEN:
        raise DegenerateCorrespondenceError(msg)
    if status == FR_ESOLVER:
        raise SolverError(msg)
    raise RuntimeError(msg)


def dptr(arr) -> ctypes.c_double * 0:
    """ctypes double* for a small host float64 vector."""
    import numpy as np
    a = np.ascontiguousarray(arr, dtype=np.float64)
    return a.ctypes.data_as(_DP), a


def device():
    """The CUDA device the engine runs on (fails loudly without one)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 FilterReg engine needs a CUDA device; none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
