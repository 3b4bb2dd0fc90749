"""ctypes binding of the C ABI in include/irkdev.h (lib/libirkdev.so).

The shared library is the product: CUDA kernels for sm_100a plus the host
setup.  Loading fails loudly when it is missing -- there is no Python or CPU
fallback for any solve-phase operation.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# IRK_LIB selects another build of the same ABI (A/B timing of two builds on
# one box, tools/ab.sh); the product default is the in-tree library.
LIB_PATH = Path(os.environ.get("IRK_LIB") or Path(__file__).resolve().parent / "lib" / "libirkdev.so")
HEADER = Path(__file__).resolve().parent.parent / "include" / "irkdev.h"

IRK_OK, IRK_EINVAL, IRK_ESINGULAR, IRK_ENUMERICAL, IRK_ECUDA, IRK_EUNSUPPORTED, IRK_EIO = 0, 1, 2, 3, 4, 5, 6

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int)


class irk_csr(C.Structure):
    _fields_ = [("n_rows", C.c_int), ("n_cols", C.c_int), ("nnz", C.c_int),
                ("row_ptr", iptr), ("col_idx", iptr), ("vals", dptr)]


class irk_amg_params(C.Structure):
    _fields_ = [("theta", C.c_double), ("pre_sweeps", C.c_int), ("post_sweeps", C.c_int),
                ("smoother", C.c_int), ("jacobi_weight", C.c_double),
                ("prolongation_weight", C.c_double), ("prolongation_steps", C.c_int),
                ("max_coarse", C.c_int), ("max_levels", C.c_int)]


class irk_gmres_cfg(C.Structure):
    _fields_ = [("side", C.c_int), ("rel_tol", C.c_double), ("max_iter", C.c_int),
                ("restart", C.c_int)]


class irk_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("cycles", C.c_int), ("n_reorth", C.c_int),
                ("converged", C.c_int), ("final_rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("solve_seconds", C.c_double),
                ("setup_seconds", C.c_double), ("history_len", C.c_int)]


V = C.c_void_p
# irk_forcing_fn / irkdev_factory_fn (irkdev.h)
FORCING_FN = C.CFUNCTYPE(C.c_int, C.c_double, dptr, C.c_int, C.c_void_p)
FACTORY_FN = C.CFUNCTYPE(C.c_void_p, C.c_double, C.c_void_p)
_SIGS = {
    "irk_last_error": (C.c_char_p, []),
    "irk_amg_params_default": (None, [C.POINTER(irk_amg_params)]),
    "irk_gmres_cfg_default": (None, [C.POINTER(irk_gmres_cfg)]),
    "irk_problem_heat": (C.c_int, [C.c_int, C.POINTER(V)]),
    "irk_problem_double_glazing": (C.c_int, [C.c_int, C.c_double, C.POINTER(V)]),
    "irk_problem_n": (C.c_int, [V]),
    "irk_problem_matrix": (C.c_int, [V, C.c_int, C.POINTER(irk_csr)]),
    "irk_problem_lift": (dptr, [V]),
    "irk_problem_initial": (C.c_int, [V, C.c_double, C.c_ulonglong, dptr]),
    "irk_problem_free": (None, [V]),
    "irk_tableau": (C.c_int, [C.c_int, C.c_int, dptr, dptr, dptr, iptr]),
    "irk_ldu": (C.c_int, [C.c_int, dptr, dptr, dptr, dptr]),
    "irk_precond_coeff": (C.c_int, [C.c_int, C.c_int, C.c_int, dptr, iptr]),
    "irk_custom_coeff": (C.c_int, [C.c_int, dptr, iptr]),
    "irk_read_coeff_file": (C.c_int, [C.c_char_p, C.c_int, iptr, dptr]),
    "irk_make_coeff": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, dptr, iptr]),
    "irk_amg_setup": (C.c_int, [C.POINTER(irk_csr), C.POINTER(irk_amg_params), C.POINTER(V)]),
    "irk_amg_setup_device": (C.c_int, [C.POINTER(irk_csr), C.POINTER(irk_amg_params), C.c_int, C.POINTER(V)]),
    "irk_hierarchy_levels": (C.c_int, [V]),
    "irk_hierarchy_level": (C.c_int, [V, C.c_int, C.c_int, C.POINTER(irk_csr)]),
    "irk_hierarchy_compose_lanes": (C.c_int, [V, C.c_int, iptr, iptr]),
    "irk_hierarchy_inv_diag": (dptr, [V, C.c_int]),
    "irk_hierarchy_coarse_inverse": (dptr, [V, iptr]),
    "irk_hierarchy_free": (None, [V]),
    "irk_hierarchy_tail": (dptr, [V, iptr, iptr, iptr]),
    "irkdev_hierarchy": (C.c_int, [V, C.c_int, C.POINTER(V)]),
    "irk_mm_write": (C.c_int, [C.POINTER(irk_csr), C.c_char_p]),
    "irk_mm_read": (C.c_int, [C.c_char_p, C.POINTER(V)]),
    "irk_matrix_view": (C.c_int, [V, C.POINTER(irk_csr)]),
    "irk_matrix_free": (None, [V]),
    "irk_csv_header": (C.c_int, [C.c_char_p, C.c_int]),
    "irk_csv_row": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                              C.c_char_p, C.c_int]),
    "irkdev_create": (C.c_int, [C.POINTER(irk_csr), C.POINTER(irk_csr), C.c_int, dptr, dptr, dptr,
                                C.c_int, C.c_double, C.POINTER(irk_amg_params), C.c_int,
                                C.POINTER(V), C.c_int, C.POINTER(V)]),
    "irkdev_destroy": (None, [V]),
    "irkdev_info": (C.c_int, [V, iptr, iptr, iptr, iptr, dptr]),
    "irkdev_level_info": (C.c_int, [V, C.c_int, C.c_int, iptr, iptr, iptr, iptr, iptr]),
    "irkdev_num_levels": (C.c_int, [V, C.c_int]),
    "irkdev_level_value_format": (C.c_int, [V, C.c_int, C.c_int, iptr]),
    "irk_set_option": (C.c_int, [C.c_char_p, C.c_longlong]),
    "irkdev_step": (C.c_int, [V, dptr, dptr, C.POINTER(irk_gmres_cfg), dptr, dptr,
                              C.POINTER(irk_report), dptr]),
    "irkdev_step_device": (C.c_int, [V, C.c_void_p, C.c_void_p, C.POINTER(irk_gmres_cfg),
                                     C.c_void_p, C.c_void_p, C.POINTER(irk_report)]),
    "irkdev_step_forced": (C.c_int, [V, dptr, dptr, C.c_double, dptr, FORCING_FN, V,
                                     C.POINTER(irk_gmres_cfg), dptr, dptr, C.POINTER(irk_report),
                                     dptr]),
    "irk_integrate_steps": (C.c_int, [C.c_double, C.c_double, iptr]),
    "irkdev_integrate": (C.c_int, [V, FACTORY_FN, V, dptr, dptr, dptr, FORCING_FN, V, C.c_double,
                                   C.c_double, C.POINTER(irk_gmres_cfg), dptr,
                                   C.POINTER(irk_report), C.c_int, dptr, iptr, dptr, iptr]),
    "irkdev_stage_apply": (C.c_int, [V, dptr, dptr]),
    "irkdev_precond_apply": (C.c_int, [V, dptr, dptr]),
    "irkdev_vcycle": (C.c_int, [V, C.c_int, dptr, dptr]),
    "irkdev_dot": (C.c_int, [V, dptr, dptr, C.c_longlong, dptr]),
    "irkdev_time_kernel": (C.c_int, [V, C.c_int, C.c_int, dptr]),
    "irkdev_last_timed_bytes": (C.c_int, [V, dptr]),
    "irkdev_graph_info": (C.c_int, [V, iptr, iptr]),
    "irkdev_launch_counts": (C.c_int, [V, iptr]),
    "irkdev_model_bytes": (C.c_int, [V, dptr]),
    "irkdev_stream": (C.c_int, [V, C.POINTER(C.c_void_p)]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded product library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the solve phase has no fallback without its CUDA library)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Every function name irkdev.h declares."""
    import re
    text = HEADER.read_text()
    decl = r"^(?:int|void|const char\s*\*|const double\s*\*)\s*\**\s*(irk(?:dev)?_[a-z_0-9]+)\s*\("
    return sorted(set(re.findall(decl, text, re.MULTILINE)))


class SingularError(RuntimeError):
    """Zero pivot / singular matrix (reference SingularError, common.hpp:16-24)."""


class NumericalError(RuntimeError):
    """Failed numerical procedure (reference NumericalError, common.hpp:28-37)."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no device."""


class Unsupported(RuntimeError):
    """A valid reference option the device path does not implement."""


class IoError(RuntimeError):
    """File I/O or parse failure (the reference's plain std::runtime_error,
    butcher.cpp:300-313, csr.cpp:240-290)."""


def check(status: int) -> None:
    if status == IRK_OK:
        return
    msg = lib().irk_last_error().decode()
    if status == IRK_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == IRK_ESINGULAR:
        raise SingularError(msg)
    if status == IRK_ENUMERICAL:
        raise NumericalError(msg)
    if status == IRK_ECUDA:
        raise CudaError(msg)
    if status == IRK_EUNSUPPORTED:
        raise Unsupported(msg)
    if status == IRK_EIO:
        raise IoError(msg)
    raise RuntimeError(f"irkdev internal error ({status}): {msg}")


def as_d(a: np.ndarray):
    return a.ctypes.data_as(dptr)


def as_i(a: np.ndarray):
    return a.ctypes.data_as(iptr)


def csr_view(rp: np.ndarray, ci: np.ndarray, v: np.ndarray, n_cols: int | None = None) -> irk_csr:
    n = len(rp) - 1
    return irk_csr(n, n if n_cols is None else n_cols, int(rp[-1]), as_i(rp), as_i(ci), as_d(v))


def csr_arrays(view: irk_csr):
    n, nnz = view.n_rows, view.nnz
    if n == 0 or not view.row_ptr:  # an absent operator (e.g. a level without composed legs)
        return np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), view.n_cols
    rp = np.ctypeslib.as_array(view.row_ptr, (n + 1,)).copy()
    ci = np.ctypeslib.as_array(view.col_idx, (max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0, np.int32)
    v = np.ctypeslib.as_array(view.vals, (max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0)
    return rp, ci, v, view.n_cols
