"""ctypes binding of the C ABI in include/stk_gpu.h (the reference-side binding a Python
maintainer would add; INTEGRATION.md shows the C++/cgo equivalents).

The CUDA library is mandatory: there is no CPU fallback.  If ``_stk_gpu.so`` is missing it
is built in-tree with nvcc; if that fails, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import build as _build

_LIB_PATH = Path(__file__).resolve().parent / "_stk_gpu.so"

c_double_p = C.POINTER(C.c_double)


class HeatDesc(C.Structure):
    _fields_ = [
        ("ndim", C.c_int),
        ("n", C.c_int64 * 3),
        ("nt", C.c_int64),
        ("d_diag", c_double_p),
        ("d_sup", c_double_p),
        ("c_diag", c_double_p),
        ("c_sup", c_double_p),
        ("X", c_double_p * 3),
        ("lambdas", c_double_p * 3),
        ("m_diag", c_double_p * 3),
        ("m_off", c_double_p * 3),
        ("a_diag", c_double_p * 3),
        ("a_off", c_double_p * 3),
        ("time_chunk", C.c_int64),
        ("transform", C.c_int),
        ("p1_h", C.c_double * 3),
    ]


class WaveDesc(C.Structure):
    _fields_ = [
        ("nh", C.c_int64),
        ("nt", C.c_int64),
        ("space_bands", c_double_p),
        ("time_bands", c_double_p),
        ("Xs", c_double_p),
        ("lambdas", c_double_p),
        ("Xt", c_double_p),
        ("thetas", c_double_p),
    ]


class GmresCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", C.c_int), ("restart", C.c_int),
                ("use_precond", C.c_int)]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("mu_mem", C.c_int),
        ("converged", C.c_int),
        ("stagnated", C.c_int),
        ("final_relres", C.c_double),
        ("wall_time_s", C.c_double),
        ("rel_res_history", c_double_p),
        ("history_capacity", C.c_int),
        ("history_length", C.c_int),
    ]


class RksmOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", C.c_int), ("fixed_iters", C.c_int),
                ("trunc_tol", C.c_double)]


VEC_OP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)

# name -> (restype, argtypes); must list every symbol include/stk_gpu.h declares
SIGNATURES = {
    "stkg_last_error_message": (C.c_char_p, []),
    "stkg_version": (C.c_char_p, []),
    "stkg_device_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "stkg_device_free": (C.c_int, [C.c_void_p]),
    "stkg_memcpy_h2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "stkg_memcpy_d2h": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "stkg_device_synchronize": (C.c_int, []),
    "stkg_fill_uniform": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64,
                                    C.c_void_p]),
    "stkg_heat_time_matrices": (C.c_int, [C.c_int, C.c_double, c_double_p, c_double_p,
                                          c_double_p, c_double_p]),
    "stkg_fem1d_matrices": (C.c_int, [C.c_double, C.c_double, C.c_int, c_double_p, c_double_p,
                                      c_double_p, c_double_p]),
    "stkg_p1_eigpair": (C.c_int, [C.c_double, C.c_double, C.c_int, c_double_p, c_double_p]),
    "stkg_sym_gen_eig": (C.c_int, [C.c_int, c_double_p, c_double_p, c_double_p, c_double_p]),
    "stkg_wave_space_matrices": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_int,
                                           c_double_p]),
    "stkg_wave_time_dim": (C.c_int, [C.c_int, C.c_int]),
    "stkg_wave_time_matrices": (C.c_int, [C.c_int, C.c_double, C.c_int, c_double_p]),
    "stkg_heat_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(HeatDesc), C.c_void_p]),
    "stkg_heat_destroy": (C.c_int, [C.c_void_p]),
    "stkg_heat_workspace_bytes": (C.c_int64, [C.c_void_p]),
    "stkg_heat_schedule": (C.c_int, [C.c_void_p]),
    "stkg_heat_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_heat_solve_factored": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                           C.c_void_p]),
    "stkg_heat_solve_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_heat_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_heat_residual": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, c_double_p, c_double_p]),
    "stkg_heat_profile": (C.c_int, [C.c_void_p, C.c_int, c_double_p, C.POINTER(C.c_int64)]),
    "stkg_gmres_op": (C.c_int, [C.c_int64, VEC_OP, C.c_void_p, VEC_OP, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.POINTER(GmresCfg), C.POINTER(Report), C.c_void_p]),
    "stkg_pcg_op": (C.c_int, [C.c_int64, VEC_OP, C.c_void_p, VEC_OP, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_double, C.c_int, C.POINTER(Report), C.c_void_p]),
    "stkg_heat_rksm": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.POINTER(RksmOpts), C.c_void_p, C.c_void_p, C.c_int64,
                                 C.POINTER(C.c_int64), C.POINTER(Report)]),
    "stkg_wave_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(WaveDesc), C.c_void_p]),
    "stkg_wave_destroy": (C.c_int, [C.c_void_p]),
    "stkg_wave_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_two_term_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_modal_banded_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stkg_wave_set_precond": (C.c_int, [C.c_void_p, C.c_int]),
    "stkg_gmres": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(GmresCfg),
                             C.POINTER(Report)]),
    "stkg_pcg": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                           C.POINTER(Report)]),
    "stkg_wave_residual_dd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_double)]),
    "stkg_wave_solve_refined": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_double, C.c_int, C.c_double, C.c_int,
                                          C.POINTER(Report)]),
}


def _load():
    override = os.environ.get("STKG_LIB_PATH")  # A/B runs of an alternative in-tree build
    if override:
        lib = C.CDLL(override)
    else:
        if _build.needs_build():
            _build.build()
        lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError => the ABI is incomplete: fail loudly
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
LIB_PATH = _LIB_PATH
