"""ctypes binding of ``libhelmb200.so`` (the C ABI declared in ``include/helmb200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or does not load, importing the operator layer raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhelmb200.so")

HELM_DIRICHLET, HELM_SOMMERFELD = 0, 1
KINDS = {"AS2": 0, "SAS2": 1, "SHS2": 2}
ABI_VERSION = 6

c_int32_p = ctypes.POINTER(ctypes.c_int32)


class HelmDesc(ctypes.Structure):
    """Mirror of ``struct helm_desc`` (include/helmb200.h)."""

    _fields_ = [
        ("n", ctypes.c_int32),
        ("bc", ctypes.c_int32),
        ("is_complex", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("weights_before_solve", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("overlap_layers", ctypes.c_int32),
        ("ratio", ctypes.c_int32),
        ("k", ctypes.c_double),
        ("box_start", c_int32_p),
        ("box_len", c_int32_p),
        ("box_class", c_int32_p),
        ("n_classes", ctypes.c_int32),
        ("class_len", c_int32_p),
        ("class_V", ctypes.c_void_p),
        ("class_lambda", ctypes.c_void_p),
        ("m0", ctypes.c_int32),
        ("coarse_scale", ctypes.c_void_p),
        ("coarse_lamT", ctypes.c_void_p),
        ("coarse_lamM", ctypes.c_void_p),
        ("coarse_qn", ctypes.c_double),
        ("t0_band", ctypes.c_void_p),
        ("m0_band", ctypes.c_void_p),
        ("band_piv", ctypes.POINTER(ctypes.c_uint8)),
        ("band_l", ctypes.c_void_p),
        ("band_u", ctypes.c_void_p),
        ("n_strip", ctypes.c_int32),
        ("strip_q", ctypes.c_void_p),
        ("cap_left", ctypes.c_void_p),
        ("cap_right", ctypes.c_void_p),
        ("cap_mode", ctypes.c_void_p),
        ("cap_vt", ctypes.c_void_p),
        ("cap_hg", ctypes.c_void_p),
        ("strip_lt", ctypes.c_void_p),
        ("strip_lm", ctypes.c_void_p),
        ("strip_refine", ctypes.c_int32),
        ("refine_steps", ctypes.c_int32),
        ("coarse_kind", ctypes.c_int32),
        ("p_width", ctypes.c_int32),
        ("p_start", c_int32_p),
        ("p_taps", ctypes.c_void_p),
        ("pt_width", ctypes.c_int32),
        ("pt_start", c_int32_p),
        ("pt_taps", ctypes.c_void_p),
        ("a0_bw", ctypes.c_int32),
        ("a0_stencil", ctypes.c_void_p),
        ("coarse_V", ctypes.c_void_p),
        ("coarse_invden", ctypes.c_void_p),
    ]


class HelmGmresReport(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("reorth", ctypes.c_int32),
        ("final_residual", ctypes.c_double),
        ("wall_seconds", ctypes.c_double),
    ]


class HelmProblem(ctypes.Structure):
    """include/helmb200.h helm_problem (native setup)."""

    _fields_ = [
        ("n", ctypes.c_int32),
        ("bc", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("weights_before_solve", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("overlap_layers", ctypes.c_int32),
        ("coarse_kind", ctypes.c_int32),
        ("ratio", ctypes.c_int32),
        ("k", ctypes.c_double),
        ("strip_refine", ctypes.c_int32),
        ("refine_steps", ctypes.c_int32),
    ]


# (name, restype, argtypes) for every symbol include/helmb200.h declares
_vp, _i32, _dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
SYMBOLS = [
    ("helm_abi_version", ctypes.c_int32, []),
    ("helm_kernel_launches", ctypes.c_uint64, []),
    ("helm_last_error", ctypes.c_char_p, []),
    ("helm_plan_create", ctypes.c_int, [ctypes.POINTER(HelmDesc), ctypes.POINTER(_vp)]),
    ("helm_plan_create_problem", ctypes.c_int, [ctypes.POINTER(HelmProblem), ctypes.POINTER(_vp)]),
    ("helm_plan_destroy", ctypes.c_int, [_vp]),
    ("helm_plan_num_unknowns", ctypes.c_int64, [_vp]),
    ("helm_plan_num_coarse", ctypes.c_int64, [_vp]),
    ("helm_workspace_create", ctypes.c_int, [_vp, _i32, ctypes.POINTER(_vp)]),
    ("helm_workspace_destroy", ctypes.c_int, [_vp]),
    ("helm_apply_A", ctypes.c_int, [_vp, _vp, _vp, _i32, _vp]),
    ("helm_deflate", ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _vp]),
    ("helm_restrict", ctypes.c_int, [_vp, _vp, _vp, _i32, _vp]),
    ("helm_prolong", ctypes.c_int, [_vp, _vp, _vp, _i32, _vp]),
    ("helm_coarse_solve", ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _vp]),
    ("helm_coarse_correct", ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _vp]),
    ("helm_local_sum", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp]),
    ("helm_apply_M", ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _vp]),
    ("helm_cgs2", ctypes.c_int, [_vp, _vp, _vp, _i32, _vp, _vp]),
    ("helm_givens", ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _dbl, ctypes.POINTER(_dbl), _vp]),
    (
        "helm_gmres",
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _dbl, _i32, _i32, _i32, ctypes.POINTER(_dbl), ctypes.POINTER(HelmGmresReport), _vp],
    ),
    (
        "helm_gmres_multi",
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _i32, _dbl, _i32, _i32, _i32, ctypes.POINTER(_dbl), ctypes.POINTER(HelmGmresReport),
         _vp],
    ),
]

_lib = None


class HelmError(RuntimeError):
    """A libhelmb200 call returned a nonzero status."""


def load() -> ctypes.CDLL:
    """Load libhelmb200.so once; raise (no fallback) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.helm_abi_version() != ABI_VERSION:
        raise ImportError("libhelmb200.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = _lib.helm_last_error().decode(errors="replace") if _lib is not None else "?"
        raise HelmError(msg)
