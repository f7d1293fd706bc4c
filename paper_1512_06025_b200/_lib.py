"""ctypes binding of libbbdg_cuda.so (the C ABI in include/bbdg.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, the solver raises instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("BBDG_LIB") or Path(__file__).resolve().parent / "libbbdg_cuda.so")

BASIS = {"bernstein": 0, "nodal": 1}
DTYPE = {"float32": 0, "float64": 1}
LIFT = {"factorized": 0, "optimal": 1, "dense": 2, "blocked": 3, "ell": 4}
# factorized and optimal both run the L0 + reduction-sweep kernels; "ell" is the paper's Alg. 3
# E_L-rows kernel; "blocked" is the nodal tensor-core path
OP = {"volume": 0, "surface": 1, "rhs": 2, "stage": 3}

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double

# (name, restype, argtypes) for every symbol declared in include/bbdg.h
SIGNATURES = [
    ("bbdg_version", C.c_int, []),
    ("bbdg_max_degree", C.c_int, []),
    ("bbdg_last_error", C.c_char_p, []),
    ("bbdg_ctx_create", C.c_int, [C.c_int, C.c_int, C.c_int, _I64, C.POINTER(_P)]),
    ("bbdg_ctx_destroy", None, [_P]),
    ("bbdg_ctx_set_geometry", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("bbdg_ctx_set_box_mesh", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _D, _D,
                                        C.c_int, _P]),
    ("bbdg_ctx_set_lift_tables", C.c_int, [_P, _P, _P, C.c_int, _P]),
    ("bbdg_ctx_set_nodal_ops", C.c_int, [_P, _P, _P, _P]),
    ("bbdg_ctx_set_halo", C.c_int, [_P, _P, _I64]),
    ("bbdg_volume", C.c_int, [_P, _P, _P, C.c_int, _P]),
    ("bbdg_surface", C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P]),
    ("bbdg_rhs", C.c_int, [_P, _P, _P, C.c_int, _P]),
    ("bbdg_lsrk_stage", C.c_int, [_P, _P, _P, _P, C.c_int, _D, _D, _D, _P]),
    ("bbdg_lsrk_stage_range", C.c_int, [_P, _P, _P, _P, C.c_int, _D, _D, _D, _I64, _I64, _P]),
    ("bbdg_rhs_range", C.c_int, [_P, _P, _P, C.c_int, _I64, _I64, _P]),
    ("bbdg_lsrk_update", C.c_int, [C.c_int, _I64, _P, _P, _P, _D, _D, _D, _P]),
    ("bbdg_step", C.c_int, [_P, _P, _P, _P, _D, C.c_int, _P]),
    ("bbdg_step2", C.c_int, [_P, _P, _P, _P, _P, _D, C.c_int, _P]),
    ("bbdg_step_host", C.c_int, [_P, _P, _P, _P, _P, _D, C.c_int, _P, C.c_int, C.c_int, _P, _P, _P]),
    ("bbdg_step_pageable", C.c_int, [_P, _P, _P, _P, _P, _D, C.c_int, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P,
                                     _P]),
    ("bbdg_halo_pack", C.c_int, [_P, _P, _P, _P, _I64, _P]),
    ("bbdg_energy", C.c_int, [C.c_int, _I64, C.c_int, _P, _P, _P, _P, _P, _P]),
    ("bbdg_error_l2", C.c_int, [C.c_int, _I64, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P]),
    ("bbdg_project_standing_wave", C.c_int, [C.c_int, _I64, C.c_int, _P, _P, _P, _D, _P, _P]),
    ("bbdg_ops_grad", C.c_int, [C.c_int, C.c_int, _I64, _P, _P, _P, _P, _P]),
    ("bbdg_ops_lift", C.c_int, [C.c_int, C.c_int, _I64, _P, _P, _P]),
    ("bbdg_dense_apply", C.c_int, [C.c_int, _I64, C.c_int, C.c_int, _P, _P, _P, _P]),
    ("bbdg_ctx_read_records", C.c_int, [_P, _P, _P, _P]),
    ("bbdg_tile_elems", C.c_int, [C.c_int, C.c_int]),
    ("bbdg_kernel_smem", C.c_int64, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
]


class BBDGError(RuntimeError):
    pass


_lib = None


def load():
    """Load (once) and return the library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1512_06025_b200.build` "
            "(there is no CPU fallback for the BB-DG hot path)")
    lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load().bbdg_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(f"{what}: {msg}")
    raise BBDGError(f"{what}: {msg} (status {rc})")


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def lib_loaded_path() -> str:
    return os.fspath(LIB_PATH)
