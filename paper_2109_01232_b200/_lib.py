"""ctypes binding of libmpgmres_b200.so (the C ABI in include/mpgmres_b200.h).

There is no fallback: if the shared library is missing or cannot be loaded,
every numeric entry point of the package raises :class:`ExtensionMissingError`.
Build it with ``python -m paper_2109_01232_b200.build``.
"""

from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPG_LIB_PATH: an alternative build of the same library (kernel A/B variants, tools/)
LIB_PATH = os.environ.get("MPG_LIB_PATH") or os.path.join(_HERE, "libmpgmres_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "mpgmres_b200.h")

FP32, FP64 = 0, 1
MODE_RESTARTED, MODE_IR = 0, 1
PC_NONE, PC_JACOBI, PC_POLY = 0, 1, 2
FLAG_NONFINITE_OP, FLAG_NONFINITE_GAMMA, FLAG_SINGULAR, FLAG_OVERFLOW, FLAG_NONFINITE_X = 1, 2, 4, 8, 16
FLAG_HALO_TIMEOUT = 32
POLY_SCALE, POLY_HORNER, POLY_ACC, POLY_NEWTON_REAL, POLY_PAIR1, POLY_PAIR2, POLY_ZERO = range(7)
STENCIL_KIND = {"laplace2d": 0, "laplace3d": 1, "convdiff2d": 2, "stretched2d": 3,
                "biharmonic2d": 4, "star2d": 5, "recirc2d": 6}


class ExtensionMissingError(ImportError):
    """The CUDA extension library is not built or cannot be loaded."""


class CudaCallError(RuntimeError):
    """A C-ABI call returned a CUDA error or an argument error."""


class StateHeader(C.Structure):
    _fields_ = [("flags", C.c_int32), ("steps", C.c_int32), ("done", C.c_int32),
                ("breakdown", C.c_int32), ("m", C.c_int32), ("prec", C.c_int32),
                ("kt_cat", C.c_int32), ("reserved1", C.c_int32),
                ("gamma", C.c_double), ("b_norm", C.c_double), ("threshold", C.c_double),
                ("rnorm", C.c_double), ("rho", C.c_double), ("rtol", C.c_double),
                ("breakdown_tol", C.c_double), ("w0", C.c_double), ("h_sub", C.c_double),
                ("outer_b_norm", C.c_double), ("reserved", C.c_double * 1),
                ("ktime_ns", C.c_uint64 * 4), ("kt_mark", C.c_uint64)]


class PolyOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32), ("x2", C.c_int32),
                ("a", C.c_double), ("b", C.c_double)]


class SolverDesc(C.Structure):
    _fields_ = [("mode", C.c_int32), ("prec", C.c_int32), ("m", C.c_int32), ("use_graph", C.c_int32),
                ("n", C.c_int64), ("ldv", C.c_int64), ("rtol", C.c_double),
                ("breakdown_tol", C.c_double),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("values64", C.c_void_p), ("x", C.c_void_p), ("b", C.c_void_p), ("r", C.c_void_p),
                ("r_in", C.c_void_p), ("V", C.c_void_p), ("w", C.c_void_p), ("u", C.c_void_p),
                ("state", C.c_void_p), ("ws", C.c_void_p),
                ("pc_kind", C.c_int32), ("pc_prec", C.c_int32), ("pc_block", C.c_int32),
                ("pc_nops", C.c_int32), ("pc_lu", C.c_void_p), ("pc_piv", C.c_void_p),
                ("pc_ops", C.POINTER(PolyOp)), ("pc_values", C.c_void_p),
                ("pc_t0", C.c_void_p), ("pc_t1", C.c_void_p), ("pc_t2", C.c_void_p),
                ("pc_t3", C.c_void_p), ("pc_t4", C.c_void_p),
                ("stencil_dims", C.c_int32), ("stencil_nx", C.c_int32),
                ("dia", C.c_void_p), ("dia64", C.c_void_p), ("pc_dia", C.c_void_p),
                ("dist", C.c_int32), ("step_kernel", C.c_int32), ("row0", C.c_int64),
                ("halo", C.c_int64), ("dia_ld", C.c_int64),
                ("peer_prev_V", C.c_void_p), ("peer_prev_ld", C.c_int64), ("peer_prev_off", C.c_int64),
                ("peer_next_V", C.c_void_p), ("peer_next_ld", C.c_int64), ("peer_next_off", C.c_int64),
                ("halo_flags", C.c_void_p), ("peer_prev_flag", C.c_void_p), ("peer_next_flag", C.c_void_p),
                ("xworld", C.c_int32), ("xrank", C.c_int32), ("xbox", C.c_void_p * 8)]


_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "mpg_version": (C.c_char_p, []),
    "mpg_workspace_bytes": (_i64, []),
    "mpg_solver_desc_bytes": (_i64, []),
    "mpg_xbox_bytes": (_i64, []),
    "mpg_enable_peer": (C.c_int, [_i32]),
    "mpg_launch_count": (_i64, []),
    "mpg_spmv": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mpg_residual": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mpg_norm2": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, _vp]),
    "mpg_gemv": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _d, _d, _vp, _vp]),
    "mpg_convert": (C.c_int, [C.c_int, C.c_int, _i64, _vp, _vp, _vp, _vp]),
    "mpg_scale_div": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, _vp]),
    "mpg_ir_correct": (C.c_int, [_i64, _vp, _vp, _vp, _vp]),
    "mpg_stencil_counts": (C.c_int, [C.c_int, _i64, C.POINTER(_i64), C.POINTER(_i64)]),
    "mpg_stencil_nnz_before": (_i64, [C.c_int, _i64, _i64]),
    "mpg_generate_stencil": (C.c_int, [C.c_int, _i64, _d, _d, _i64, _i64, _vp, _vp, _vp, _vp]),
    "mpg_stencil_pack": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "mpg_spmv_dia": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "mpg_stencil_pack_rows": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp,
                                        _i64, _vp, _vp]),
    "mpg_solver_phase": (C.c_int, [_vp, _i32, _i32, _i32, _vp]),
    "mpg_jacobi_apply": (C.c_int, [C.c_int, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "mpg_jacobi_build": (C.c_int, [C.c_int, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mpg_poly_apply": (C.c_int, [C.c_int, _i64, _vp, _vp, _vp, C.POINTER(PolyOp), _i32, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp]),
    "mpg_state_bytes": (_i64, [C.c_int, _i32]),
    "mpg_state_offset": (_i64, [C.c_int, _i32, _i32]),
    "mpg_cycle_start": (C.c_int, [C.c_int, _i64, _i64, _i32, _vp, _vp, _vp, _d, _d, _d, _i32, _vp, _vp]),
    "mpg_arnoldi_step": (C.c_int, [C.c_int, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "mpg_cycle_finish": (C.c_int, [C.c_int, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "mpg_solver_create": (C.c_int, [C.POINTER(SolverDesc), C.POINTER(C.c_void_p)]),
    "mpg_solver_destroy": (C.c_int, [_vp]),
    "mpg_solver_begin": (C.c_int, [_vp, _vp]),
    "mpg_solver_cycle": (C.c_int, [_vp, _i32, _vp]),
    "mpg_solver_profile_cycle": (C.c_int, [_vp, _i32, _vp, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
}
PROFILE_CLASSES = ("start", "precond", "spmv_dot1", "update_dot", "update_norm_givens",
                   "scale", "finish", "residual", "dot1", "step")
# with K_A split "spmv_dot1" times the SpMV alone and "dot1" the pass-1 dots; "step" is the
# persistent per-step kernel (stencil storage, no preconditioner; MPG_MEGA=0 disables it)

_LIB = None
_ERR: str | None = None


def header_symbols() -> list[str]:
    """Every function the public header declares (used by the symbol test)."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(mpg_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load the library (once).  Raises ExtensionMissingError if unavailable."""
    global _LIB, _ERR
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissingError(
            f"{LIB_PATH} is not built; run `python -m paper_2109_01232_b200.build`")
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover
        raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise on a non-zero status."""
    rc = getattr(load(), name)(*args)
    if rc != 0:
        kind = {-1: "invalid argument", -2: "unsupported configuration",
                -3: "invalid solver handle"}.get(rc, f"CUDA error {rc}")
        raise CudaCallError(f"{name} failed: {kind}")


def launch_count() -> int:
    return int(load().mpg_launch_count())
