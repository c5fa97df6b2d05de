"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares; host-side (no-GPU) entry points agree with the oracle."""

import ctypes as C
import os

import numpy as np
import pytest

from oracle import cpu_gmres as O
from paper_2109_01232_b200 import _lib


def test_library_exports_header_symbols():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib._SIGS)


def test_version_and_workspace():
    lib = _lib.load()
    assert b"sm_100a" in lib.mpg_version()
    assert lib.mpg_workspace_bytes() > 1 << 20


def test_solver_descriptor_layout_matches_binding():
    """The ctypes mirror of mpg_solver_desc has the C struct's size and field order."""
    lib = _lib.load()
    assert lib.mpg_solver_desc_bytes() == C.sizeof(_lib.SolverDesc)
    assert C.sizeof(_lib.StateHeader) == 8 * 4 + 8 * 16


def test_header_kernel_time_fields_and_exchange_box():
    """The state header carries the four kernel-time bins after the distributed
    raw-sum slot; the exchange box holds 3 x 8 x 72 values plus sequence words."""
    H = _lib.StateHeader
    assert H.reserved.offset + 8 == H.ktime_ns.offset
    assert H.ktime_ns.offset + 4 * 8 == H.kt_mark.offset
    assert H.kt_mark.offset + 8 == C.sizeof(H)
    lib = _lib.load()
    assert lib.mpg_xbox_bytes() >= 3 * 8 * 72 * 8 + 3 * 8 * 4 + 4
    assert _lib.SolverDesc.xbox.offset + 8 * C.sizeof(C.c_void_p) == C.sizeof(_lib.SolverDesc)


def test_state_layout_monotone():
    lib = _lib.load()
    for prec in (0, 1):
        for m in (1, 25, 50, 512):
            offs = [lib.mpg_state_offset(prec, m, w) for w in range(9)]
            assert all(o > 0 for o in offs)
            assert lib.mpg_state_bytes(prec, m) > max(offs)
            assert C.sizeof(_lib.StateHeader) <= lib.mpg_state_offset(prec, m, 8)
        assert lib.mpg_state_bytes(prec, 513) == -1


@pytest.mark.parametrize("kind", list(_lib.STENCIL_KIND))
def test_host_stencil_counts_match_oracle(kind):
    lib = _lib.load()
    for nx in (2, 3, 5, 13):
        n, nnz = C.c_int64(), C.c_int64()
        assert lib.mpg_stencil_counts(_lib.STENCIL_KIND[kind], nx, C.byref(n), C.byref(nnz)) == 0
        assert (n.value, nnz.value) == O.stencil_size(kind, nx)
        A = O.stencil_csr(kind, nx)
        for r in (0, 1, nx - 1, nx, n.value // 2, n.value - 1, n.value):
            assert lib.mpg_stencil_nnz_before(_lib.STENCIL_KIND[kind], nx, r) == A.row_ptr[r]


def test_cfg_sizes_without_materialising():
    lib = _lib.load()
    n, nnz = C.c_int64(), C.c_int64()
    lib.mpg_stencil_counts(1, 400, C.byref(n), C.byref(nnz))
    assert (n.value, nnz.value) == (64_000_000, 447_040_000)
    lib.mpg_stencil_counts(6, 1500, C.byref(n), C.byref(nnz))
    assert (n.value, nnz.value) == (2_250_000, 11_244_000)


def test_argument_errors_without_gpu():
    lib = _lib.load()
    assert lib.mpg_stencil_counts(99, 10, None, None) == _lib.load().mpg_stencil_counts(99, 10, None, None)
    assert lib.mpg_spmv(0, -1, None, None, None, None, None, None, None) == -1
    assert lib.mpg_solver_create(None, None) == -1


def test_poly_program_lowering_counts_spmvs():
    # exactly `degree` SpMV-bearing ops (precond.py:272-319, tests/test_precond.py:113-148)
    from paper_2109_01232_b200.precond import PolyBasis, PolynomialPreconditioner, poly_program
    from paper_2109_01232_b200.core import FP32, FP64
    spmv_ops = {_lib.POLY_HORNER, _lib.POLY_NEWTON_REAL, _lib.POLY_PAIR1, _lib.POLY_PAIR2}
    for d in (0, 1, 4, 10):
        M = PolynomialPreconditioner(d, PolyBasis.POWER, FP64, coefficients=np.arange(1.0, d + 2))
        assert sum(op[0] in spmv_ops for op in poly_program(M)) == d
        assert poly_program(M)[-1][2] == 1   # result lands in y
    roots = np.array([2.0, 1 + 1j, 1 - 1j, 3.0, 0.5 + 2j, 0.5 - 2j, 4.0])
    M = PolynomialPreconditioner(6, PolyBasis.NEWTON_ROOTS, FP32, roots=roots)
    prog = poly_program(M)
    assert sum(op[0] in spmv_ops for op in prog) == 6
    assert all(op[2] != 0 for op in prog)   # the input is never written
