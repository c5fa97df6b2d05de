"""Right preconditioners: GMRES polynomial and block Jacobi, on the device.

Mirrors the reference's ``mpgmres.precond`` (pkg/src/mpgmres/precond.py):

* ``PolynomialPreconditioner`` / ``PolyBasis``   precond.py:58-91
* ``build_poly_precond``   precond.py:148-192 — degree+1 Arnoldi steps run on
  the device (ArnoldiWorkspace + fused CGS2 step); the (degree+1)-sized
  Hessenberg post-processing (power coefficients, harmonic Ritz values,
  Leja order; precond.py:195-269) stays on the host, as in the reference.
* ``apply_poly``           precond.py:272-319 — the polynomial is lowered to a
  short op program (``poly_program``) whose SpMV steps carry their axpy
  epilogues (Horner, Newton real root, conjugate pair), issuing exactly
  ``degree`` SpMV launches.
* ``BlockJacobiPreconditioner`` / ``build_block_jacobi`` / ``apply_block_jacobi``
  precond.py:94-110, 326-390 — block extraction and pivoted LU on the device.
* ``cast_apply``           precond.py:393-414.

Reference preconditioner objects (duck-typed) are accepted everywhere.
RCM reordering (precond.py:421-515) is host preprocessing; it lives in
``paper_2109_01232_b200.io.rcm_reorder``.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass
from enum import Enum

import numpy as np
import scipy.linalg
import torch

from . import _lib
from .core import (FP32, FP64, CsrMatrix, Precision, PrecisionError, ShapeError, convert_matrix,
                   ctx, device, dvec, norm2, ptr, stream_handle, to_device, to_host)
from .krylov import ArnoldiWorkspace, arnoldi_step, solve_least_squares

__all__ = ["PolyBasis", "PolynomialPreconditioner", "BlockJacobiPreconditioner",
           "SingularBlockError", "build_poly_precond", "apply_poly", "build_block_jacobi",
           "apply_block_jacobi", "cast_apply", "poly_program"]

POWER_DEGREE_LIMIT = 10


class SingularBlockError(np.linalg.LinAlgError):
    """A diagonal block has no LU factorization."""


class PolyBasis(Enum):
    POWER = "power"
    NEWTON_ROOTS = "newton-roots"


@dataclass(frozen=True)
class PolynomialPreconditioner:
    degree: int
    basis: PolyBasis
    precision: Precision
    coefficients: np.ndarray | None = None
    roots: np.ndarray | None = None

    def __post_init__(self) -> None:
        if self.basis is PolyBasis.POWER:
            if self.coefficients is None or len(self.coefficients) != self.degree + 1:
                raise ValueError("power basis needs degree + 1 coefficients")
            if not np.all(np.isfinite(self.coefficients)):
                raise ValueError("polynomial coefficients are not finite")
        else:
            if self.roots is None or len(self.roots) != self.degree + 1:
                raise ValueError("root basis needs degree + 1 roots")
            if not np.all(np.isfinite(self.roots)) or np.any(self.roots == 0):
                raise ValueError("polynomial roots must be finite and nonzero")


@dataclass(frozen=True)
class BlockJacobiPreconditioner:
    """LU factors of the diagonal blocks, held on the device."""

    block_size: int
    n: int
    precision: Precision
    block_lu: torch.Tensor | np.ndarray   # (n_blocks, k, k)
    block_piv: torch.Tensor | np.ndarray  # (n_blocks, k)

    @property
    def n_blocks(self) -> int:
        return int(self.block_lu.shape[0])


# ---------------------------------------------------------------------------
# duck typing of reference objects

def precision_of(M) -> Precision:
    p = getattr(M, "precision", None)
    if isinstance(p, Precision):
        return p
    if p is None and hasattr(M, "dtype"):       # oracle objects carry a numpy dtype
        return Precision.of(np.zeros(0, dtype=M.dtype))
    val = getattr(p, "value", p)
    if val == "fp32":
        return FP32
    if val == "fp64":
        return FP64
    raise PrecisionError(f"cannot read the precision of {type(M).__name__}")


def is_poly(M) -> bool:
    return hasattr(M, "degree") and hasattr(M, "basis")


def is_jacobi(M) -> bool:
    return hasattr(M, "block_lu") and hasattr(M, "block_piv")


def _basis_name(M) -> str:
    return getattr(M.basis, "value", str(M.basis))


# ---------------------------------------------------------------------------
# polynomial: lowering to a device op program

def poly_program(M, dt=None) -> list[tuple]:
    """Lower a polynomial preconditioner to (op, src, dst, x2, a, b) steps.

    Buffer ids: 0 = x (input, never written), 1 = y (output), 2..4 scratch.
    Scalars are rounded to the working precision exactly as numpy does in
    precond.py:286-319, then carried as doubles.
    """
    T = (precision_of(M).dtype if dt is None else np.dtype(dt)).type
    ops: list[tuple] = []
    if _basis_name(M) == "power":
        c = np.asarray(M.coefficients)
        d = int(M.degree)
        cur = 1 if d % 2 == 0 else 2
        ops.append((_lib.POLY_SCALE, 0, cur, 0, float(T(c[d])), 0.0))   # y = c[d] * x
        for i in range(d - 1, -1, -1):                                 # y = A y + c[i] x
            nxt = 2 if cur == 1 else 1
            ops.append((_lib.POLY_HORNER, cur, nxt, 0, float(T(c[i])), 0.0))
            cur = nxt
        return ops
    roots = np.asarray(M.roots, dtype=np.complex128)
    k = len(roots)
    ops.append((_lib.POLY_ZERO, 0, 1, 0, 0.0, 0.0))                    # y = 0
    cur, i = 0, 0
    while i < k:
        t = roots[i]
        if t.imag == 0:
            inv = float(T(1.0 / t.real))
            if i < k - 1:                      # y += inv p ; p <- p - inv A p
                nxt = 2 if cur != 2 else 3
                ops.append((_lib.POLY_NEWTON_REAL, cur, nxt, 0, inv, 0.0))
                cur = nxt
            else:                              # y += inv p
                ops.append((_lib.POLY_ACC, cur, 1, 0, inv, 0.0))
            i += 1
        else:
            mod2 = float(t.real ** 2 + t.imag ** 2)
            a = float(T(2.0 * t.real / mod2))
            b = float(T(1.0 / mod2))
            ops.append((_lib.POLY_PAIR1, cur, 4, 0, a, b))    # ap = A p ; y += a p - b ap
            if i < k - 2:                                     # p <- p - a ap + b A ap
                dst = cur if cur != 0 else 2
                ops.append((_lib.POLY_PAIR2, 4, dst, cur, a, b))
                cur = dst
            i += 2
    return ops


def poly_ops_struct(ops: list[tuple]):
    arr = (_lib.PolyOp * len(ops))()
    for i, (op, src, dst, x2, a, b) in enumerate(ops):
        arr[i] = _lib.PolyOp(op, src, dst, x2, a, b)
    return arr


def apply_poly(M, A, x):
    """p(A) x with exactly M.degree SpMV launches (precond.py:272-293)."""
    A = CsrMatrix.from_any(A)
    prec = precision_of(M)
    if A.precision is not prec:
        raise PrecisionError("matrix and preconditioner precisions differ")
    if Precision.of(x) is not prec:
        raise PrecisionError("operand precision differs from the preconditioner's")
    if tuple(x.shape) != (A.n_cols,):
        raise ShapeError("operand length does not match the matrix")
    host = not isinstance(x, torch.Tensor)
    n = A.n_rows
    xd = to_device(x)
    y, t0, t1, t2 = (dvec(n, prec) for _ in range(4))
    ops = poly_ops_struct(poly_program(M))
    _lib.call("mpg_poly_apply", prec.code, n, ptr(A.row_ptr), ptr(A.col_idx), ptr(A.values), ops,
              len(ops), ptr(xd), ptr(y), ptr(t0), ptr(t1), ptr(t2), ptr(ctx().ws), stream_handle())
    out = y[:n]
    return to_host(out) if host else out.clone()


def build_poly_precond(A, degree: int, seed: int = 0) -> PolynomialPreconditioner:
    """Residual-minimising polynomial from degree+1 device Arnoldi steps
    (precond.py:148-192).  The start vector is numpy's
    ``default_rng(seed).standard_normal(n)`` rounded to the matrix precision,
    exactly as the reference draws it."""
    from .spmv import spmv
    A = CsrMatrix.from_any(A)
    if A.n_rows != A.n_cols:
        raise ShapeError("polynomial preconditioner needs a square matrix")
    if degree < 0:
        raise ValueError("degree must be nonnegative")
    prec = A.precision
    steps = degree + 1
    v = np.random.default_rng(seed).standard_normal(A.n_rows).astype(prec.dtype)
    vd = to_device(v)
    gamma = norm2(vd)
    ws = ArnoldiWorkspace(A.n_rows, steps, prec)
    ws.start_from_residual(vd, 0.0, -1.0)
    for _ in range(steps):
        st = arnoldi_step(ws, lambda u: spmv(A, u))
        if st.breakdown:
            break
    k = ws.j
    if k < steps:
        warnings.warn(f"subspace became invariant after {k} steps; "
                      f"polynomial degree reduced from {degree} to {k - 1}", stacklevel=2)
    solve_least_squares(ws, k)
    y = ws.state.array("d", k)
    if not np.all(np.isfinite(y)):
        raise ValueError("polynomial construction produced non-finite coefficients")
    H = ws.hls.H
    built = k - 1
    if built <= POWER_DEGREE_LIMIT:
        coeffs = _power_coefficients(H, k, float(gamma), y)
        return PolynomialPreconditioner(built, PolyBasis.POWER, prec,
                                        coefficients=coeffs.astype(prec.dtype))
    roots = _leja_order(_harmonic_ritz_values(H, k))
    return PolynomialPreconditioner(built, PolyBasis.NEWTON_ROOTS, prec, roots=roots)


def _power_coefficients(H, k, gamma, y):
    """Monomial coefficients via s_{j+1} recurrence (precond.py:195-209)."""
    H64 = np.asarray(H)[: k + 1, :k].astype(np.float64)
    S = np.zeros((k, k))
    S[0, 0] = 1.0 / gamma
    for j in range(k - 1):
        shifted = np.zeros(k)
        shifted[1:] = S[j, :-1]
        S[j + 1] = (shifted - H64[: j + 1, j] @ S[: j + 1]) / H64[j + 1, j]
    return np.asarray(y, dtype=np.float64) @ S


def _harmonic_ritz_values(H, k):
    """Roots of the k-step residual polynomial (precond.py:212-227)."""
    Hk = np.asarray(H)[:k, :k].astype(np.float64)
    h2 = float(np.asarray(H)[k, k - 1]) ** 2
    e_k = np.zeros(k)
    e_k[-1] = 1.0
    try:
        f = scipy.linalg.solve(Hk.T, e_k)
    except scipy.linalg.LinAlgError as exc:
        raise ValueError("polynomial construction produced non-finite coefficients") from exc
    Mx = Hk.copy()
    Mx[:, -1] += h2 * f
    theta = np.linalg.eigvals(Mx)
    if not np.all(np.isfinite(theta)) or np.any(theta == 0):
        raise ValueError("polynomial construction produced non-finite coefficients")
    return theta


def _leja_order(roots):
    """Greedy Leja order, conjugate partners adjacent (precond.py:230-269)."""
    roots = np.asarray(roots, dtype=np.complex128)
    pending = list(range(len(roots)))
    order: list[int] = []

    def place(i):
        pending.remove(i)
        order.append(i)
        if roots[i].imag != 0:
            want = np.conj(roots[i])
            best, mate = math.inf, None
            for t in pending:
                if roots[t].imag != 0:
                    dd = abs(roots[t] - want)
                    if dd < best:
                        best, mate = dd, t
            if mate is not None:
                pending.remove(mate)
                order.append(mate)

    place(max(pending, key=lambda i: (abs(roots[i]), -i)))
    while pending:
        chosen = roots[order]
        scores = [(float(np.sum(np.log(np.maximum(np.abs(roots[t] - chosen), 1e-300)))), t)
                  for t in pending]
        best_v, best_i = -math.inf, None
        for v, t in scores:
            if v > best_v:
                best_v, best_i = v, t
        place(best_i)
    return roots[order]


# ---------------------------------------------------------------------------
# block Jacobi

def build_block_jacobi(A, block_size: int) -> BlockJacobiPreconditioner:
    """Factor the dense diagonal blocks on the device (precond.py:326-360)."""
    A = CsrMatrix.from_any(A)
    if A.n_rows != A.n_cols:
        raise ShapeError("block Jacobi needs a square matrix")
    if block_size < 1:
        raise ValueError("block size must be positive")
    n, k = A.n_rows, min(block_size, A.n_rows)
    nb = -(-n // k)
    prec = A.precision
    lu = torch.zeros(nb * k * k, dtype=prec.torch_dtype, device=device())
    piv = torch.zeros(nb * k, dtype=torch.int64, device=device())
    bad = torch.full((1,), -1, dtype=torch.int64, device=device())
    _lib.call("mpg_jacobi_build", prec.code, n, k, ptr(A.row_ptr), ptr(A.col_idx), ptr(A.values),
              ptr(lu), ptr(piv), ptr(bad), stream_handle())
    b = int(bad.item())
    if b >= 0:
        raise SingularBlockError(f"diagonal block {b} is singular")
    return BlockJacobiPreconditioner(k, n, prec, lu.view(nb, k, k), piv.view(nb, k))


def jacobi_device_arrays(M) -> tuple[torch.Tensor, torch.Tensor]:
    lu = to_device(np.asarray(M.block_lu) if not isinstance(M.block_lu, torch.Tensor) else M.block_lu)
    piv = M.block_piv
    piv = to_device(np.asarray(piv, dtype=np.int64)) if not isinstance(piv, torch.Tensor) else piv.to(torch.int64)
    return lu.reshape(-1).contiguous(), piv.reshape(-1).contiguous()


def apply_block_jacobi(M, x):
    """Block-diagonal solve (precond.py:363-390)."""
    prec = precision_of(M)
    if Precision.of(x) is not prec:
        raise PrecisionError("operand precision differs from the preconditioner's")
    if tuple(x.shape) != (M.n,):
        raise ShapeError("operand length does not match the preconditioner")
    host = not isinstance(x, torch.Tensor)
    lu, piv = jacobi_device_arrays(M)
    xd = to_device(x)
    y = torch.empty(M.n, dtype=prec.torch_dtype, device=xd.device)
    _lib.call("mpg_jacobi_apply", prec.code, M.n, int(M.block_size), ptr(lu), ptr(piv), ptr(xd),
              ptr(y), stream_handle())
    return to_host(y) if host else y


def cast_apply(M, A32, x):
    """fp32 preconditioner applied to an fp64 vector (precond.py:393-414)."""
    from .core import convert_vector
    if precision_of(M) is not FP32:
        raise PrecisionError("cast_apply requires an fp32 preconditioner")
    if Precision.of(x) is not FP64:
        raise PrecisionError("cast_apply expects an fp64 operand")
    x32 = convert_vector(x, FP32)
    if is_poly(M):
        if A32 is None:
            raise ValueError("polynomial cast_apply needs the fp32 matrix")
        y32 = apply_poly(M, A32, x32)
    elif is_jacobi(M):
        y32 = apply_block_jacobi(M, x32)
    else:
        raise TypeError(f"unsupported preconditioner type {type(M).__name__}")
    return convert_vector(y32, FP64)
