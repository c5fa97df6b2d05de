"""CPU ORACLE for the mixed-precision GMRES hot path — TEST INFRASTRUCTURE ONLY.

This module restates, on the CPU with numpy/scipy, the algorithm of the
reference package ``mpgmres`` (``/root/reference/pkg/src/mpgmres``) for the
hot path named in BASELINE.json: stencil assembly, CSR SpMV, CGS2 Arnoldi,
Givens least squares, the restart loop, GMRES-IR, GMRES-FD and the Jacobi /
polynomial preconditioner applications.  Every function cites the reference
``file:line`` it follows.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product package
``paper_2109_01232_b200`` never imports anything from ``oracle/``.

Pinning.  The oracle issues the same floating-point operations in the same
order as the reference (numpy ``add.reduceat`` SpMV, single-thread BLAS
``?gemv`` for the CGS2 passes, ``sqrt(dot)`` norms, numpy-scalar Givens), so
on the same machine it reproduces the reference bit for bit.
``tests/golden/make_golden.py`` records the reference's own outputs (run in
the build container, where ``/root/reference`` exists) into
``tests/golden/*.json|npz``; ``tests/test_oracle.py`` pins this module to
those fixtures and to the reference's golden iteration counts
(235 for Laplace2D(50), 1172/1200 for Laplace2D(100), ...).
"""

from __future__ import annotations

import math
import time
import warnings
from contextlib import contextmanager
from typing import Callable, NamedTuple

import numpy as np
import scipy.linalg
import scipy.linalg.blas as _blas

try:  # the reference pins BLAS to one thread inside every solve (core.py:51-67)
    from threadpoolctl import threadpool_limits as _tp_limits
except ImportError:  # pragma: no cover
    _tp_limits = None

F32 = np.dtype(np.float32)
F64 = np.dtype(np.float64)
UNIT_ROUNDOFF = {F32: 2.0 ** -24, F64: 2.0 ** -53}          # core.py:98-101
BREAKDOWN_FACTOR = 10.0                                      # krylov.py:32
LOSS_FACTOR = 10.0                                           # solvers.py:51
STALL_IMPROVEMENT, STALL_RESTARTS = 0.01, 2                  # solvers.py:55-56
POWER_DEGREE_LIMIT = 10                                      # precond.py:55

_BLAS_THREADS = 1


@contextmanager
def blas_threads(n: int | None):
    """Scope the BLAS thread count (reference: ``deterministic_kernels``,
    core.py:51-67, always 1).  ``None`` keeps the library default."""
    if _tp_limits is None or n is None:
        yield
        return
    with _tp_limits(limits=n, user_api="blas"):
        yield


class Csr(NamedTuple):
    """Canonical CSR (reference ``CsrMatrix``, core.py:123-199)."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray   # int32[n_rows + 1]
    col_idx: np.ndarray   # int32[nnz]
    values: np.ndarray    # float32 | float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def astype(self, dt) -> "Csr":
        """Narrow/widen values, pattern shared (core.py:275-289)."""
        return Csr(self.n_rows, self.n_cols, self.row_ptr, self.col_idx,
                   self.values.astype(dt))

    def dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), dtype=self.values.dtype)
        r = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        out[r, self.col_idx] = self.values
        return out


def csr_from_dense(a) -> Csr:
    a = np.asarray(a)
    if a.dtype not in (F32, F64):
        a = a.astype(np.float64)
    r, c = np.nonzero(a)
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=a.shape[0]))])
    return Csr(a.shape[0], a.shape[1], ptr.astype(np.int32), c.astype(np.int32),
               np.ascontiguousarray(a[r, c]))


# ---------------------------------------------------------------------------
# stencil assembly, generated row by row (no sort).  Restates gen.py:129-202
# (+ the lexsort canonicalisation of core.py:229-249): within a row the
# entries come out in ascending column order because the offsets are visited
# in ascending ``dz*nx*nx + dy*nx + dx`` order.

_TABLE_2D = {  # gen.py:67-80, offset (dx, dy) -> coefficient
    "laplace2d": {(0, 0): 4.0, (-1, 0): -1.0, (1, 0): -1.0, (0, -1): -1.0, (0, 1): -1.0},
    "star2d": {(0, 0): 8.0, (-1, 0): -1.0, (1, 0): -1.0, (0, -1): -1.0, (0, 1): -1.0,
               (-1, -1): -1.0, (1, -1): -1.0, (-1, 1): -1.0, (1, 1): -1.0},
    "biharmonic2d": {(0, 0): 20.0, (-1, 0): -8.0, (1, 0): -8.0, (0, -1): -8.0,
                     (0, 1): -8.0, (-1, -1): 2.0, (1, -1): 2.0, (-1, 1): 2.0,
                     (1, 1): 2.0, (-2, 0): 1.0, (2, 0): 1.0, (0, -2): 1.0, (0, 2): 1.0},
}
KINDS = ("laplace2d", "laplace3d", "convdiff2d", "stretched2d", "biharmonic2d",
         "star2d", "recirc2d")


def stencil_size(kind: str, nx: int) -> tuple[int, int]:
    """(n, nnz) without materialising (gen.py:111-126)."""
    if kind == "laplace3d":
        offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    else:
        offs = list(_TABLE_2D.get(kind, _TABLE_2D["laplace2d"]))
    nnz = sum(math.prod(nx - abs(d) for d in o) for o in offs)
    return nx ** (3 if kind == "laplace3d" else 2), nnz


def _row_entries(kind, nx, rows, convection, stretch):
    """Per-row candidate entries: list of (col_offset, keep_mask, value_array)
    in ascending column order, for the global row indices ``rows``."""
    rows = np.asarray(rows, dtype=np.int64)
    out = []
    if kind == "laplace3d":                                   # gen.py:184-202
        ix, iy, iz = rows % nx, (rows // nx) % nx, rows // (nx * nx)
        for dx, dy, dz, v in ((0, 0, -1, -1.0), (0, -1, 0, -1.0), (-1, 0, 0, -1.0),
                              (0, 0, 0, 6.0), (1, 0, 0, -1.0), (0, 1, 0, -1.0),
                              (0, 0, 1, -1.0)):
            keep = ((ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < nx)
                    & (iz + dz >= 0) & (iz + dz < nx))
            out.append(((dz * nx + dy) * nx + dx, keep, np.full(rows.shape, v)))
        return out
    ix, iy = rows % nx, rows // nx
    if kind in ("convdiff2d", "recirc2d"):                    # gen.py:146-169
        h = 1.0 / (nx + 1)
        xh = 2.0 * (ix + 1) * h - 1.0
        yh = 2.0 * (iy + 1) * h - 1.0
        c = convection
        if kind == "convdiff2d":                              # gen.py:139-140
            cx, cy = np.full_like(xh, c), np.zeros_like(yh)
        else:                                                 # gen.py:141-142
            cx = c * 2.0 * yh * (1.0 - xh ** 2)
            cy = -c * 2.0 * xh * (1.0 - yh ** 2)
        ddx, ddy = cx * (h / 2.0), cy * (h / 2.0)
        coeff = {(0, -1): -1.0 - ddy, (-1, 0): -1.0 - ddx, (0, 0): np.full(rows.shape, 4.0),
                 (1, 0): -1.0 + ddx, (0, 1): -1.0 + ddy}
    elif kind == "stretched2d":                               # gen.py:159-163
        s = stretch
        coeff = {(0, -1): -s, (-1, 0): -1.0, (0, 0): 2.0 + 2.0 * s, (1, 0): -1.0, (0, 1): -s}
    else:
        coeff = _TABLE_2D[kind]
    for (dx, dy) in sorted(coeff, key=lambda o: o[1] * nx + o[0]):
        keep = (ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < nx)
        val = np.broadcast_to(np.asarray(coeff[(dx, dy)], dtype=np.float64), rows.shape)
        out.append((dy * nx + dx, keep, val))
    return out


def stencil_csr(kind: str, nx: int, convection: float = 1.0, stretch: float = 1.0e4,
                row_begin: int = 0, row_end: int | None = None) -> Csr:
    """fp64 canonical CSR of rows [row_begin, row_end) with global columns.
    For the full range this equals ``mpgmres.gen.generate`` bit for bit."""
    if kind not in KINDS:
        raise ValueError(f"unknown stencil kind {kind!r}")
    n, _ = stencil_size(kind, nx)
    row_end = n if row_end is None else row_end
    rows = np.arange(row_begin, row_end, dtype=np.int64)
    ents = _row_entries(kind, nx, rows, convection, stretch)
    keep = np.stack([e[1] for e in ents], axis=1)
    cols = np.stack([rows + e[0] for e in ents], axis=1)
    vals = np.stack([np.asarray(e[2], dtype=np.float64) for e in ents], axis=1)
    ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=ptr[1:])
    if row_begin:  # global row_ptr offsets for a partition slice
        _, before = _nnz_before(kind, nx, row_begin, convection, stretch)
        ptr += before
    return Csr(len(rows), n, ptr.astype(np.int32), cols[keep].astype(np.int32),
               np.ascontiguousarray(vals[keep]))


def _nnz_before(kind, nx, row, convection, stretch):
    """Number of stored entries in rows [0, row) (brute force, small nx)."""
    if row == 0:
        return 0, 0
    ents = _row_entries(kind, nx, np.arange(row), convection, stretch)
    return row, int(sum(int(e[1].sum()) for e in ents))


def ones_rhs(n: int) -> np.ndarray:
    return np.ones(n, dtype=np.float64)                      # gen.py:207-208


def row_partition(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks [floor(r n / P), floor((r+1) n / P)).
    The reference is single-process; this is the restatement the device
    partitioner is checked against."""
    return [((r * n) // world, ((r + 1) * n) // world) for r in range(world)]


# ---------------------------------------------------------------------------
# dense/sparse kernels with the reference's exact operation order

def spmv(A: Csr, x: np.ndarray) -> np.ndarray:
    """y = A x: products rounded, each row reduced by numpy add.reduceat
    (spmv.py:48-72).  Empty rows give 0."""
    if x.dtype != A.values.dtype or x.shape != (A.n_cols,):
        raise ValueError("spmv operand mismatch")
    if A.nnz == 0:
        return np.zeros(A.n_rows, dtype=A.values.dtype)
    prod = A.values * x[A.col_idx]
    cnt = np.diff(A.row_ptr)
    if cnt.min() > 0:
        return np.add.reduceat(prod, A.row_ptr[:-1])
    y = np.zeros(A.n_rows, dtype=A.values.dtype)
    nz = cnt > 0
    y[nz] = np.add.reduceat(prod, A.row_ptr[:-1][nz])
    return y


_GEMV_FN = {F32: _blas.sgemv, F64: _blas.dgemv}


def basis_dots(V: np.ndarray, w: np.ndarray) -> np.ndarray:
    """c = V^T w with V a Fortran-ordered column block (core.py:326-336, trans)."""
    return _GEMV_FN[V.dtype](1.0, V, w, trans=1)


def basis_update(V: np.ndarray, c: np.ndarray, w: np.ndarray) -> np.ndarray:
    """w <- w - V c in place (core.py:333-336, alpha=-1, beta=1, no trans)."""
    return _GEMV_FN[V.dtype](-1.0, V, c, beta=1.0, y=w, trans=0, overwrite_y=1)


def basis_combine(V: np.ndarray, d: np.ndarray) -> np.ndarray:
    """u = V d (solvers.py:171)."""
    if V.shape[1] == 0:
        return np.zeros(V.shape[0], dtype=V.dtype)
    return _GEMV_FN[V.dtype](1.0, V, d, trans=0)


def nrm2(x: np.ndarray) -> float:
    """sqrt(dot(x, x)) in x's precision, as a Python float (core.py:341-354)."""
    if x.size == 0:
        return 0.0
    return float(np.sqrt(np.dot(x, x)))


def narrow(x: np.ndarray, dt) -> np.ndarray:
    """convert_vector (core.py:252-272): round to nearest; overflow raises."""
    dt = np.dtype(dt)
    if x.dtype == dt:
        return x.copy()
    with np.errstate(over="ignore"):
        y = x.astype(dt)
    if dt == F32:
        bad = np.isinf(y) & np.isfinite(x)
        if bad.any():
            raise OverflowError(f"entry {int(np.argmax(bad))} overflows fp32")
    return y


# ---------------------------------------------------------------------------
# Arnoldi (CGS2) + Givens least squares  (krylov.py:43-202)

class DivergenceError(ArithmeticError):
    pass


class ArnoldiState:
    """Basis V (n x (m+1), F order) plus the rotated Hessenberg system."""

    def __init__(self, n: int, m: int, dt, breakdown_tol: float | None = None):
        dt = np.dtype(dt)
        self.dt, self.m, self.j = dt, m, 0
        self.V = np.zeros((n, m + 1), dtype=dt, order="F")
        self.H = np.zeros((m + 1, m), dtype=dt)
        self.R = np.zeros((m + 1, m), dtype=dt)
        self.cs = np.zeros(m, dtype=dt)
        self.sn = np.zeros(m, dtype=dt)
        self.g = np.zeros(m + 1, dtype=dt)
        self.broke = False
        self.tol = BREAKDOWN_FACTOR * UNIT_ROUNDOFF[dt] if breakdown_tol is None \
            else breakdown_tol

    def begin(self, v0: np.ndarray, gamma: float) -> None:      # krylov.py:96-100,62-68
        self.V[:, 0] = v0
        self.j, self.broke = 0, False
        for a in (self.H, self.R, self.cs, self.sn, self.g):
            a[:] = 0
        self.g[0] = gamma

    def step(self, op: Callable[[np.ndarray], np.ndarray]):
        """One CGS2 Arnoldi step (krylov.py:112-151). Returns (h, h_sub, breakdown)."""
        j = self.j
        w = np.asarray(op(self.V[:, j]))
        if w.dtype != self.dt or w.shape != (self.V.shape[0],):
            raise ValueError("operator changed shape or precision")
        if not np.all(np.isfinite(w)):
            raise DivergenceError("operator output contains non-finite values")
        w0 = nrm2(w)
        Vk = self.V[:, : j + 1]
        h = np.zeros(j + 1, dtype=self.dt)
        for _ in (0, 1):                       # exactly two classical GS passes
            c = basis_dots(Vk, w)
            w = basis_update(Vk, c, w)
            h += c
        hs = nrm2(w)
        self.H[: j + 1, j] = h
        self.H[j + 1, j] = hs
        brk = hs <= self.tol * w0
        if not brk:
            self.V[:, j + 1] = w / hs
        self.broke = brk
        self.j += 1
        return h, hs, brk

    def rotate(self, j: int) -> float:
        """Fold column j into the rotated system (krylov.py:154-187)."""
        col = self.H[: j + 2, j].copy()
        cs, sn = self.cs, self.sn
        for i in range(j):
            top = cs[i] * col[i] + sn[i] * col[i + 1]
            col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
            col[i] = top
        a, b = col[j], col[j + 1]
        r = np.hypot(a, b)
        if r == 0:
            cs[j], sn[j] = 1.0, 0.0
            self.R[: j + 2, j] = col
            return float(abs(self.g[j]))
        c, s = a / r, b / r
        cs[j], sn[j] = c, s
        col[j] = c * a + s * b
        col[j + 1] = 0
        self.R[: j + 2, j] = col
        g = self.g
        top = c * g[j] + s * g[j + 1]
        g[j + 1] = -s * g[j] + c * g[j + 1]
        g[j] = top
        return float(abs(g[j + 1]))

    def coefficients(self, k: int) -> np.ndarray:
        """Back-solve R[:k,:k] d = g[:k] (krylov.py:190-202)."""
        if k == 0:
            return np.zeros(0, dtype=self.dt)
        Rk = self.R[:k, :k]
        dg = np.abs(np.diag(Rk))
        if np.any(dg == 0) or not np.all(np.isfinite(dg)):
            raise np.linalg.LinAlgError("zero diagonal in triangular factor")
        return scipy.linalg.solve_triangular(Rk, self.g[:k], lower=False)


class Cycle(NamedTuple):
    x: np.ndarray
    implicit: list
    steps: int
    breakdown: bool


def cycle(apply_a, b, x0, m, rtol, *, m_inv=None, b_norm=None, r0=None,
          breakdown_tol=None) -> Cycle:
    """One restart cycle (solvers.py:122-174)."""
    if b_norm is None:
        b_norm = nrm2(b)
    if r0 is None:
        r0 = b - apply_a(x0)
    gamma = nrm2(r0)
    if gamma == 0.0:
        return Cycle(x0.copy(), [], 0, False)
    if not np.isfinite(gamma):
        raise DivergenceError("initial residual is not finite")
    op = apply_a if m_inv is None else (lambda v: apply_a(m_inv(v)))
    st = ArnoldiState(b.shape[0], m, b.dtype, breakdown_tol)
    st.begin(r0 / gamma, gamma)
    imp, brk, thr = [], False, rtol * b_norm
    while st.j < m:
        _, _, bd = st.step(op)
        res = st.rotate(st.j - 1)
        imp.append(res)
        if bd:
            brk = True
            break
        if res <= thr:
            break
    k = st.j
    u = basis_combine(st.V[:, :k], st.coefficients(k))
    if m_inv is not None:
        u = m_inv(u)
    return Cycle(x0 + u, imp, k, brk)


def residual(A: Csr, b, x):
    """(||b - A x||, b - A x) in A's precision (solvers.py:443-453)."""
    r = b - spmv(A, x)
    return nrm2(r), r


class Report(NamedTuple):
    """Mirror of SolveReport (solvers.py:83-106); history entries are
    (iteration, implicit, explicit|None, phase)."""
    x: np.ndarray
    converged: bool
    total_iters: int
    iters_fp32: int
    iters_fp64: int
    history: list
    loss_of_accuracy: bool
    stalled_at: int | None
    total_time: float


def _rel(v, s):
    if s > 0.0:
        return v / s
    return 0.0 if v == 0.0 else float("inf")


def restart_loop(A: Csr, b, x, rtol, m, max_iters, m_inv, phase, hist,
                 offset=0, limit=None, stop_on_stall=False):
    """Restart loop (solvers.py:177-227)."""
    apply_a = lambda v: spmv(A, v)
    bn = nrm2(b)
    rn, r = residual(A, b, x)
    rel = _rel(rn, bn)
    hist.append((offset, rel, rel, phase))
    limit = max_iters if limit is None else limit
    total, conv, loss, stalled, run, prev = 0, rel <= rtol, False, None, 0, rel
    while not conv and not loss and total < limit:
        cy = cycle(apply_a, b, x, min(m, limit - total), rtol, m_inv=m_inv,
                   b_norm=bn, r0=r)
        x = cy.x
        for i, res in enumerate(cy.implicit[:-1]):
            hist.append((offset + total + i + 1, _rel(res, bn), None, phase))
        total += cy.steps
        rn, r = residual(A, b, x)
        rel = _rel(rn, bn)
        irel = _rel(cy.implicit[-1], bn) if cy.implicit else rel
        hist.append((offset + total, irel, rel, phase))
        if rel <= rtol:
            conv = True
        elif irel <= rtol and rel > LOSS_FACTOR * rtol:
            loss = True
        if not conv:
            run = run + 1 if (prev > 0 and (prev - rel) < STALL_IMPROVEMENT * prev) else 0
            if run >= STALL_RESTARTS:
                if stalled is None:
                    stalled = offset + total
                if stop_on_stall:
                    break
            prev = rel
    return x, conv, total, loss, stalled


def _precond_fn(M, A: Csr, dt):
    """Right-preconditioner closure (solvers.py:230-244, precond.py:393-414)."""
    if M is None:
        return None
    if M.dtype == np.dtype(dt):
        return (lambda v: poly_apply(M, A, v)) if isinstance(M, Poly) else \
            (lambda v: jacobi_apply(M, v))
    if M.dtype == F32 and np.dtype(dt) == F64:
        A32 = A.astype(np.float32) if isinstance(M, Poly) else None

        def cast(v):
            v32 = narrow(v, F32)
            y = poly_apply(M, A32, v32) if isinstance(M, Poly) else jacobi_apply(M, v32)
            return y.astype(np.float64)
        return cast
    raise TypeError("an fp64 preconditioner cannot run inside an fp32 solve")


def solve_restarted(A: Csr, b, x0=None, rtol=1e-10, m=50, max_iters=100_000,
                    precond=None, dtype=None, stop_on_stall=False,
                    threads=_BLAS_THREADS) -> Report:
    """Restarted GMRES in one precision (solvers.py:251-294)."""
    dt = np.dtype(dtype) if dtype is not None else A.values.dtype
    if A.values.dtype != dt:
        A = A.astype(dt)
    b = narrow(np.asarray(b), dt) if np.asarray(b).dtype != dt else np.asarray(b)
    x = np.zeros(A.n_cols, dtype=dt) if x0 is None else np.asarray(x0)
    if x.dtype != dt:
        x = narrow(x, dt)
    mi = _precond_fn(precond, A, dt)
    hist: list = []
    phase = "fp32" if dt == F32 else "fp64"
    t0 = time.perf_counter()
    with blas_threads(threads):
        x, conv, tot, loss, st = restart_loop(A, b, x, rtol, m, max_iters, mi,
                                              phase, hist, stop_on_stall=stop_on_stall)
    el = time.perf_counter() - t0
    f32 = dt == F32
    return Report(x.astype(np.float64) if f32 else x, conv, tot, tot if f32 else 0,
                  0 if f32 else tot, hist, loss, st, el)


def solve_ir(A: Csr, b, x0=None, rtol=1e-10, m=50, max_iters=100_000,
             precond32=None, threads=_BLAS_THREADS) -> Report:
    """GMRES-IR: fp32 correction cycles, fp64 residual (solvers.py:297-384)."""
    if A.values.dtype != F64 or np.asarray(b).dtype != F64:
        raise TypeError("iterative refinement expects fp64 A and b")
    x = np.zeros(A.n_cols) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    A32 = A.astype(np.float32)
    mi = _precond_fn(precond32, A32, F32)
    apply32 = lambda v: spmv(A32, v)
    zero32 = np.zeros(A.n_cols, dtype=np.float32)
    hist: list = []
    t0 = time.perf_counter()
    with blas_threads(threads):
        bn = nrm2(b)
        rn, r = residual(A, b, x)
        rel = _rel(rn, bn)
        hist.append((0, rel, rel, "fp32"))
        total, conv, stalled, run, prev = 0, rel <= rtol, None, 0, rel
        while not conv and total < max_iters:
            rho = rn
            r32 = narrow(r / rho, F32)
            cy = cycle(apply32, r32, zero32, min(m, max_iters - total), rtol,
                       m_inv=mi, r0=r32)
            if not np.all(np.isfinite(cy.x)):
                raise DivergenceError("fp32 correction is not finite")
            sc = rho / bn if bn > 0 else 1.0
            for i, res in enumerate(cy.implicit[:-1]):
                hist.append((total + i + 1, res * sc, None, "fp32"))
            x = x + rho * cy.x.astype(np.float64)
            rn, r = residual(A, b, x)
            total += cy.steps
            rel = _rel(rn, bn)
            irel = cy.implicit[-1] * sc if cy.implicit else rel
            hist.append((total, irel, rel, "fp32"))
            conv = rel <= rtol
            if not conv:
                run = run + 1 if (prev > 0 and (prev - rel) < STALL_IMPROVEMENT * prev) else 0
                if run >= STALL_RESTARTS and stalled is None:
                    stalled = total
                prev = rel
    el = time.perf_counter() - t0
    return Report(x, conv, total, total, 0, hist, False, stalled, el)


def solve_fd(A: Csr, b, x0=None, rtol=1e-10, m=50, max_iters=100_000,
             switch_iter=0, threads=_BLAS_THREADS) -> Report:
    """fp32 leg up to switch_iter (or stall), then fp64 (solvers.py:387-440)."""
    if switch_iter < 0 or switch_iter % m:
        raise ValueError("switch_iter must be a nonnegative multiple of m")
    x = np.zeros(A.n_cols) if x0 is None else np.asarray(x0, dtype=np.float64)
    hist: list = []
    n32, loss32, stalled = 0, False, None
    t0 = time.perf_counter()
    with blas_threads(threads):
        if switch_iter > 0:
            A32 = A.astype(np.float32)
            x32, _, n32, loss32, stalled = restart_loop(
                A32, narrow(np.asarray(b), F32), narrow(x, F32), rtol, m, max_iters,
                None, "fp32", hist, 0, min(switch_iter, max_iters), True)
            x = x32.astype(np.float64)
            if hist and hist[-1][0] == n32:
                hist.pop()
        x, conv, n64, loss64, st64 = restart_loop(
            A, np.asarray(b), x, rtol, m, max_iters, None, "fp64", hist,
            n32, max(max_iters - n32, 0))
    el = time.perf_counter() - t0
    return Report(x, conv, n32 + n64, n32, n64, hist, loss32 or loss64,
                  stalled if stalled is not None else st64, el)


# ---------------------------------------------------------------------------
# preconditioners (precond.py:65-414)

class Poly(NamedTuple):
    degree: int
    basis: str                 # "power" | "newton-roots"
    dtype: np.dtype
    coefficients: np.ndarray | None
    roots: np.ndarray | None


class Jacobi(NamedTuple):
    block_size: int
    n: int
    dtype: np.dtype
    block_lu: np.ndarray             # (nb, k, k)
    block_piv: np.ndarray            # (nb, k)


def poly_build(A: Csr, degree: int, seed: int = 0, threads=_BLAS_THREADS) -> Poly:
    """Residual-minimising polynomial from degree+1 Arnoldi steps
    (precond.py:148-192)."""
    dt = A.values.dtype
    steps = degree + 1
    v = np.random.default_rng(seed).standard_normal(A.n_rows).astype(dt)
    gamma = nrm2(v)
    st = ArnoldiState(A.n_rows, steps, dt)
    st.begin(v / gamma, gamma)
    with blas_threads(threads):
        for j in range(steps):
            _, _, bd = st.step(lambda u: spmv(A, u))
            st.rotate(j)
            if bd:
                break
    k = st.j
    if k < steps:
        warnings.warn(f"subspace became invariant after {k} steps; polynomial "
                      f"degree reduced from {degree} to {k - 1}", stacklevel=2)
    y = st.coefficients(k)
    if not np.all(np.isfinite(y)):
        raise ValueError("non-finite polynomial coefficients")
    d = k - 1
    if d <= POWER_DEGREE_LIMIT:
        return Poly(d, "power", dt, _monomials(st.H, k, float(gamma), y).astype(dt), None)
    return Poly(d, "newton-roots", dt, None, _leja(_harmonic_ritz(st.H, k)))


def _monomials(H, k, gamma, y):
    """precond.py:195-209."""
    H64 = H[: k + 1, :k].astype(np.float64)
    S = np.zeros((k, k))
    S[0, 0] = 1.0 / gamma
    for j in range(k - 1):
        sh = np.zeros(k)
        sh[1:] = S[j, :-1]
        S[j + 1] = (sh - H64[: j + 1, j] @ S[: j + 1]) / H64[j + 1, j]
    return y.astype(np.float64) @ S


def _harmonic_ritz(H, k):
    """precond.py:212-227."""
    Hk = H[:k, :k].astype(np.float64)
    h2 = float(H[k, k - 1]) ** 2
    ek = np.zeros(k)
    ek[-1] = 1.0
    f = scipy.linalg.solve(Hk.T, ek)
    M = Hk.copy()
    M[:, -1] += h2 * f
    th = np.linalg.eigvals(M)
    if not np.all(np.isfinite(th)) or np.any(th == 0):
        raise ValueError("non-finite polynomial roots")
    return th


def _leja(roots):
    """Greedy Leja order, conjugates adjacent, low-index tie break
    (precond.py:230-269)."""
    roots = np.asarray(roots, dtype=np.complex128)
    left = list(range(len(roots)))
    order: list[int] = []

    def take(i):
        left.remove(i)
        order.append(i)
        if roots[i].imag != 0:
            tgt, best, mate = np.conj(roots[i]), math.inf, None
            for t in left:
                if roots[t].imag == 0:
                    continue
                dd = abs(roots[t] - tgt)
                if dd < best:
                    mate, best = t, dd
            if mate is not None:
                left.remove(mate)
                order.append(mate)

    take(max(left, key=lambda i: (abs(roots[i]), -i)))
    while left:
        chosen = roots[order]
        bi, bv = None, -math.inf
        for t in left:
            v = float(np.sum(np.log(np.maximum(np.abs(roots[t] - chosen), 1e-300))))
            if v > bv:
                bi, bv = t, v
        take(bi)
    return roots[order]


def poly_apply(M: Poly, A: Csr, x: np.ndarray) -> np.ndarray:
    """p(A) x with exactly M.degree SpMVs (precond.py:272-319)."""
    if M.basis == "power":
        c = M.coefficients
        y = c[M.degree] * x
        for i in range(M.degree - 1, -1, -1):
            y = spmv(A, y)
            y += c[i] * x
        return y
    T = x.dtype.type
    th = M.roots
    y, p, i = np.zeros_like(x), x.copy(), 0
    while i < len(th):
        t = th[i]
        if t.imag == 0:
            inv = T(1.0 / t.real)
            y += inv * p
            if i < len(th) - 1:
                p = p - inv * spmv(A, p)
            i += 1
        else:
            mod2 = float(t.real ** 2 + t.imag ** 2)
            a, bb = T(2.0 * t.real / mod2), T(1.0 / mod2)
            ap = spmv(A, p)
            y += a * p - bb * ap
            if i < len(th) - 2:
                p = p - a * ap + bb * spmv(A, ap)
            i += 2
    return y


def jacobi_build(A: Csr, block_size: int) -> Jacobi:
    """LU-factored diagonal blocks (precond.py:326-360), vectorised extraction."""
    n, k = A.n_rows, min(block_size, A.n_rows)
    nb = -(-n // k)
    blocks = np.zeros((nb, k, k), dtype=A.values.dtype)
    rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
    cols = A.col_idx.astype(np.int64)
    inside = (cols // k) == (rows // k)
    blocks[rows[inside] // k, rows[inside] % k, cols[inside] % k] = A.values[inside]
    for i in range(n - (nb - 1) * k, k):
        blocks[-1, i, i] = 1.0
    lus = np.empty_like(blocks)
    pivs = np.empty((nb, k), dtype=np.int64)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", scipy.linalg.LinAlgWarning)
        for bi in range(nb):
            lu, pv = scipy.linalg.lu_factor(blocks[bi], check_finite=False)
            dg = np.diag(lu)
            if np.any(dg == 0) or not np.all(np.isfinite(dg)):
                raise np.linalg.LinAlgError(f"diagonal block {bi} is singular")
            lus[bi], pivs[bi] = lu, pv
    return Jacobi(k, n, A.values.dtype, lus, pivs)


def jacobi_apply(M: Jacobi, x: np.ndarray) -> np.ndarray:
    """Batched block LU solves (precond.py:363-390)."""
    nb, k = M.block_lu.shape[:2]
    xb = np.zeros((nb, k), dtype=x.dtype)
    xb.reshape(-1)[: M.n] = x
    rr = np.arange(nb)
    for i in range(k):
        j = M.block_piv[:, i]
        vi = xb[rr, i].copy()
        xb[rr, i] = xb[rr, j]
        xb[rr, j] = vi
    for i in range(1, k):
        xb[:, i] -= np.einsum("bt,bt->b", M.block_lu[:, i, :i], xb[:, :i])
    for i in range(k - 1, -1, -1):
        if i < k - 1:
            xb[:, i] -= np.einsum("bt,bt->b", M.block_lu[:, i, i + 1:], xb[:, i + 1:])
        xb[:, i] /= M.block_lu[:, i, i]
    return xb.reshape(-1)[: M.n].copy()
