"""Restarted GMRES drivers: fp64/fp32 GMRES(m), GMRES-IR and GMRES-FD.

Drop-in for the reference's ``mpgmres.solvers`` (pkg/src/mpgmres/solvers.py):
same entry points, arguments, report type, history semantics, stall and
loss-of-accuracy rules and exceptions.  What changes is where the work runs:
each restart cycle — start vector, m CGS2 Arnoldi steps with on-device
Givens rotations and a device-side early-exit flag, the back-solve, the
(preconditioned) solution update and the explicit residual — is enqueued by
the native driver (csrc/solver.cu, ``mpg_solver_cycle``) and replayed as a
CUDA graph.  The host reads one small record per cycle (state header +
implicit residuals) and runs the restart bookkeeping of
``_run_restarted`` (solvers.py:177-227) / ``gmres_ir`` (:297-384) on it.

Inputs may be the reference's numpy objects (uploaded once per call, x
returned as numpy) or device objects (CsrMatrix / CUDA tensors, x returned
as a CUDA tensor).
"""

from __future__ import annotations

import contextlib

import ctypes as C
from dataclasses import dataclass
from typing import Callable, NamedTuple

import numpy as np
import torch

from . import _lib, timing
from .core import (FP32, FP64, CsrMatrix, Precision, PrecisionError, PrecisionOverflowError,
                   ShapeError, convert_matrix, convert_vector, ctx, device, dvec, norm2,
                   padded_copy, padded_length, ptr, stream_handle, to_device, to_host)
from .krylov import (ArnoldiWorkspace, DeviceState, DivergenceError, SingularHessenbergError,
                     arnoldi_step, solve_least_squares)
from .precond import (apply_block_jacobi, apply_poly, cast_apply, is_jacobi, is_poly,
                      jacobi_device_arrays, poly_ops_struct, poly_program, precision_of)
from .spmv import spmv

__all__ = ["StopCriteria", "SolveReport", "HistoryEntry", "CycleResult", "DivergenceError",
           "gmres_cycle", "gmres_restarted", "gmres_ir", "gmres_fd", "explicit_residual"]

LOSS_OF_ACCURACY_FACTOR = 10.0   # solvers.py:51
STALL_IMPROVEMENT = 0.01         # solvers.py:55
STALL_RESTARTS = 2               # solvers.py:56
_ERROR_FLAGS = (_lib.FLAG_NONFINITE_OP | _lib.FLAG_NONFINITE_GAMMA | _lib.FLAG_SINGULAR |
                _lib.FLAG_OVERFLOW | _lib.FLAG_NONFINITE_X | _lib.FLAG_HALO_TIMEOUT)


@dataclass(frozen=True)
class StopCriteria:
    """rtol, iteration budget, restart length (solvers.py:59-73)."""

    rtol: float = 1e-10
    max_iters: int = 100_000
    m: int = 50

    def __post_init__(self) -> None:
        if not 0.0 < self.rtol < 1.0:
            raise ValueError(f"rtol must be in (0, 1), got {self.rtol}")
        if self.m < 1:
            raise ValueError("restart length must be at least 1")
        if self.max_iters < 1:
            raise ValueError("iteration budget must be at least 1")


class HistoryEntry(NamedTuple):
    iteration: int
    implicit: float
    explicit: float | None
    phase: str


@dataclass
class SolveReport:
    """Outcome of one solve (solvers.py:83-106)."""

    x: np.ndarray | torch.Tensor
    converged: bool
    total_iters: int
    iters_fp32: int
    iters_fp64: int
    residual_history: list[HistoryEntry]
    kernel_times: dict[str, float]
    loss_of_accuracy: bool
    stalled_at: int | None = None
    total_time: float = 0.0

    def best_explicit(self) -> float:
        vals = [e.explicit for e in self.residual_history if e.explicit is not None]
        return min(vals) if vals else float("inf")


class CycleResult(NamedTuple):
    x: np.ndarray | torch.Tensor
    implicit_norms: list[float]
    steps: int
    breakdown: bool


def _relative(value: float, scale: float) -> float:
    if scale > 0.0:
        return value / scale
    return 0.0 if value == 0.0 else float("inf")


# ---------------------------------------------------------------------------
# generic-operator cycle (solvers.py:122-174)

def gmres_cycle(apply_a: Callable, b, x0, m: int, rtol: float, *,
                m_inv: Callable | None = None, b_norm: float | None = None, r0=None,
                breakdown_tol: float | None = None) -> CycleResult:
    """One restart cycle for an arbitrary operator.  The operator is called in
    the caller's array type (numpy in -> numpy operator); every Arnoldi step
    after it (CGS2 + Givens) runs on the device."""
    host = not isinstance(b, torch.Tensor)
    if tuple(b.shape) != tuple(x0.shape):
        raise ShapeError("right-hand side and initial guess lengths differ")
    precision = Precision.of(b)
    if x0.dtype != b.dtype:
        raise PrecisionError("operands must share one precision")
    if b_norm is None:
        b_norm = norm2(b)
    if r0 is None:
        r0 = b - apply_a(x0)
    gamma = norm2(r0)
    if gamma == 0.0:
        return CycleResult(x0.copy() if host else x0.clone(), [], 0, False)
    if not np.isfinite(gamma):
        raise DivergenceError("initial residual is not finite")
    op = apply_a if m_inv is None else (lambda v: apply_a(m_inv(v)))
    n = int(b.shape[0])
    ws = ArnoldiWorkspace(n, m, precision, breakdown_tol)
    ws.start_from_residual(r0, rtol, float(b_norm))
    implicit: list[float] = []
    threshold = rtol * b_norm
    breakdown = False
    while ws.j < m:
        st = arnoldi_step(ws, op, host_operator=host)
        res = ws._last_implicit
        implicit.append(res)
        if st.breakdown:
            breakdown = True
            break
        if res <= threshold:
            break
    k = ws.j
    u = solve_least_squares(ws, k)
    if host:
        u = to_host(u)
    if m_inv is not None:
        u = m_inv(u)
    return CycleResult(x0 + u, implicit, k, breakdown)


def explicit_residual(A, b, x) -> tuple[float, np.ndarray | torch.Tensor]:
    """r = b - A x and ||r|| in A's precision (solvers.py:443-453)."""
    A = CsrMatrix.from_any(A)
    if b.dtype != A.values.dtype and Precision.of(b) is not A.precision:
        raise PrecisionError("residual operands must match the matrix precision")
    if Precision.of(b) is not A.precision or Precision.of(x) is not A.precision:
        raise PrecisionError("residual operands must match the matrix precision")
    if tuple(b.shape) != (A.n_rows,) or tuple(x.shape) != (A.n_cols,):
        raise ShapeError("residual operand lengths do not match the matrix")
    host = not isinstance(b, torch.Tensor)
    bd, xd = to_device(b), to_device(x)
    r = torch.empty(A.n_rows, dtype=A.precision.torch_dtype, device=bd.device)
    out = ctx().scalars[1:2]
    t0 = timing.tick()
    _lib.call("mpg_residual", A.precision.code, A.n_rows, ptr(A.row_ptr), ptr(A.col_idx),
              ptr(A.values), ptr(bd), ptr(xd), ptr(r), ptr(out), ptr(ctx().ws), stream_handle())
    nr = float(out.item())
    timing.tock(timing.SPMV, t0)
    return nr, (to_host(r) if host else r)


# ---------------------------------------------------------------------------
# native fused-cycle solve

class _Prepared(NamedTuple):
    kind: int
    prec: Precision
    block: int
    lu: torch.Tensor | None
    piv: torch.Tensor | None
    ops: list
    values: torch.Tensor | None


def _prepare_precond(M, A: CsrMatrix, solve_prec: Precision) -> _Prepared | None:
    """Validate and upload a right preconditioner (solvers.py:230-244)."""
    if M is None:
        return None
    pp = precision_of(M)
    if not (pp is solve_prec or (pp is FP32 and solve_prec is FP64)):
        raise PrecisionError("an fp64 preconditioner cannot run inside an fp32 solve")
    if is_poly(M):
        vals = A.values if A.precision is pp else convert_matrix(A, pp).values
        return _Prepared(_lib.PC_POLY, pp, 0, None, None, poly_program(M, pp.dtype), vals)
    if is_jacobi(M):
        lu, piv = jacobi_device_arrays(M)
        if Precision.of(lu) is not pp:
            raise PrecisionError("block Jacobi factors do not match their precision tag")
        return _Prepared(_lib.PC_JACOBI, pp, int(M.block_size), lu, piv, [], None)
    raise TypeError(f"unsupported preconditioner type {type(M).__name__}")


_STEP_KERNEL = {"auto": 0, "split": 1, "persistent": 2}
_step_kernel_mode = "auto"


@contextlib.contextmanager
def step_kernel(mode: str):
    """Select the Arnoldi-step implementation of solvers created inside the
    block: "auto" (default: the persistent per-step kernel for small vectors),
    "split" (four launches per step) or "persistent" (csrc/step_kernel.cu)."""
    global _step_kernel_mode
    if mode not in _STEP_KERNEL:
        raise ValueError(f"step kernel must be one of {sorted(_STEP_KERNEL)}")
    prev, _step_kernel_mode = _step_kernel_mode, mode
    try:
        yield
    finally:
        _step_kernel_mode = prev


class NativeSolve:
    """Device buffers + a native solver handle for one restarted solve.

    mode RESTARTED: working precision == outer precision (fp64 GMRES, the
    fp32 solver and both legs of GMRES-FD).  mode IR: fp32 working
    precision, fp64 outer residual/iterate.
    """

    def __init__(self, mode: int, prec: Precision, A: CsrMatrix, A64: CsrMatrix | None,
                 b: torch.Tensor, x: torch.Tensor, m: int, rtol: float,
                 pc: _Prepared | None = None, use_graph: bool = True, storage: str = "auto"):
        self.mode, self.prec, self.m, self.n = mode, prec, m, A.n_rows
        n = self.n
        outer = FP64 if mode == _lib.MODE_IR else prec
        self.outer = outer
        self.ldv = padded_length(n)
        if storage not in ("auto", "csr", "stencil"):
            raise ValueError("storage must be 'auto', 'csr' or 'stencil'")
        shape = A.stencil_shape() if storage != "csr" else None
        if shape is None and storage == "stencil":
            raise ValueError("the matrix is not a 5/7-point Dirichlet stencil")
        # stencil storage: every SpMV input gets one zeroed grid plane of guard
        # rows on each side, so the kernel loads all neighbours unconditionally
        # (absent ones are marked in the packed values, spmv.cuh stencil_row_padded)
        self.guard = 0 if shape is None else padded_length(shape[1] ** (shape[0] - 1))
        self.A, self.A64, self.b = A, A64, b
        self.x = self._guarded(1, outer)
        self.x.copy_(x[: self.ldv])
        self.r = dvec(n, outer)
        self.r_in = dvec(n, FP32) if mode == _lib.MODE_IR else None
        self.V = self._guarded(m + 1, prec)
        self.w = dvec(n, prec)
        self.u = self._guarded(1, prec)
        x = self.x
        self.state = DeviceState(m, prec)
        self.ws = torch.zeros(int(_lib.load().mpg_workspace_bytes()), dtype=torch.uint8,
                              device=device())
        d = _lib.SolverDesc()
        d.mode, d.prec, d.m, d.use_graph = mode, prec.code, m, 1 if use_graph else 0
        d.step_kernel = _STEP_KERNEL[_step_kernel_mode]
        d.n, d.ldv, d.rtol = n, self.ldv, float(rtol)
        d.breakdown_tol = 10.0 * prec.unit_roundoff
        d.row_ptr, d.col_idx, d.values = ptr(A.row_ptr), ptr(A.col_idx), ptr(A.values)
        d.values64 = ptr(A64.values) if A64 is not None else None
        d.x, d.b, d.r = ptr(x), ptr(b), ptr(self.r)
        d.r_in = ptr(self.r_in) if self.r_in is not None else None
        d.V, d.w, d.u = ptr(self.V), ptr(self.w), ptr(self.u)
        d.state, d.ws = ptr(self.state.buf), ptr(self.ws)
        self._keep = []
        if pc is not None:
            d.pc_kind, d.pc_prec, d.pc_block = pc.kind, pc.prec.code, pc.block
            temps = [self._guarded(1, pc.prec) for _ in range(5)]
            self._keep += temps
            d.pc_t0, d.pc_t1, d.pc_t2, d.pc_t3, d.pc_t4 = (ptr(t) for t in temps)
            if pc.kind == _lib.PC_JACOBI:
                d.pc_lu, d.pc_piv = ptr(pc.lu), ptr(pc.piv)
                self._keep += [pc.lu, pc.piv]
            else:
                ops = poly_ops_struct(pc.ops)
                self._keep.append(ops)
                d.pc_ops, d.pc_nops = ops, len(pc.ops)
                d.pc_values = ptr(pc.values)
                self._keep.append(pc.values)
        # stencil-specialised storage: every SpMV of the cycle (Arnoldi operator,
        # polynomial steps, explicit residual) reads packed values instead of CSR
        self.storage = "csr"
        if shape is not None:
            dia = A.dia()
            dia64 = A64.dia() if A64 is not None else None
            pc_dia = None
            if pc is not None and pc.kind == _lib.PC_POLY:
                pc_dia = A.with_values(pc.values).dia()
            if dia is not None and (A64 is None or dia64 is not None) and \
                    (pc is None or pc.kind != _lib.PC_POLY or pc_dia is not None):
                d.stencil_dims, d.stencil_nx = shape
                d.dia = ptr(dia)
                d.dia64 = ptr(dia64) if dia64 is not None else None
                d.pc_dia = ptr(pc_dia) if pc_dia is not None else None
                d.halo = self.guard
                self._keep += [t for t in (dia, dia64, pc_dia) if t is not None]
                # one coefficient per slot: the SpMV streams x alone (csrc/spmv.cuh StencilConst)
                self.storage = "stencil-const" if A.stencil_const() else "stencil"
        self.desc = d
        h = C.c_void_p()
        _lib.call("mpg_solver_create", C.byref(d), C.byref(h))
        self.handle = h

    def _guarded(self, rows: int, prec: Precision) -> torch.Tensor:
        """`rows` zeroed vectors of stride ldv with `guard` readable rows on each side."""
        g = self.guard
        buf = torch.zeros(rows * self.ldv + 2 * g, dtype=prec.torch_dtype, device=device())
        return buf[g: g + rows * self.ldv]

    def close(self) -> None:
        if self.handle:
            _lib.load().mpg_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def begin(self) -> tuple[float, float]:
        _lib.call("mpg_solver_begin", self.handle, stream_handle())
        hdr, _ = self.state.read()
        self.last_hdr = hdr
        return float(hdr.outer_b_norm), float(hdr.rnorm)

    def cycle(self, m_limit: int):
        _lib.call("mpg_solver_cycle", self.handle, int(m_limit), stream_handle())
        hdr, imp = self.state.read()
        self.last_hdr = hdr
        return hdr, imp

    def bin_kernel_times(self, timer: timing.KernelTimer | None) -> None:
        """Add the device's per-category kernel time (globaltimer stamps of the
        cycle kernels, accumulated in the state header since begin()) to
        ``timer``: the reference's tick/tock binning (timing.py:88-98)."""
        hdr = getattr(self, "last_hdr", None)
        if timer is None or hdr is None:
            return
        for i, cat in enumerate(timing.KERNEL_CATEGORIES):
            timer.add(cat, hdr.ktime_ns[i] * 1e-9)

    def profile_cycle(self, m_limit: int) -> dict[str, tuple[float, int]]:
        """One eager cycle with per-kernel-class CUDA events: {class: (ms, launches)}."""
        ms = (C.c_double * 16)()
        cnt = (C.c_int32 * 16)()
        _lib.call("mpg_solver_profile_cycle", self.handle, int(m_limit), stream_handle(), ms, cnt)
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(_lib.PROFILE_CLASSES)}


def _raise_flags(hdr, total: int, ir: bool) -> None:
    f = hdr.flags
    if not f & _ERROR_FLAGS:
        return
    if f & _lib.FLAG_HALO_TIMEOUT:
        raise RuntimeError("distributed peer halo: a neighbour's halo flag did not arrive within 20 s")
    if f & _lib.FLAG_OVERFLOW:
        raise PrecisionOverflowError("an entry of the scaled residual overflows fp32")
    if f & (_lib.FLAG_NONFINITE_OP | _lib.FLAG_NONFINITE_GAMMA):
        msg = ("operator output contains non-finite values" if f & _lib.FLAG_NONFINITE_OP
               else "initial residual is not finite")
        if ir:
            raise DivergenceError(f"fp32 correction solve diverged after {total} iterations: {msg}")
        raise DivergenceError(msg)
    if f & _lib.FLAG_SINGULAR:
        raise SingularHessenbergError("zero diagonal in triangular factor")
    if f & _lib.FLAG_NONFINITE_X:
        raise DivergenceError(f"fp32 correction is not finite after {total} iterations")


def _run_restarted(ns: NativeSolve, criteria: StopCriteria, phase: str,
                   history: list[HistoryEntry], iter_offset: int = 0, limit: int | None = None,
                   stop_on_stall: bool = False):
    """Restart bookkeeping of solvers.py:177-227 over native cycles."""
    b_norm, rnorm = ns.begin()
    explicit_rel = _relative(rnorm, b_norm)
    history.append(HistoryEntry(iter_offset, explicit_rel, explicit_rel, phase))
    limit = criteria.max_iters if limit is None else limit
    total = 0
    converged = explicit_rel <= criteria.rtol
    loss = False
    stalled_at = None
    stall_run = 0
    prev_rel = explicit_rel
    while not converged and not loss and total < limit:
        hdr, imp = ns.cycle(min(criteria.m, limit - total))
        _raise_flags(hdr, total, ir=False)
        implicit = [float(v) for v in imp[: hdr.steps]]
        for i, res in enumerate(implicit[:-1]):
            history.append(HistoryEntry(iter_offset + total + i + 1, _relative(res, b_norm), None, phase))
        total += hdr.steps
        rnorm = float(hdr.rnorm)
        explicit_rel = _relative(rnorm, b_norm)
        implicit_rel = _relative(implicit[-1], b_norm) if implicit else explicit_rel
        history.append(HistoryEntry(iter_offset + total, implicit_rel, explicit_rel, phase))
        if explicit_rel <= criteria.rtol:
            converged = True
        elif implicit_rel <= criteria.rtol and explicit_rel > LOSS_OF_ACCURACY_FACTOR * criteria.rtol:
            loss = True
        if not converged:
            if prev_rel > 0 and (prev_rel - explicit_rel) < STALL_IMPROVEMENT * prev_rel:
                stall_run += 1
            else:
                stall_run = 0
            if stall_run >= STALL_RESTARTS:
                if stalled_at is None:
                    stalled_at = iter_offset + total
                if stop_on_stall:
                    break
            prev_rel = explicit_rel
    return converged, total, loss, stalled_at


def _phase_of(p: Precision) -> str:
    return "fp32" if p is FP32 else "fp64"


def _out(x: torch.Tensor, n: int, host: bool):
    v = x[:n]
    return to_host(v) if host else v.clone()


def _as_vector(v, prec: Precision) -> torch.Tensor:
    """Padded device copy of v in `prec` (overflow-checked narrowing)."""
    if Precision.of(v) is not prec:
        v = convert_vector(v if isinstance(v, torch.Tensor) else np.asarray(v), prec)
    return padded_copy(v, prec)


def gmres_restarted(A, b, x0=None, criteria: StopCriteria | None = None, precond=None,
                    precision: Precision | None = None, *,
                    timer: timing.KernelTimer | None = None, stop_on_stall: bool = False,
                    use_graph: bool = True, storage: str = "auto") -> SolveReport:
    """Restarted GMRES in one working precision (solvers.py:251-294)."""
    criteria = criteria or StopCriteria()
    host = not isinstance(b, torch.Tensor)
    A = CsrMatrix.from_any(A)
    precision = precision or A.precision
    if A.precision is not precision:
        A = convert_matrix(A, precision)
    if not host:
        Precision.of(b)
    bd = _as_vector(b if not host else np.asarray(b), precision)
    n = A.n_cols
    xd = dvec(n, precision) if x0 is None else _as_vector(x0, precision)
    pc = _prepare_precond(precond, A, precision)
    timer = timer if timer is not None else timing.KernelTimer()
    history: list[HistoryEntry] = []
    phase = _phase_of(precision)
    ns = NativeSolve(_lib.MODE_RESTARTED, precision, A, None, bd, xd, criteria.m, criteria.rtol,
                     pc, use_graph, storage)
    try:
        with timing.active(timer):
            converged, total, loss, stalled_at = _run_restarted(
                ns, criteria, phase, history, stop_on_stall=stop_on_stall)
        ns.bin_kernel_times(timer)
    finally:
        ns.close()
    fp32 = precision is FP32
    x = ns.x[:n]
    if fp32:
        x = convert_vector(x, FP64)
    return SolveReport(
        x=to_host(x) if host else x.clone(), converged=converged, total_iters=total,
        iters_fp32=total if fp32 else 0, iters_fp64=0 if fp32 else total,
        residual_history=history, kernel_times=timer.breakdown(), loss_of_accuracy=loss,
        stalled_at=stalled_at, total_time=timer.total)


def gmres_ir(A, b, x0=None, criteria: StopCriteria | None = None, precond_fp32=None, *,
             timer: timing.KernelTimer | None = None, use_graph: bool = True, storage: str = "auto") -> SolveReport:
    """GMRES-IR: fp32 correction cycles, fp64 residual updates (solvers.py:297-384).

    The fp32 copy of A is made up front and excluded from ``total_time``, as in
    the reference; the per-cycle casts, correction and fp64 residual are
    inside it (fused into the cycle's kernels)."""
    criteria = criteria or StopCriteria()
    A = CsrMatrix.from_any(A)
    if A.precision is not FP64:
        raise PrecisionError("iterative refinement expects the matrix in fp64")
    host = not isinstance(b, torch.Tensor)
    if Precision.of(b if not host else np.asarray(b)) is not FP64:
        raise PrecisionError("iterative refinement expects an fp64 right-hand side")
    n = A.n_cols
    bd = padded_copy(b if not host else np.asarray(b), FP64)
    xd = dvec(n, FP64) if x0 is None else padded_copy(
        x0 if isinstance(x0, torch.Tensor) and x0.dtype == torch.float64 else
        np.asarray(x0, dtype=np.float64), FP64)
    if precond_fp32 is not None and precision_of(precond_fp32) is not FP32:
        raise PrecisionError("the inner preconditioner must be fp32")
    A32 = convert_matrix(A, FP32)
    pc = _prepare_precond(precond_fp32, A32, FP32)
    timer = timer if timer is not None else timing.KernelTimer()
    history: list[HistoryEntry] = []
    ns = NativeSolve(_lib.MODE_IR, FP32, A32, A, bd, xd, criteria.m, criteria.rtol, pc, use_graph,
                     storage)
    try:
        with timing.active(timer):
            b_norm, rnorm = ns.begin()                      # suspended in the reference (:328-330)
            explicit_rel = _relative(rnorm, b_norm)
            history.append(HistoryEntry(0, explicit_rel, explicit_rel, "fp32"))
            total = 0
            converged = explicit_rel <= criteria.rtol
            stalled_at = None
            stall_run = 0
            prev_rel = explicit_rel
            while not converged and total < criteria.max_iters:
                rho = rnorm
                hdr, imp = ns.cycle(min(criteria.m, criteria.max_iters - total))
                _raise_flags(hdr, total, ir=True)
                implicit = [float(v) for v in imp[: hdr.steps]]
                scale = rho / b_norm if b_norm > 0 else 1.0
                for i, res in enumerate(implicit[:-1]):
                    history.append(HistoryEntry(total + i + 1, res * scale, None, "fp32"))
                rnorm = float(hdr.rnorm)
                total += hdr.steps
                explicit_rel = _relative(rnorm, b_norm)
                implicit_rel = implicit[-1] * scale if implicit else explicit_rel
                history.append(HistoryEntry(total, implicit_rel, explicit_rel, "fp32"))
                converged = explicit_rel <= criteria.rtol
                if not converged:
                    if prev_rel > 0 and (prev_rel - explicit_rel) < STALL_IMPROVEMENT * prev_rel:
                        stall_run += 1
                    else:
                        stall_run = 0
                    if stall_run >= STALL_RESTARTS and stalled_at is None:
                        stalled_at = total
                    prev_rel = explicit_rel
        ns.bin_kernel_times(timer)
    finally:
        ns.close()
    return SolveReport(
        x=_out(ns.x, n, host), converged=converged, total_iters=total, iters_fp32=total,
        iters_fp64=0, residual_history=history, kernel_times=timer.breakdown(),
        loss_of_accuracy=False, stalled_at=stalled_at, total_time=timer.total)


def gmres_fd(A, b, x0=None, criteria: StopCriteria | None = None, switch_iter: int = 0, *,
             timer: timing.KernelTimer | None = None, use_graph: bool = True, storage: str = "auto") -> SolveReport:
    """fp32 leg up to ``switch_iter`` (or a stall), then fp64 (solvers.py:387-440)."""
    criteria = criteria or StopCriteria()
    if switch_iter < 0 or switch_iter % criteria.m != 0:
        raise ValueError("switch_iter must be a nonnegative multiple of the restart length")
    A = CsrMatrix.from_any(A)
    if A.precision is not FP64:
        raise PrecisionError("the precision-switching solver expects the matrix in fp64")
    host = not isinstance(b, torch.Tensor)
    if Precision.of(b if not host else np.asarray(b)) is not FP64:
        raise PrecisionError("the precision-switching solver expects an fp64 right-hand side")
    n = A.n_cols
    bd = padded_copy(b if not host else np.asarray(b), FP64)
    xd = dvec(n, FP64) if x0 is None else padded_copy(
        x0 if isinstance(x0, torch.Tensor) else np.asarray(x0, dtype=np.float64), FP64)
    timer = timer if timer is not None else timing.KernelTimer()
    history: list[HistoryEntry] = []
    iters32, loss32, stalled_at = 0, False, None
    if switch_iter > 0:
        A32 = convert_matrix(A, FP32)
        b32 = _as_vector(bd[:n], FP32)
        x32 = _as_vector(xd[:n], FP32)
        ns32 = NativeSolve(_lib.MODE_RESTARTED, FP32, A32, None, b32, x32, criteria.m,
                           criteria.rtol, None, use_graph, storage)
        try:
            with timing.active(timer):
                _, iters32, loss32, stalled_at = _run_restarted(
                    ns32, criteria, "fp32", history, iter_offset=0,
                    limit=min(switch_iter, criteria.max_iters), stop_on_stall=True)
                xd = padded_copy(convert_vector(ns32.x[:n], FP64), FP64)
            ns32.bin_kernel_times(timer)
        finally:
            ns32.close()
        if history and history[-1].iteration == iters32:
            history.pop()
    ns = NativeSolve(_lib.MODE_RESTARTED, FP64, A, None, bd, xd, criteria.m, criteria.rtol,
                     None, use_graph, storage)
    try:
        with timing.active(timer):
            converged, iters64, loss64, st64 = _run_restarted(
                ns, criteria, "fp64", history, iter_offset=iters32,
                limit=max(criteria.max_iters - iters32, 0))
        ns.bin_kernel_times(timer)
    finally:
        ns.close()
    return SolveReport(
        x=_out(ns.x, n, host), converged=converged, total_iters=iters32 + iters64,
        iters_fp32=iters32, iters_fp64=iters64, residual_history=history,
        kernel_times=timer.breakdown(), loss_of_accuracy=loss32 or loss64,
        stalled_at=stalled_at if stalled_at is not None else st64, total_time=timer.total)
