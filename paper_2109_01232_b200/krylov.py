"""Device Arnoldi workspace, CGS2 step and rotated least squares.

Mirrors the reference's ``mpgmres.krylov`` (pkg/src/mpgmres/krylov.py) for
callers that drive the Arnoldi process with an arbitrary operator:

* ``ArnoldiWorkspace``   krylov.py:73-103  — basis V ((m+1) x ldv, one padded
  row per basis vector) and the cycle state (H, R, cos, sin, rhs) in device
  memory (layout: include/mpgmres_b200.h, mpg_state_header).
* ``arnoldi_step``       krylov.py:112-151 — w = op(v_j) is computed by the
  caller's operator; then ONE C-ABI call (mpg_arnoldi_step) runs the finite
  check, both classical Gram-Schmidt passes (fused: 3 basis sweeps), h_sub,
  the breakdown test, V[:, j+1] = w / h_sub AND the Givens update of
  krylov.py:154-187 on the device.
* ``givens_update``      krylov.py:154-187 — returns the implicit residual the
  fused step already computed for column j.
* ``solve_least_squares`` krylov.py:190-202 — back-substitution on the device.

The restart drivers in solvers.py do not use this module: they run whole
cycles natively (mpg_solver_cycle).
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, NamedTuple

import numpy as np
import torch

from . import _lib
from .core import (Precision, PrecisionError, ShapeError, ctx, device, dvec, padded_length, ptr,
                   stream_handle, to_device, to_host)

__all__ = ["ArnoldiWorkspace", "HessenbergLS", "ArnoldiStep", "DivergenceError",
           "SingularHessenbergError", "arnoldi_step", "givens_update", "solve_least_squares"]

DEFAULT_BREAKDOWN_FACTOR = 10.0


class DivergenceError(ArithmeticError):
    """Non-finite values appeared during the iteration (the solve is diverging)."""


class SingularHessenbergError(np.linalg.LinAlgError):
    """The rotated triangular factor has a zero diagonal (mishandled breakdown)."""


_ARR = {"H": 0, "R": 1, "cos": 2, "sin": 3, "rhs": 4, "c1": 5, "c2": 6, "d": 7, "implicit": 8}


class DeviceState:
    """A cycle state buffer (header + arrays) and typed host readback."""

    def __init__(self, m: int, precision: Precision):
        lib = _lib.load()
        self.m, self.precision = m, precision
        self.nbytes = int(lib.mpg_state_bytes(precision.code, m))
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device())
        self.off = {k: int(lib.mpg_state_offset(precision.code, m, v)) for k, v in _ARR.items()}
        self._hdr_len = self.off["implicit"] + 8 * m
        self._host = torch.empty(self._hdr_len, dtype=torch.uint8, pin_memory=True)

    def read(self) -> tuple[_lib.StateHeader, np.ndarray]:
        """One D2H copy of the header and the implicit-residual record."""
        self._host.copy_(self.buf[: self._hdr_len], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        raw = self._host.numpy()
        hdr = _lib.StateHeader.from_buffer_copy(raw[: C.sizeof(_lib.StateHeader)].tobytes())
        imp = raw[self.off["implicit"]: self.off["implicit"] + 8 * self.m].view(np.float64).copy()
        return hdr, imp

    def array(self, name: str, count: int) -> np.ndarray:
        dt = self.precision.dtype
        o = self.off[name]
        return to_host(self.buf[o: o + count * dt.itemsize]).view(dt).copy()


class HessenbergLS:
    """Host snapshot of the rotated Hessenberg system (krylov.py:43-70)."""

    def __init__(self, state: DeviceState):
        m = state.m
        self.m = m
        self._state = state

    def _mat(self, name):
        a = self._state.array(name, (self.m + 1) * self.m)
        return a.reshape(self.m, self.m + 1).T.copy()   # stored column-major

    @property
    def H(self):
        return self._mat("H")

    @property
    def R(self):
        return self._mat("R")

    @property
    def givens_cos(self):
        return self._state.array("cos", self.m)

    @property
    def givens_sin(self):
        return self._state.array("sin", self.m)

    @property
    def rhs(self):
        return self._state.array("rhs", self.m + 1)

    @property
    def implicit_resnorm(self) -> float:
        hdr, imp = self._state.read()
        return float(imp[hdr.steps - 1]) if hdr.steps else float(abs(hdr.gamma))


class ArnoldiWorkspace:
    """Single-owner device state for one restart cycle (krylov.py:73-103)."""

    def __init__(self, n: int, m: int, precision: Precision, breakdown_tol: float | None = None):
        if m < 1:
            raise ValueError("at least one step is required")
        self.n, self.m, self.precision = n, m, precision
        self.ldv = padded_length(n)
        self.V_buf = torch.zeros((m + 1) * self.ldv, dtype=precision.torch_dtype, device=device())
        self.w = dvec(n, precision)
        self.state = DeviceState(m, precision)
        self.hls = HessenbergLS(self.state)
        self.j = 0
        self.broke_down = False
        if breakdown_tol is None:
            breakdown_tol = DEFAULT_BREAKDOWN_FACTOR * precision.unit_roundoff
        self.breakdown_tol = breakdown_tol
        self._ws = torch.zeros(int(_lib.load().mpg_workspace_bytes()), dtype=torch.uint8,
                               device=device())

    @property
    def V(self) -> torch.Tensor:
        """(n, m+1) view with basis vectors as columns (like the reference's F-order V)."""
        return self.V_buf.view(self.m + 1, self.ldv)[:, : self.n].t()

    def column(self, j: int) -> torch.Tensor:
        return self.V_buf[j * self.ldv: j * self.ldv + self.n]

    def start(self, v0, gamma: float, rtol: float = 0.0, b_norm: float = -1.0) -> None:
        """V[:,0] = v0 and the rotated system reset to gamma*e1.  On the device
        the start kernel recomputes gamma = ||r0|| from r0 = gamma*v0; callers
        that hold r0 pass it through :func:`start_from_residual`."""
        r0 = to_device(v0) * gamma if gamma != 1.0 else to_device(v0)
        self.start_from_residual(r0, rtol, b_norm)

    def start_from_residual(self, r0, rtol: float, b_norm: float) -> None:
        r = dvec(self.n, self.precision)
        r[: self.n].copy_(to_device(r0))
        _lib.call("mpg_cycle_start", self.precision.code, self.n, self.ldv, self.m, ptr(r),
                  ptr(self.V_buf), ptr(self.state.buf), float(rtol), float(b_norm),
                  float(self.breakdown_tol), self.m, ptr(self._ws), stream_handle())
        self.j = 0
        self.broke_down = False

    def basis(self) -> torch.Tensor:
        return self.V[:, : self.j + (0 if self.broke_down else 1)]


class ArnoldiStep(NamedTuple):
    h_col: np.ndarray
    h_subdiag: float
    breakdown: bool


def arnoldi_step(ws: ArnoldiWorkspace, apply_op: Callable, *, host_operator: bool = False,
                 m_limit: int | None = None) -> ArnoldiStep:
    """One CGS2 Arnoldi step + Givens update (krylov.py:112-187) on the device."""
    j = ws.j
    if j >= ws.m:
        raise ValueError("workspace already holds the maximum number of steps")
    v = ws.column(j)
    w = apply_op(to_host(v) if host_operator else v)
    if tuple(w.shape) != (ws.n,):
        raise ShapeError(f"operator returned length {tuple(w.shape)}, expected {(ws.n,)}")
    if Precision.of(w) is not ws.precision:
        raise PrecisionError("operator changed the working precision")
    ws.w[: ws.n].copy_(to_device(w))
    _lib.call("mpg_arnoldi_step", ws.precision.code, ws.n, ws.ldv, ws.m, j,
              ws.m if m_limit is None else m_limit, ptr(ws.V_buf), ptr(ws.w), ptr(ws.state.buf),
              ptr(ws._ws), stream_handle())
    hdr, imp = ws.state.read()
    if hdr.flags & _lib.FLAG_NONFINITE_OP:
        raise DivergenceError("operator output contains non-finite values")
    ws.broke_down = bool(hdr.breakdown)
    ws.j += 1
    hcol = ws.state.array("H", (ws.m + 1) * (j + 1))[j * (ws.m + 1): j * (ws.m + 1) + j + 1]
    ws._last_implicit = float(imp[j])
    ws._last_done = bool(hdr.done)
    return ArnoldiStep(hcol, float(hdr.h_sub), bool(hdr.breakdown))


def givens_update(hls, j: int) -> float:
    """Implicit residual after folding column j (computed by the fused step)."""
    if isinstance(hls, ArnoldiWorkspace):
        hls = hls.hls
    hdr, imp = hls._state.read()
    if j >= hdr.steps:
        raise ValueError(f"column {j} has not been computed")
    return float(imp[j])


def solve_least_squares(ws: ArnoldiWorkspace, k: int | None = None) -> torch.Tensor:
    """u = V[:, :k] d with R d = rhs (krylov.py:190-202 + solvers.py:171).
    Returns u on the device; raises SingularHessenbergError like the reference."""
    u = dvec(ws.n, ws.precision)
    _lib.call("mpg_cycle_finish", ws.precision.code, ws.n, ws.ldv, ws.m, ptr(ws.V_buf),
              ptr(ws.state.buf), ptr(u), stream_handle())
    hdr, _ = ws.state.read()
    if hdr.flags & _lib.FLAG_SINGULAR:
        raise SingularHessenbergError("zero diagonal in triangular factor")
    return u[: ws.n]
