"""DEVICE-ORDER ORACLE — TEST INFRASTRUCTURE ONLY.

Host loops over ``oracle/devorder.c`` (built by ``oracle/Makefile`` into
``oracle/_build/libdevorder.so``): GMRES-IR, restarted GMRES (fp32 / fp64)
and GMRES-FD with the reference's restart bookkeeping (solvers.py:177-227,
297-440 of /root/reference/pkg/src/mpgmres, identical to oracle/cpu_gmres.py
and to paper_2109_01232_b200/solvers.py), but every dot product, norm and
basis update associated the way the single-GPU kernels associate them.

Purpose: the parity tests assert (1) the GPU solve equals this restatement
bit for bit, and (2) it shares every other operation with the reference-order
oracle, so where the GPU's iteration count differs from the reference's, the
difference is the reduction order and nothing else.

Scope: unpreconditioned solves on stencil storage, restart length <= 55 (every
step runs the persistent step kernel), n*sizeof <= 20 MB, and residual
launches of at most one tile wave (n <= 148 * 256 * VN rows): the sizes the
parity tests run.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import NamedTuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libdevorder.so")

STALL_IMPROVEMENT = 0.01        # solvers.py:55
STALL_RESTARTS = 2              # solvers.py:56
LOSS_FACTOR = 10.0              # solvers.py:51
U32, U64 = 2.0 ** -24, 2.0 ** -53
MEGA_MAX_K = 56                 # csrc/state.cuh kMegaMaxK

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P, I, D, LL = C.c_void_p, C.c_int, C.c_double, C.c_longlong
        for name in ("devorder_cycle_f32", "devorder_cycle_f64"):
            getattr(L, name).argtypes = [I, P, P, P, P, D, D, D, I, I, P, P, P, I]
        L.devorder_cycle_ir.argtypes = [I, P, P, P, P, D, D, D, I, I, P, P, P, I]
        for name in ("devorder_residual_f32", "devorder_residual_f64"):
            getattr(L, name).argtypes = [I, P, P, P, P, P, P, LL]
            getattr(L, name).restype = D
        for name in ("devorder_norm2_f32", "devorder_norm2_f64"):
            getattr(L, name).argtypes = [P, LL, I]
            getattr(L, name).restype = D
        L.devorder_residual_grid.argtypes = [LL, I, I, I]
        L.devorder_residual_grid.restype = LL
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Report(NamedTuple):
    x: np.ndarray
    converged: bool
    total_iters: int
    iters_fp32: int
    iters_fp64: int
    history: list          # (iteration, implicit, explicit | None, phase)
    loss_of_accuracy: bool
    stalled_at: int | None


def _rel(v, s):
    if s > 0.0:
        return v / s
    return 0.0 if v == 0.0 else float("inf")


class _Op:
    """One working precision of A plus the launch geometry."""

    def __init__(self, A, dt, nsm: int):
        self.n = A.n_rows
        self.dt = np.dtype(dt)
        self.rp = np.ascontiguousarray(A.row_ptr, dtype=np.int32)
        self.ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
        self.v = np.ascontiguousarray(A.values, dtype=self.dt)
        self.suf = "f32" if self.dt == np.float32 else "f64"
        self.nsm = nsm
        vn = 4 if self.suf == "f32" else 2
        tiles = -(-self.n // (256 * vn))
        if tiles > nsm:
            raise ValueError("device-order oracle: the residual grid would depend on occupancy")
        if self.n * self.dt.itemsize > 20e6:
            raise ValueError("device-order oracle: the solver would use the four-launch step")
        self.rgrid = lib().devorder_residual_grid(self.n, vn, nsm, 1 << 20)

    def norm2(self, x):
        x = np.ascontiguousarray(x, dtype=self.dt)
        return getattr(lib(), f"devorder_norm2_{self.suf}")(_p(x), self.n, self.nsm)

    def residual(self, b, x):
        r = np.empty(self.n, dtype=self.dt)
        nr = getattr(lib(), f"devorder_residual_{self.suf}")(
            self.n, _p(self.rp), _p(self.ci), _p(self.v), _p(b), _p(x), _p(r), self.rgrid)
        return nr, r

    def cycle(self, r, bnorm, rtol, m, m_limit, x):
        imp = np.zeros(m, dtype=np.float64)
        info = np.zeros(3, dtype=np.int32)
        btol = 10.0 * (U32 if self.suf == "f32" else U64)
        getattr(lib(), f"devorder_cycle_{self.suf}")(
            self.n, _p(self.rp), _p(self.ci), _p(self.v), _p(r), bnorm, rtol, btol, m, m_limit,
            _p(x), _p(imp), _p(info), self.nsm)
        return int(info[0]), [float(v) for v in imp[: info[0]]], int(info[2])


def _check_m(m):
    if m > MEGA_MAX_K - 1:
        raise ValueError("device-order oracle covers restart lengths <= 55 (persistent step)")


def _restart_loop(op: _Op, b, x, rtol, m, limit, phase, hist, offset=0, stop_on_stall=False):
    """solvers.py _run_restarted over device-order cycles (reference solvers.py:177-227)."""
    bn = op.norm2(b)
    rn, r = op.residual(b, x)
    rel = _rel(rn, bn)
    hist.append((offset, rel, rel, phase))
    total, conv, loss, stalled, run, prev = 0, rel <= rtol, False, None, 0, rel
    while not conv and not loss and total < limit:
        steps, imp, flags = op.cycle(r, bn, rtol, m, min(m, limit - total), x)
        if flags:
            raise ArithmeticError(f"device-order cycle flags {flags}")
        for i, res in enumerate(imp[:-1]):
            hist.append((offset + total + i + 1, _rel(res, bn), None, phase))
        total += steps
        rn, r = op.residual(b, x)
        rel = _rel(rn, bn)
        irel = _rel(imp[-1], bn) if imp else rel
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


def solve_restarted(A, b, rtol=1e-10, m=50, max_iters=100_000, dtype=np.float64, nsm=148) -> Report:
    _check_m(m)
    op = _Op(A, dtype, nsm)
    b = np.ascontiguousarray(np.asarray(b).astype(op.dt))
    x = np.zeros(op.n, dtype=op.dt)
    hist: list = []
    phase = "fp32" if op.dt == np.float32 else "fp64"
    x, conv, tot, loss, st = _restart_loop(op, b, x, rtol, m, max_iters, phase, hist)
    f32 = op.dt == np.float32
    return Report(x.astype(np.float64), conv, tot, tot if f32 else 0, 0 if f32 else tot, hist, loss, st)


def solve_ir(A, b, rtol=1e-10, m=50, max_iters=100_000, nsm=148) -> Report:
    """GMRES-IR host loop of solvers.py gmres_ir (reference solvers.py:297-384)."""
    _check_m(m)
    op64, op32 = _Op(A, np.float64, nsm), _Op(A.astype(np.float32), np.float32, nsm)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(op64.n)
    hist: list = []
    bn = op64.norm2(b)
    rn, r = op64.residual(b, x)
    rel = _rel(rn, bn)
    hist.append((0, rel, rel, "fp32"))
    total, conv, stalled, run, prev = 0, rel <= rtol, None, 0, rel
    btol = 10.0 * U32
    while not conv and total < max_iters:
        rho = rn
        imp = np.zeros(m, dtype=np.float64)
        info = np.zeros(3, dtype=np.int32)
        lib().devorder_cycle_ir(op32.n, _p(op32.rp), _p(op32.ci), _p(op32.v), _p(r), rho, rtol, btol, m,
                                min(m, max_iters - total), _p(x), _p(imp), _p(info), nsm)
        if info[2]:
            raise ArithmeticError(f"device-order cycle flags {int(info[2])}")
        implicit = [float(v) for v in imp[: info[0]]]
        sc = rho / bn if bn > 0 else 1.0
        for i, res in enumerate(implicit[:-1]):
            hist.append((total + i + 1, res * sc, None, "fp32"))
        rn, r = op64.residual(b, x)
        total += int(info[0])
        rel = _rel(rn, bn)
        irel = implicit[-1] * sc if implicit else rel
        hist.append((total, irel, rel, "fp32"))
        conv = rel <= rtol
        if not conv:
            run = run + 1 if (prev > 0 and (prev - rel) < STALL_IMPROVEMENT * prev) else 0
            if run >= STALL_RESTARTS and stalled is None:
                stalled = total
            prev = rel
    return Report(x, conv, total, total, 0, hist, False, stalled)


def solve_fd(A, b, rtol=1e-10, m=50, max_iters=100_000, switch_iter=0, nsm=148) -> Report:
    """GMRES-FD host loop of solvers.py gmres_fd (reference solvers.py:387-440)."""
    _check_m(m)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n_rows)
    hist: list = []
    n32, loss32, stalled = 0, False, None
    if switch_iter > 0:
        op32 = _Op(A.astype(np.float32), np.float32, nsm)
        x32, _, n32, loss32, stalled = _restart_loop(
            op32, b.astype(np.float32), np.zeros(A.n_rows, dtype=np.float32), rtol, m,
            min(switch_iter, max_iters), "fp32", hist, 0, True)
        x = x32.astype(np.float64)
        if hist and hist[-1][0] == n32:
            hist.pop()
    op64 = _Op(A, np.float64, nsm)
    x, conv, n64, loss64, st64 = _restart_loop(op64, b, x, rtol, m, max(max_iters - n32, 0), "fp64",
                                               hist, n32)
    return Report(x, conv, n32 + n64, n32, n64, hist, loss32 or loss64,
                  stalled if stalled is not None else st64)
