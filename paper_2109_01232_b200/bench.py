"""Benchmark protocols of the reference (bench.py:40-343) on the device.

``spmv_bench`` / ``classify_speedup`` / ``Quadrant`` / ``SpmvBenchResult``
follow bench.py:49-119: an untimed warm-up, then ``trials`` timed batches of
``reps`` products per precision on the same seeded vector (narrowed for
fp32), keeping the minimum batch time; the quadrant uses the reference's
thresholds (densest row < 15 nonzeros = left; speedup >= 1.7 = top).  Here
the products are CSR SpMV launches on device-resident operands timed with
CUDA events, so the batch time is device time.

``sweep_switch_point`` / ``sweep_restart`` / ``sweep_rhs`` follow
bench.py:243-343: the same rows (fp64 and refinement baselines plus one
GMRES-FD run per switch point; fp64 and refinement per restart length and per
right-hand-side kind) with ``time_s`` the solver's ``total_time``.  ``config`` is the reference's ``RunConfig`` (io.py:243),
accepted duck-typed; Matrix Market input and RCM reordering go through
``paper_2109_01232_b200.io``.
"""

from __future__ import annotations

import csv
import os
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .core import FP32, FP64, CsrMatrix, convert_matrix, ctx, ptr, stream_handle, to_device
from .gen import generate, make_rhs
from .io import load_matrix_market, rcm_reorder, write_convergence_csv, write_summary_csv
from .solvers import StopCriteria, gmres_fd, gmres_ir, gmres_restarted
from .spmv import predicted_speedup

__all__ = ["Quadrant", "SpmvBenchResult", "classify_speedup", "spmv_bench", "run_experiment", "summary_row",
           "sweep_switch_point", "sweep_restart", "sweep_rhs", "SWITCH_FIELDS", "RESTART_FIELDS", "RHS_FIELDS"]

MAX_ROW_NNZ_THRESHOLD = 15      # bench.py:42
SPEEDUP_THRESHOLD = 1.7         # bench.py:43
DEFAULT_WARMUP = 50             # bench.py:45


class Quadrant(Enum):
    TOP_LEFT = "top-left"
    TOP_RIGHT = "top-right"
    BOTTOM_LEFT = "bottom-left"
    BOTTOM_RIGHT = "bottom-right"


@dataclass
class SpmvBenchResult:
    name: str
    n: int
    nnz: int
    max_nnz_row: int
    t_fp64: float
    t_fp32: float
    measured_speedup: float
    predicted: float
    quadrant: Quadrant
    gbps_fp64: float = float("nan")   # algorithmic CSR bytes per product / time (device only)
    gbps_fp32: float = float("nan")


def classify_speedup(result: SpmvBenchResult) -> Quadrant:
    """Quadrant from (max nonzeros in a row, measured speedup) (bench.py:69-79)."""
    left = result.max_nnz_row < MAX_ROW_NNZ_THRESHOLD
    top = result.measured_speedup >= SPEEDUP_THRESHOLD
    if top:
        return Quadrant.TOP_LEFT if left else Quadrant.TOP_RIGHT
    return Quadrant.BOTTOM_LEFT if left else Quadrant.BOTTOM_RIGHT


def _csr_bytes(A: CsrMatrix, s: int) -> float:
    return A.nnz * (s + 4) + 4 * (A.n_rows + 1) + (A.n_cols + A.n_rows) * s


def spmv_bench(A, reps: int = 1000, trials: int = 3, seed: int = 0, *, warmup: int = DEFAULT_WARMUP,
               name: str = "") -> SpmvBenchResult:
    """Time repeated sparse products in fp64 and fp32 (bench.py:82-119)."""
    if reps < 1:
        raise ValueError("reps must be at least 1")
    if trials < 1:
        raise ValueError("trials must be at least 1")
    A = CsrMatrix.from_any(A)
    A64 = A if A.precision is FP64 else convert_matrix(A, FP64)
    A32 = convert_matrix(A64, FP32)
    x64 = to_device(np.random.default_rng(seed).standard_normal(A.n_cols))
    x32 = x64.to(torch.float32)
    y64 = torch.empty(A.n_rows, dtype=torch.float64, device=x64.device)
    y32 = torch.empty(A.n_rows, dtype=torch.float32, device=x64.device)
    lib, ws, st = _lib.load(), ptr(ctx().ws), stream_handle()

    def launch(M, x, y, code):
        rc = lib.mpg_spmv(code, M.n_rows, ptr(M.row_ptr), ptr(M.col_idx), ptr(M.values), ptr(x), ptr(y), ws, st)
        if rc:
            raise _lib.CudaCallError(f"mpg_spmv failed ({rc})")

    for _ in range(warmup):
        launch(A64, x64, y64, _lib.FP64)
        launch(A32, x32, y32, _lib.FP32)
    times = {}
    for key, M, x, y, code in (("fp64", A64, x64, y64, _lib.FP64), ("fp32", A32, x32, y32, _lib.FP32)):
        best = np.inf
        for _ in range(trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                launch(M, x, y, code)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        times[key] = best
    w = A.nnz / A.n_rows if A.n_rows else 0.0
    res = SpmvBenchResult(
        name=name, n=A.n_rows, nnz=A.nnz, max_nnz_row=A.max_row_nnz(),
        t_fp64=times["fp64"], t_fp32=times["fp32"], measured_speedup=times["fp64"] / times["fp32"],
        predicted=predicted_speedup(w) if w >= 1 else float("nan"), quadrant=Quadrant.TOP_LEFT,
        gbps_fp64=_csr_bytes(A, 8) * reps / times["fp64"] / 1e9,
        gbps_fp32=_csr_bytes(A, 4) * reps / times["fp32"] / 1e9)
    res.quadrant = classify_speedup(res)
    return res


# ---------------------------------------------------------------------------
# sweeps (bench.py:227-312)

def _problem(config, keep_perm: bool = False):
    """(name, A, b[, perm]) as bench.py:134-148: a Matrix Market file or a
    generated stencil, the seeded right-hand side, optional RCM reordering."""
    if hasattr(config, "validate"):
        config.validate()
    if getattr(config, "matrix", None):
        A = load_matrix_market(config.matrix)
        name = os.path.splitext(os.path.basename(config.matrix))[0]
    else:
        A = generate(config.gen)
        name = config.gen.name
    rhs = config.rhs
    if getattr(rhs, "seed", None) != config.seed:
        from dataclasses import replace
        rhs = replace(rhs, seed=config.seed)
    b = make_rhs(rhs, A.n_rows)
    perm = None
    if getattr(config, "rcm", False):
        perm, A = rcm_reorder(A)
        b = perm.apply(b)
    return (name, A, b, perm) if keep_perm else (name, A, b)


def _precond(config, A, precision):
    """bench.py:151-158: none, jacobi:K or poly:D built on A in `precision`."""
    from .precond import build_block_jacobi, build_poly_precond
    spec = config.precond
    if spec.kind == "none":
        return None
    At = A if A.precision is precision else convert_matrix(A, precision)
    if spec.kind == "poly":
        return build_poly_precond(At, spec.param, seed=config.seed)
    return build_block_jacobi(At, spec.param)


def _solve_once(config, A, b, perm=None):
    """bench.py:165-188: the configured solver on (A, b)."""
    criteria = StopCriteria(rtol=config.rtol, max_iters=config.max_iters, m=config.m)
    kind = config.solver.value if hasattr(config.solver, "value") else str(config.solver)
    if kind == "double":
        pc = _precond(config, A, FP32 if getattr(config, "precond_fp32", False) else FP64)
        rep = gmres_restarted(A, b, criteria=criteria, precond=pc, precision=FP64)
    elif kind == "single":
        rep = gmres_restarted(A, b, criteria=criteria, precond=_precond(config, A, FP32), precision=FP32)
    elif kind == "ir":
        rep = gmres_ir(A, b, criteria=criteria, precond_fp32=_precond(config, A, FP32))
    elif kind == "fd":
        if config.precond.kind != "none":
            raise ValueError("the precision-switching solver does not take a preconditioner")
        rep = gmres_fd(A, b, criteria=criteria, switch_iter=config.switch_iter)
    else:
        raise ValueError(f"unknown solver {kind}")
    if perm is not None:
        rep.x = perm.invert_apply(rep.x)
    return rep


def summary_row(name: str, A, config, report) -> dict:
    """bench.py:213-224."""
    kind = config.solver.value if hasattr(config.solver, "value") else str(config.solver)
    return {"name": name, "n": A.n_rows, "nnz": A.nnz, "solver": kind, "precond": str(config.precond),
            "time_s": repr(report.total_time), "iters": report.total_iters, "converged": report.converged,
            "loss_of_accuracy": report.loss_of_accuracy}


def run_experiment(config, out_dir: str | None = None, repeats: int = 3):
    """Run the configured solver ``repeats`` times and keep the median-time run,
    writing the convergence history and a one-row summary CSV when an output
    directory is given (bench.py:191-210)."""
    name, A, b, perm = _problem(config, keep_perm=True)
    reports = sorted((_solve_once(config, A, b, perm) for _ in range(repeats)), key=lambda r: r.total_time)
    report = reports[len(reports) // 2]
    out = out_dir or getattr(config, "out", None)
    if out:
        os.makedirs(out, exist_ok=True)
        kind = config.solver.value if hasattr(config.solver, "value") else str(config.solver)
        tag = f"{name.replace(':', '_')}_{kind}"
        write_convergence_csv(report, os.path.join(out, f"convergence_{tag}.csv"))
        write_summary_csv([summary_row(name, A, config, report)], os.path.join(out, f"summary_{tag}.csv"))
    return report


def _write_rows(rows: list[dict], fields: list[str], path: str) -> None:
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w", encoding="utf-8", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=fields, extrasaction="ignore")
        writer.writeheader()
        writer.writerows(rows)


SWITCH_FIELDS = ["solver", "switch_iter", "total_iters", "iters_fp32", "iters_fp64", "converged", "time_s"]


def _switch_row(solver: str, switch_iter, report) -> dict:
    return {"solver": solver, "switch_iter": switch_iter, "total_iters": report.total_iters,
            "iters_fp32": report.iters_fp32, "iters_fp64": report.iters_fp64,
            "converged": report.converged, "time_s": repr(report.total_time)}


def sweep_switch_point(config, switch_points: list[int], out_dir: str | None = None) -> list[dict]:
    """fp64 and refinement baselines plus one GMRES-FD run per switch point
    (bench.py:243-264).  Rows are deterministic except the time column."""
    name, A, b = _problem(config)
    criteria = StopCriteria(rtol=config.rtol, max_iters=config.max_iters, m=config.m)
    rows = [_switch_row("double", "", gmres_restarted(A, b, criteria=criteria, precision=FP64)),
            _switch_row("ir", "", gmres_ir(A, b, criteria=criteria))]
    for sp in switch_points:
        if sp % config.m:
            raise ValueError(f"switch point {sp} is not a multiple of m={config.m}")
        rows.append(_switch_row("fd", sp, gmres_fd(A, b, criteria=criteria, switch_iter=sp)))
    out = out_dir or getattr(config, "out", None)
    if out:
        _write_rows(rows, SWITCH_FIELDS, os.path.join(out, f"sweep_switch_{name.replace(':', '_')}.csv"))
    return rows


RESTART_FIELDS = ["m", "iters_double", "time_double", "iters_ir", "time_ir", "speedup"]


def sweep_restart(config, sizes: list[int], out_dir: str | None = None) -> list[dict]:
    """fp64 and refinement solves at each restart length (bench.py:283-312)."""
    name, A, b = _problem(config)
    rows = []
    for m in sizes:
        criteria = StopCriteria(rtol=config.rtol, max_iters=config.max_iters, m=m)
        dbl = gmres_restarted(A, b, criteria=criteria, precision=FP64)
        ir = gmres_ir(A, b, criteria=criteria)
        rows.append({"m": m, "iters_double": dbl.total_iters, "time_double": repr(dbl.total_time),
                     "iters_ir": ir.total_iters, "time_ir": repr(ir.total_time),
                     "speedup": repr(dbl.total_time / ir.total_time if ir.total_time else float("nan")),
                     "converged_double": dbl.converged, "converged_ir": ir.converged})
    out = out_dir or getattr(config, "out", None)
    if out:
        _write_rows(rows, RESTART_FIELDS, os.path.join(out, f"sweep_restart_{name.replace(':', '_')}.csv"))
    return rows


RHS_FIELDS = ["rhs", "time_double", "iters_double", "time_ir", "iters_ir", "speedup"]


def sweep_rhs(config, kinds: list, out_dir: str | None = None) -> list[dict]:
    """fp64 and refinement solves for each right-hand-side kind (bench.py:318-343)."""
    from dataclasses import replace
    if hasattr(config, "validate"):
        config.validate()
    criteria = StopCriteria(rtol=config.rtol, max_iters=config.max_iters, m=config.m)
    rows, name = [], None
    for rhs in kinds:
        name, A, b = _problem(replace(config, rhs=rhs))
        dbl = gmres_restarted(A, b, criteria=criteria, precision=FP64)
        ir = gmres_ir(A, b, criteria=criteria)
        kind = rhs.kind.value if hasattr(rhs.kind, "value") else str(rhs.kind)
        rows.append({"rhs": kind, "time_double": repr(dbl.total_time), "iters_double": dbl.total_iters,
                     "time_ir": repr(ir.total_time), "iters_ir": ir.total_iters,
                     "speedup": repr(dbl.total_time / ir.total_time if ir.total_time else float("nan")),
                     "converged_double": dbl.converged, "converged_ir": ir.converged})
    out = out_dir or getattr(config, "out", None)
    if out and name:
        _write_rows(rows, RHS_FIELDS, os.path.join(out, f"sweep_rhs_{name.replace(':', '_')}.csv"))
    return rows
