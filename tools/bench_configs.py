"""Solve-time sweep over the BASELINE.json configs on one GPU (not the driver's
bench line; that is bench.py on configs[1]).  One JSON line per solve.

    python tools/bench_configs.py cfg3|cfg4|cfg5|all [--reps 1]

cfg3  convdiff2d:1500:c1501 (UniFlow2D, 2.25M rows): fp64 GMRES(50) and
      GMRES-IR + fp32 Jacobi(1)  (reference: 2744 / 3100 iterations)
cfg4  laplace3d:200 (8M rows): GMRES-IR + GMRES-polynomial preconditioner of
      degree 25 and 40 (Newton/Leja form, seed 0), plus plain IR and fp64
cfg5  laplace3d:400 (64M rows) on ONE B200: GMRES-IR and fp64 GMRES(50) to 1e-10
      (the north star's 8-GPU target problem, single-GPU here)

Times are CUDA-event solve times (the reference's total_time span: the fp32
matrix copy and the preconditioner build are excluded and reported apart).
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2109_01232_b200 as P


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = fn()
    e1.record()
    e1.synchronize()
    return rep, e0.elapsed_time(e1) / 1e3


def line(cfg, name, A, b, rep, secs, extra=None):
    nr, _ = P.explicit_residual(A, b, rep.x)
    d = {"config": cfg, "solver": name, "n": A.n_rows, "nnz": A.nnz, "converged": rep.converged,
         "iters": rep.total_iters, "iters_fp32": rep.iters_fp32, "iters_fp64": rep.iters_fp64,
         "solve_s": [round(s, 4) for s in secs], "s_per_iter": round(min(secs) / max(rep.total_iters, 1), 7),
         "final_rel_residual": nr / float(torch.linalg.norm(b))}
    d.update(extra or {})
    print(json.dumps(d), flush=True)
    return d


def run(cfg, name, A, b, fn, reps, extra=None, warm=None):
    """warm: a short solve (graph capture, first-touch) run before timing."""
    if warm is not None:
        warm()
    rep, secs = None, []
    for _ in range(reps):
        rep, s = timed(fn)
        secs.append(s)
    return line(cfg, name, A, b, rep, secs, extra)


def cfg3(reps):
    A = P.generate(P.StencilSpec(P.StencilKind.CONVDIFF2D, 1500, convection=1501.0))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50)
    w = P.StopCriteria(rtol=1e-10, m=50, max_iters=100)
    run("cfg3 convdiff2d:1500:c1501", "fp64", A, b, lambda: P.gmres_restarted(A, b, criteria=crit), reps,
        {"reference_iters": 2744}, lambda: P.gmres_restarted(A, b, criteria=w))
    t0 = time.perf_counter()
    M = P.build_block_jacobi(P.convert_matrix(A, P.FP32), 1)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t0
    run("cfg3 convdiff2d:1500:c1501", "ir+jacobi1", A, b,
        lambda: P.gmres_ir(A, b, criteria=crit, precond_fp32=M), reps,
        {"reference_iters": 3100, "precond_build_s": round(tb, 4)},
        lambda: P.gmres_ir(A, b, criteria=w, precond_fp32=M))


def cfg4(reps):
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 200))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50)
    w = P.StopCriteria(rtol=1e-10, m=50, max_iters=100)
    run("cfg4 laplace3d:200", "ir", A, b, lambda: P.gmres_ir(A, b, criteria=crit), reps, None,
        lambda: P.gmres_ir(A, b, criteria=w))
    A32 = P.convert_matrix(A, P.FP32)
    for deg in (25, 40):
        t0 = time.perf_counter()
        M = P.build_poly_precond(A32, deg, seed=0)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        run("cfg4 laplace3d:200", f"ir+poly{deg}", A, b,
            lambda: P.gmres_ir(A, b, criteria=crit, precond_fp32=M), reps,
            {"precond_build_s": round(tb, 4), "poly_basis": str(M.basis), "spmv_per_iter": deg + 1},
            lambda: P.gmres_ir(A, b, criteria=w, precond_fp32=M))
    run("cfg4 laplace3d:200", "fp64", A, b, lambda: P.gmres_restarted(A, b, criteria=crit), reps, None,
        lambda: P.gmres_restarted(A, b, criteria=w))


def cfg5(reps):
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 400))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50)
    w = P.StopCriteria(rtol=1e-10, m=50, max_iters=100)
    ir = run("cfg5 laplace3d:400 (1 GPU)", "ir", A, b, lambda: P.gmres_ir(A, b, criteria=crit), reps, None,
             lambda: P.gmres_ir(A, b, criteria=w))
    f64 = run("cfg5 laplace3d:400 (1 GPU)", "fp64", A, b, lambda: P.gmres_restarted(A, b, criteria=crit), reps,
              None, lambda: P.gmres_restarted(A, b, criteria=w))
    print(json.dumps({"config": "cfg5 laplace3d:400 (1 GPU)", "speedup_ir_vs_fp64":
                      round(min(f64["solve_s"]) / min(ir["solve_s"]), 3)}), flush=True)


def spmv(reps):
    """bench.spmv_bench (the reference's SpMV protocol, bench.py:82-119) on the config matrices."""
    from paper_2109_01232_b200 import bench as B
    for name, spec in (("laplace3d:150", P.StencilSpec(P.StencilKind.LAPLACE3D, 150)),
                       ("convdiff2d:1500:c1501", P.StencilSpec(P.StencilKind.CONVDIFF2D, 1500, convection=1501.0)),
                       ("laplace3d:200", P.StencilSpec(P.StencilKind.LAPLACE3D, 200))):
        A = P.generate(spec)
        r = B.spmv_bench(A, reps=200, trials=3, name=name)
        print(json.dumps({"spmv_bench": name, "n": r.n, "nnz": r.nnz, "max_nnz_row": r.max_nnz_row,
                          "t_fp64_per_product_us": round(r.t_fp64 / 200 * 1e6, 2),
                          "t_fp32_per_product_us": round(r.t_fp32 / 200 * 1e6, 2),
                          "measured_speedup": round(r.measured_speedup, 3), "predicted": round(r.predicted, 3),
                          "quadrant": r.quadrant.value, "GBps_fp64": round(r.gbps_fp64, 1),
                          "GBps_fp32": round(r.gbps_fp32, 1)}), flush=True)
        del A
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg3", "cfg4", "cfg5", "spmv", "all"])
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    for c in (("cfg3", "cfg4", "cfg5") if a.which == "all" else (a.which,)):
        globals()[c](a.reps)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
