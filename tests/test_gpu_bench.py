"""Device versions of the reference's benchmark protocols (bench.py:49-312):
spmv_bench / classify_speedup and the switch-point and restart sweeps,
checked against the counts the reference itself reports for Laplace2D(100)
(pkg/test_output.txt:312 and SURVEY.md §8c)."""

from types import SimpleNamespace

import pytest

pytestmark = pytest.mark.gpu

import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import bench as B


def _config(kind, nx, m=50, **kw):
    return SimpleNamespace(gen=P.StencilSpec(P.StencilKind(kind), nx, **kw), rhs=P.RhsSpec(P.RhsKind.ONES),
                           seed=0, m=m, rtol=1e-10, max_iters=100_000, out=None, matrix=None, rcm=False)


def test_spmv_bench_protocol_and_quadrant():
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 60))
    r = B.spmv_bench(A, reps=50, trials=2, warmup=5, name="laplace3d:60")
    assert r.n == 216_000 and r.nnz == A.nnz and r.max_nnz_row == 7
    assert r.t_fp64 > 0 and r.t_fp32 > 0
    assert abs(r.measured_speedup - r.t_fp64 / r.t_fp32) < 1e-12
    assert abs(r.predicted - P.predicted_speedup(A.nnz / A.n_rows)) < 1e-12
    assert r.quadrant is B.classify_speedup(r)
    assert r.quadrant in (B.Quadrant.TOP_LEFT, B.Quadrant.BOTTOM_LEFT)   # 7 < 15 nonzeros per row
    fake = B.SpmvBenchResult("x", 1, 1, 20, 2.0, 1.0, 2.0, 1.0, B.Quadrant.TOP_LEFT)
    assert B.classify_speedup(fake) is B.Quadrant.TOP_RIGHT


def test_sweep_switch_point_laplace2d100_matches_reference(tmp_path):
    rows = B.sweep_switch_point(_config("laplace2d", 100), [0, 100, 200, 500], out_dir=str(tmp_path))
    by = {(r["solver"], r["switch_iter"]): r for r in rows}
    assert by[("double", "")]["total_iters"] == 1172          # reference: 1172
    assert by[("ir", "")]["total_iters"] == 1200              # reference: 1200
    for sp in (0, 100, 200, 500):
        r = by[("fd", sp)]
        assert r["converged"] and r["iters_fp32"] == min(sp, r["total_iters"])
        assert 1168 - 24 <= r["total_iters"] <= 1177 + 24     # reference FD 0..500: 1168-1177 (+-2 %)
    assert (tmp_path / "sweep_switch_laplace2d_100.csv").exists()


def test_sweep_restart_laplace2d100_matches_reference():
    rows = B.sweep_restart(_config("laplace2d", 100), [25, 50, 100])
    got = {r["m"]: (r["iters_double"], r["iters_ir"]) for r in rows}
    assert got == {25: (2039, 2050), 50: (1172, 1200), 100: (469, 500)}   # the reference's counts


def test_matrix_market_and_rcm_device_path(tmp_path):
    """load_matrix_market -> device CSR bit-identical to the reference's;
    rcm_reorder -> the reference's permutation and P A P^T; a solve on the
    reordered system through the sweep plumbing (config.matrix + config.rcm)."""
    import hashlib
    import json
    import os
    import numpy as np
    gold = os.path.join(os.path.dirname(__file__), "golden")
    with open(os.path.join(gold, "reference_io.json")) as f:
        ref = json.load(f)

    def sha(t):
        return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).hexdigest()
    for name in ("general_dups.mtx", "symmetric.mtx", "integer_rect.mtx"):
        A = P.load_matrix_market(os.path.join(gold, "mm", name))
        g = ref["mm"][name]
        assert (A.n_rows, A.n_cols, A.nnz) == (g["n_rows"], g["n_cols"], g["nnz"])
        assert (sha(A.row_ptr), sha(A.col_idx), sha(A.values)) == (g["row_ptr"], g["col_idx"], g["values"])
    A = P.load_matrix_market(os.path.join(gold, "mm", "symmetric.mtx"))
    perm, B = P.rcm_reorder(A)
    g = ref["rcm"]["symmetric.mtx"]
    assert perm.perm.tolist() == g["perm"]
    assert (sha(B.row_ptr), sha(B.col_idx), sha(B.values)) == (g["permuted_row_ptr"], g["permuted_col_idx"],
                                                                g["permuted_values"])
    # round trip through the writer, then the sweep plumbing on the reordered file
    path = str(tmp_path / "lap.mtx")
    P.write_matrix_market(P.generate(P.StencilSpec(P.StencilKind.LAPLACE2D, 30)), path)
    cfg = _config("laplace2d", 30)
    cfg.matrix, cfg.rcm = path, True
    rows = B_.sweep_restart(cfg, [50])
    assert rows[0]["converged_double"] and rows[0]["converged_ir"]


B_ = B


def test_run_experiment_median_and_csv_artefacts(tmp_path):
    """run_experiment (bench.py:191-210): median-time run of `repeats`, the
    convergence and summary CSVs the reference writes (io.py:165-201)."""
    from types import SimpleNamespace
    from paper_2109_01232_b200 import io as mio
    cfg = _config("laplace2d", 50)
    cfg.solver = SimpleNamespace(value="ir")
    cfg.precond = SimpleNamespace(kind="jacobi", param=1, __str__=lambda self: "jacobi:1")
    cfg.precond_fp32, cfg.switch_iter = False, 0
    rep = B.run_experiment(cfg, out_dir=str(tmp_path), repeats=3)
    assert rep.converged and rep.total_iters == 250          # reference: laplace2d:50 IR = 250
    hist = mio.read_convergence_csv(str(tmp_path / "convergence_laplace2d_50_ir.csv"))
    assert hist == rep.residual_history
    text = (tmp_path / "summary_laplace2d_50_ir.csv").read_text().splitlines()
    assert text[0].split(",") == mio.SUMMARY_FIELDS and ",250,True,False" in text[1]
