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


def test_sweeps_reject_out_of_scope_inputs():
    cfg = _config("laplace2d", 20)
    cfg.matrix = "A.mtx"
    with pytest.raises(NotImplementedError):
        B.sweep_restart(cfg, [10])
