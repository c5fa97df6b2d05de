"""Pin the CPU oracle (oracle/cpu_gmres.py) before trusting it.

1. Against the reference's own golden numbers (pkg/tests/test_solvers.py:16
   GOLDEN_LAPLACE2D50_ITERS = 235; pkg/test_output.txt:312 1172/1200/...).
2. Against fixtures recorded from the reference itself
   (tests/golden/make_golden.py): iteration counts, every restart-boundary
   residual, and the sha256 of the solution bits.
3. Directly against the reference package when it is importable (build
   container only).
"""

import hashlib

import numpy as np
import pytest

from oracle import cpu_gmres as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _solve(name, spec, solver, kw):
    kind, nx, sk = spec
    A = O.stencil_csr(kind, nx, **sk)
    b = O.ones_rhs(A.n_rows)
    m = kw["m"]
    mi = kw.get("max_iters", 100_000)
    if solver == "fp64":
        return O.solve_restarted(A, b, m=m, max_iters=mi)
    if solver == "fp32":
        return O.solve_restarted(A, b, m=m, max_iters=mi, dtype=np.float32)
    if solver == "ir":
        return O.solve_ir(A, b, m=m, max_iters=mi)
    if solver == "fd":
        return O.solve_fd(A, b, m=m, max_iters=mi, switch_iter=kw["switch_iter"])
    A32 = A.astype(np.float32)
    if solver == "ir+jacobi1":
        return O.solve_ir(A, b, m=m, precond32=O.jacobi_build(A32, 1))
    if solver.startswith("ir+poly"):
        return O.solve_ir(A, b, m=m, precond32=O.poly_build(A32, int(solver[7:]), seed=0))
    if solver == "fp64+poly25_32":
        return O.solve_restarted(A, b, m=m, precond=O.poly_build(A32, 25, seed=0))
    raise ValueError(solver)


# name -> spec/solver, mirrors make_golden.SMALL_RUNS
CASES = {
    "laplace2d:50/fp64/m50": (("laplace2d", 50, {}), "fp64", {"m": 50}),
    "laplace2d:50/ir/m50": (("laplace2d", 50, {}), "ir", {"m": 50}),
    "laplace2d:100/fp64/m50": (("laplace2d", 100, {}), "fp64", {"m": 50}),
    "laplace2d:100/ir/m50": (("laplace2d", 100, {}), "ir", {"m": 50}),
    "laplace2d:100/fd200/m50": (("laplace2d", 100, {}), "fd", {"m": 50, "switch_iter": 200}),
    "laplace2d:100/fp64/m25": (("laplace2d", 100, {}), "fp64", {"m": 25}),
    "laplace2d:100/ir/m100": (("laplace2d", 100, {}), "ir", {"m": 100}),
    "laplace3d:40/ir/m50": (("laplace3d", 40, {}), "ir", {"m": 50}),
    "laplace3d:30/fd100/m50": (("laplace3d", 30, {}), "fd", {"m": 50, "switch_iter": 100}),
    "convdiff2d:100:c100/fp64/m50": (("convdiff2d", 100, {"convection": 100.0}), "fp64", {"m": 50}),
    "convdiff2d:60:c61/ir+jacobi1/m50": (("convdiff2d", 60, {"convection": 61.0}), "ir+jacobi1", {"m": 50}),
    "recirc2d:40:c0.5/ir/m50": (("recirc2d", 40, {"convection": 0.5}), "ir", {"m": 50}),
    "laplace3d:20/ir+poly25/m50": (("laplace3d", 20, {}), "ir+poly25", {"m": 50}),
    "laplace3d:20/fp64+poly25_32/m50": (("laplace3d", 20, {}), "fp64+poly25_32", {"m": 50}),
    "laplace2d:20/fp64/m10/max15": (("laplace2d", 20, {}), "fp64", {"m": 10, "max_iters": 15}),
}


def test_reference_published_goldens(golden_runs):
    # the reference's own pinned numbers
    assert golden_runs["laplace2d:50/fp64/m50"]["total_iters"] == 235
    assert golden_runs["laplace2d:100/fp64/m50"]["total_iters"] == 1172
    assert golden_runs["laplace2d:100/ir/m50"]["total_iters"] == 1200


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_fixture(name, golden_runs):
    spec, solver, kw = CASES[name]
    rep = _solve(name, spec, solver, kw)
    g = golden_runs[name]
    assert rep.total_iters == g["total_iters"]
    assert rep.converged == g["converged"]
    assert rep.loss_of_accuracy == g["loss_of_accuracy"]
    assert rep.stalled_at == g["stalled_at"]
    bounds = [[it, imp, exp, ph] for (it, imp, exp, ph) in rep.history if exp is not None]
    assert bounds == g["boundaries"]
    assert sha(rep.x) == g["x_sha256"]


def test_oracle_generator_small_hashes(golden_assembly):
    for key, g in golden_assembly.items():
        if g["n"] > 500_000:
            continue
        A = O.stencil_csr(g["kind"], g["nx"], **g["kwargs"])
        assert (A.n_rows, A.nnz) == (g["n"], g["nnz"])
        assert sha(A.row_ptr) == g["row_ptr"], key
        assert sha(A.col_idx) == g["col_idx"], key
        assert sha(A.values) == g["values"], key


def test_oracle_generator_counts():
    for nx in (2, 3, 7, 50):
        assert O.stencil_size("laplace2d", nx) == (nx ** 2, 5 * nx ** 2 - 4 * nx)
        assert O.stencil_size("laplace3d", nx) == (nx ** 3, 7 * nx ** 3 - 6 * nx ** 2)
    assert O.stencil_size("recirc2d", 1500) == (2_250_000, 11_244_000)


def test_oracle_spmv_matches_fixtures(spmv_cases):
    for (name, prec), c in spmv_cases.items():
        A = O.Csr(len(c["row_ptr"]) - 1, len(c["x"]), c["row_ptr"], c["col_idx"], c["values"])
        y = O.spmv(A, c["x"])
        assert np.array_equal(y.view(np.uint8), c["y"].view(np.uint8)), (name, prec)


def test_row_partition_covers_rows():
    for n, p in ((10, 3), (64_000_000, 8), (7, 7), (5, 8)):
        parts = O.row_partition(n, p)
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def test_oracle_slices_concatenate():
    full = O.stencil_csr("convdiff2d", 17, convection=30.0)
    a, b = 100, 200
    s = O.stencil_csr("convdiff2d", 17, convection=30.0, row_begin=a, row_end=b)
    assert np.array_equal(s.row_ptr, full.row_ptr[a:b + 1])
    lo, hi = full.row_ptr[a], full.row_ptr[b]
    assert np.array_equal(s.col_idx, full.col_idx[lo:hi])
    assert np.array_equal(s.values, full.values[lo:hi])


def test_oracle_equals_reference_directly(reference):
    mp = reference
    for kind, nx, kw in (("laplace2d", 30, {}), ("convdiff2d", 25, {"convection": 40.0})):
        A = mp.generate(mp.StencilSpec(mp.StencilKind(kind), nx, **kw))
        b = np.ones(A.n_rows)
        for m in (20, 50):
            crit = mp.StopCriteria(rtol=1e-10, m=m)
            Ao = O.Csr(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
            for ref, ora in ((mp.gmres_restarted(A, b, criteria=crit), O.solve_restarted(Ao, b, m=m)),
                             (mp.gmres_ir(A, b, criteria=crit), O.solve_ir(Ao, b, m=m))):
                assert ref.total_iters == ora.total_iters
                assert np.array_equal(ref.x, ora.x)


def test_order_study_fixture_is_anchored_on_the_reference(golden_runs):
    """The reduction-order study (tests/golden/order_spread.py) starts from the
    unperturbed oracle, which must reproduce the reference's count."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "order_spread.json")) as f:
        spread = json.load(f)
    for name, sp in spread.items():
        assert sp["counts"]["reference"] == golden_runs[name]["total_iters"]
        assert sp["min"] <= sp["counts"]["reference"] <= sp["max"]
        assert "device_order" in sp


# ------------------------------------------------------------ device-order oracle

def test_device_order_oracle_builds_and_shares_the_reference_spmv(rng):
    """oracle/devorder.c (the reference algorithm with the GPU kernels'
    reduction association) computes every SpMV exactly as the reference-order
    oracle: the row order of spmv.py:48-72 is the same on both."""
    import ctypes as C
    from oracle import devorder as D
    L = D.lib()
    for kind, nx, kw in (("laplace3d", 9, {}), ("recirc2d", 17, {"convection": 3.0}),
                         ("convdiff2d", 12, {"convection": 40.0})):
        A = O.stencil_csr(kind, nx, **kw)
        for dt, fn in ((np.float64, L.devorder_spmv_f64), (np.float32, L.devorder_spmv_f32)):
            Ad = A.astype(dt)
            x = rng.standard_normal(A.n_rows).astype(dt)
            y = np.empty(A.n_rows, dtype=dt)
            fn(C.c_int(A.n_rows), D._p(np.ascontiguousarray(Ad.row_ptr, np.int32)),
               D._p(np.ascontiguousarray(Ad.col_idx, np.int32)), D._p(np.ascontiguousarray(Ad.values)),
               D._p(x), D._p(y))
            assert np.array_equal(y.view(np.uint8), O.spmv(Ad, x).view(np.uint8))


def test_device_order_oracle_converges_like_the_reference_where_order_is_benign(golden_runs):
    """Where the count is insensitive to the association, the
    device-order oracle reproduces the reference's golden counts; its
    solutions agree with the reference-order oracle to 1e-8."""
    from oracle import devorder as D
    for name, kind, nx, solver in (("laplace2d:50/fp64/m50", "laplace2d", 50, "fp64"),
                                   ("laplace2d:50/ir/m50", "laplace2d", 50, "ir"),
                                   ("laplace2d:100/ir/m50", "laplace2d", 100, "ir")):
        A = O.stencil_csr(kind, nx)
        b = O.ones_rhs(A.n_rows)
        dv = D.solve_ir(A, b, m=50) if solver == "ir" else D.solve_restarted(A, b, m=50)
        ref = O.solve_ir(A, b, m=50) if solver == "ir" else O.solve_restarted(A, b, m=50)
        assert dv.total_iters == golden_runs[name]["total_iters"] == ref.total_iters
        assert np.linalg.norm(dv.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
