"""GPU solver parity against the reference (via its recorded fixtures) and the
oracle, at sizes the oracle finishes in seconds.

North-star bars (BASELINE.json): iteration counts within +-2 % of the CPU
reference for the same solver, final fp64 relative residual <= rtol, and the
solution within 1e-8 relative of the reference's.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2109_01232_b200 as P
from oracle import cpu_gmres as O
from paper_2109_01232_b200 import _lib


def dev(Ao):
    return P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)


def within_2pct(got, want):
    return abs(got - want) <= max(0.02 * want, 0)


def _order_study():
    import json, os
    with open(os.path.join(os.path.dirname(__file__), "golden", "order_spread.json")) as f:
        return json.load(f)


ORDER_STUDY = _order_study()


def iters_match(rep, g, m, rtol=1e-10, name=None):
    """+-2 % of the reference count, or -- IR counts being quantised to whole
    restart cycles -- exactly one cycle off where the crossing
    is marginal: the side that did not converge at that boundary was within
    2x of rtol there.  Anything else is a parity failure.  (Cases whose count
    depends on the reduction order beyond this, e.g. laplace3d:40 GMRES-IR,
    are judged by ORDER_SENSITIVE below instead.)"""
    got, want = rep.total_iters, g["total_iters"]
    if within_2pct(got, want):
        return True
    if abs(got - want) != m:
        return False
    if got < want:   # we converged one cycle earlier than the reference
        ref_marks = {b[0]: b[2] for b in g["boundaries"]}
        return ref_marks.get(got, 1.0) <= 2 * rtol
    ours = {e.iteration: e.explicit for e in rep.residual_history if e.explicit is not None}
    return ours.get(want, 1.0) <= 2 * rtol


# Cases whose iteration count is decided by the association of the fp32 dot
# products: the reference needs 250 iterations for
# laplace3d:40 GMRES-IR, while blocked / pairwise / device-ordered sums of the
# same algorithm need 200 (tests/golden/order_spread.json).  For these the bar
# is the device-order oracle (oracle/devorder.c, the reference's algorithm
# with the kernels' association): the GPU solve must equal it BIT FOR BIT, and
# the oracle must reproduce the reference count with the reference's own
# order (test_oracle.py).  No band is widened.
ORDER_SENSITIVE = {"laplace3d:40/ir/m50"}


def rel_err(x, y):
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / np.linalg.norm(np.asarray(y)))


SOLVER_CASES = [
    # name, kind, nx, kwargs, solver, extra
    ("laplace2d:50/fp64/m50", "laplace2d", 50, {}, "fp64", {"m": 50}),
    ("laplace2d:50/ir/m50", "laplace2d", 50, {}, "ir", {"m": 50}),
    ("laplace2d:100/fp64/m50", "laplace2d", 100, {}, "fp64", {"m": 50}),
    ("laplace2d:100/ir/m50", "laplace2d", 100, {}, "ir", {"m": 50}),
    ("laplace2d:100/fd200/m50", "laplace2d", 100, {}, "fd", {"m": 50, "switch_iter": 200}),
    ("laplace2d:100/fp64/m25", "laplace2d", 100, {}, "fp64", {"m": 25}),
    ("laplace2d:100/ir/m25", "laplace2d", 100, {}, "ir", {"m": 25}),
    ("laplace2d:100/fp64/m100", "laplace2d", 100, {}, "fp64", {"m": 100}),
    ("laplace2d:100/ir/m100", "laplace2d", 100, {}, "ir", {"m": 100}),
    ("laplace3d:40/fp64/m50", "laplace3d", 40, {}, "fp64", {"m": 50}),
    ("laplace3d:40/ir/m50", "laplace3d", 40, {}, "ir", {"m": 50}),
    ("laplace3d:30/fd100/m50", "laplace3d", 30, {}, "fd", {"m": 50, "switch_iter": 100}),
    ("convdiff2d:100:c100/fp64/m50", "convdiff2d", 100, {"convection": 100.0}, "fp64", {"m": 50}),
    ("convdiff2d:100:c100/ir/m50", "convdiff2d", 100, {"convection": 100.0}, "ir", {"m": 50}),
    ("recirc2d:40:c0.5/ir/m50", "recirc2d", 40, {"convection": 0.5}, "ir", {"m": 50}),
]


def _nsm():
    return torch.cuda.get_device_properties(0).multi_processor_count


def run(A, b, solver, extra):
    crit = P.StopCriteria(rtol=1e-10, m=extra["m"], max_iters=extra.get("max_iters", 100_000))
    if solver == "fp64":
        return P.gmres_restarted(A, b, criteria=crit)
    if solver == "fp32":
        return P.gmres_restarted(A, b, criteria=crit, precision=P.FP32)
    if solver == "ir":
        return P.gmres_ir(A, b, criteria=crit)
    if solver == "fd":
        return P.gmres_fd(A, b, criteria=crit, switch_iter=extra["switch_iter"])
    raise ValueError(solver)


def oracle_run(Ao, b, solver, extra):
    m, mi = extra["m"], extra.get("max_iters", 100_000)
    if solver == "fp64":
        return O.solve_restarted(Ao, b, m=m, max_iters=mi)
    if solver == "fp32":
        return O.solve_restarted(Ao, b, m=m, max_iters=mi, dtype=np.float32)
    if solver == "ir":
        return O.solve_ir(Ao, b, m=m, max_iters=mi)
    return O.solve_fd(Ao, b, m=m, max_iters=mi, switch_iter=extra["switch_iter"])


@pytest.mark.parametrize("case", SOLVER_CASES, ids=[c[0] for c in SOLVER_CASES])
def test_solver_parity(case, golden_runs):
    name, kind, nx, kw, solver, extra = case
    Ao = O.stencil_csr(kind, nx, **kw)
    b = O.ones_rhs(Ao.n_rows)
    rep = run(dev(Ao), b, solver, extra)
    g = golden_runs[name]
    assert rep.converged == g["converged"]
    if name in ORDER_SENSITIVE:
        from oracle import devorder as D
        dv = {"ir": D.solve_ir, "fp64": D.solve_restarted}[solver](Ao, b, m=extra["m"], nsm=_nsm())
        assert rep.total_iters == dv.total_iters and np.array_equal(rep.x, dv.x), (rep.total_iters, dv.total_iters)
        study = ORDER_STUDY[name]
        assert study["device_order"] == dv.total_iters and study["counts"]["reference"] == g["total_iters"]
    else:
        assert iters_match(rep, g, extra["m"], name=name), (rep.total_iters, g["total_iters"], g["boundaries"][-3:])
    orep = oracle_run(Ao, b, solver, extra)
    assert orep.total_iters == g["total_iters"]          # oracle pinned to the reference
    assert rel_err(rep.x, orep.x) <= 1e-8
    rn, _ = O.residual(Ao, b, np.asarray(rep.x))
    assert rn / np.linalg.norm(b) <= 1e-10
    assert isinstance(rep.x, np.ndarray) and rep.x.dtype == np.float64
    assert len(rep.residual_history) >= 2
    assert rep.iters_fp32 + rep.iters_fp64 == rep.total_iters
    assert set(rep.kernel_times) == {"SpMV", "GemvTrans", "Norm", "GemvNoTrans", "Other"}


@pytest.mark.parametrize("solver,step", [("fp64", "split"), ("ir", "split"), ("ir", "persistent"),
                                         ("fp64", "persistent"), ("fd", "auto")])
def test_kernel_times_partition_total(solver, step):
    """SolveReport.kernel_times is the reference's partition of total_time
    (timing.py:40-47): the four kernel bins are filled from the device's
    globaltimer stamps -- each > 0 for these solves -- and Other is the
    remainder, so the five sum to total_time."""
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 40))
    b = np.ones(A.n_rows)
    crit = P.StopCriteria(rtol=1e-10, m=50)

    def solve():
        if solver == "fp64":
            return P.gmres_restarted(A, b, criteria=crit)
        if solver == "ir":
            return P.gmres_ir(A, b, criteria=crit)
        return P.gmres_fd(A, b, criteria=crit, switch_iter=100)

    with P.solvers.step_kernel(step):
        solve()   # warm: the first launch of each kernel in a process pays its module load
        rep = solve()
    kt = rep.kernel_times
    assert set(kt) == {"SpMV", "GemvTrans", "Norm", "GemvNoTrans", "Other"}
    for cat in ("SpMV", "GemvTrans", "Norm", "GemvNoTrans"):
        assert kt[cat] > 0, kt
    assert all(v >= 0 for v in kt.values())
    assert abs(sum(kt.values()) - rep.total_time) <= 1e-9 * max(1.0, rep.total_time) + 1e-12
    # the binned device time is most of the solve (graph-replayed cycles)
    assert sum(kt[c] for c in ("SpMV", "GemvTrans", "Norm", "GemvNoTrans")) >= 0.5 * rep.total_time, kt
    # CGS2 moves ~3 basis sweeps per step against one SpMV: the Gemv bins dominate
    assert kt["GemvTrans"] + kt["GemvNoTrans"] > kt["SpMV"], kt


def test_golden_235_and_determinism():
    Ao = O.stencil_csr("laplace2d", 50)
    A = dev(Ao)
    b = np.ones(Ao.n_rows)
    crit = P.StopCriteria(rtol=1e-10, m=50)
    r1 = P.gmres_restarted(A, b, criteria=crit)
    r2 = P.gmres_restarted(A, b, criteria=crit)
    assert r1.total_iters == 235                 # tests/test_solvers.py:16 GOLDEN_LAPLACE2D50_ITERS
    assert np.array_equal(r1.x, r2.x)            # bitwise reproducible (fixed-order reductions)
    assert r1.residual_history == r2.residual_history
    r3 = P.gmres_restarted(A, b, criteria=crit, use_graph=False)   # eager launches, same bits
    assert np.array_equal(r1.x, r3.x)


def test_device_inputs_stay_on_device():
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE2D, 40))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    rep = P.gmres_ir(A, b, criteria=P.StopCriteria(m=30))
    assert isinstance(rep.x, torch.Tensor) and rep.x.is_cuda
    assert rep.converged
    nr, _ = P.explicit_residual(A, b, rep.x)
    assert nr / float(torch.linalg.norm(b)) <= 1e-10


def test_ir_boundaries_and_fd_switch_zero():
    Ao = O.stencil_csr("laplace2d", 40)
    A, b = dev(Ao), np.ones(Ao.n_rows)
    crit = P.StopCriteria(rtol=1e-10, m=30)
    rep = P.gmres_ir(A, b, criteria=crit)
    marks = [e.iteration for e in rep.residual_history if e.explicit is not None]
    assert rep.total_iters in marks
    fd = P.gmres_fd(A, b, criteria=P.StopCriteria(m=50), switch_iter=0)
    dbl = P.gmres_restarted(A, b, criteria=P.StopCriteria(m=50))
    assert fd.total_iters == dbl.total_iters and np.array_equal(fd.x, dbl.x)
    assert fd.residual_history == dbl.residual_history
    fd = P.gmres_fd(A, b, criteria=P.StopCriteria(m=25), switch_iter=50)
    phases = [e.phase for e in fd.residual_history]
    assert sum(1 for a, c in zip(phases, phases[1:]) if a != c) == 1
    with pytest.raises(ValueError):
        P.gmres_fd(A, b, criteria=P.StopCriteria(m=50), switch_iter=75)


def test_fp32_plateau_and_stall(golden_runs):
    Ao = O.stencil_csr("laplace2d", 100)
    rep = P.gmres_restarted(dev(Ao), np.ones(Ao.n_rows), precision=P.FP32,
                            criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=5000))
    g = golden_runs["laplace2d:100/fp32/m50/max5000"]
    assert not rep.converged and rep.total_iters == 5000
    assert 1e-8 <= rep.best_explicit() <= 1e-4
    assert rep.x.dtype == np.float64
    assert rep.stalled_at is not None and g["stalled_at"] is not None
    Ao = O.stencil_csr("laplace2d", 20)
    rep = P.gmres_restarted(dev(Ao), np.ones(Ao.n_rows), criteria=P.StopCriteria(m=10, max_iters=15))
    assert not rep.converged and rep.total_iters == 15


def test_small_exact_cases():
    A = P.CsrMatrix.from_dense(np.eye(37))
    b = np.random.default_rng(3).standard_normal(37)
    rep = P.gmres_restarted(A, b)
    assert rep.converged and rep.total_iters == 1 and np.allclose(rep.x, b, atol=1e-12)
    A = P.CsrMatrix.from_dense(np.array([[4.0, 1.0], [1.0, 3.0]]))
    res = P.gmres_cycle(lambda v: P.spmv(A, v), np.array([1.0, 2.0]), np.zeros(2), 2, 1e-12)
    assert np.abs(res.x - [1.0 / 11.0, 7.0 / 11.0]).max() <= 1e-10
    A = P.CsrMatrix.from_dense(np.eye(8))
    b = np.zeros(8); b[0] = 2.5
    rep = P.gmres_ir(A, b)
    assert rep.converged and rep.iters_fp32 == 1
    with pytest.raises(P.PrecisionError):
        P.gmres_ir(P.convert_matrix(P.CsrMatrix.from_dense(np.eye(4)), P.FP32), np.ones(4))


def test_gmres_cycle_generic_operator_matches_oracle(rng):
    Ao = O.stencil_csr("convdiff2d", 30, convection=20.0)
    A = dev(Ao)
    b = rng.standard_normal(Ao.n_rows)
    cy = P.gmres_cycle(lambda v: P.spmv(A, v), b, np.zeros_like(b), 40, 1e-300)
    co = O.cycle(lambda v: O.spmv(Ao, v), b, np.zeros_like(b), 40, 1e-300)
    assert cy.steps == co.steps == 40
    assert np.allclose(cy.implicit_norms, co.implicit, rtol=1e-8)
    assert rel_err(cy.x, co.x) <= 1e-8


def test_ir_with_oracle_jacobi_and_poly(golden_runs):
    Ao = O.stencil_csr("convdiff2d", 60, convection=61.0)
    A, b = dev(Ao), np.ones(Ao.n_rows)
    Mo = O.jacobi_build(Ao.astype(np.float32), 1)
    rep = P.gmres_ir(A, b, precond_fp32=Mo)
    g = golden_runs["convdiff2d:60:c61/ir+jacobi1/m50"]
    assert rep.converged and iters_match(rep, g, 50), (rep.total_iters, g["total_iters"])
    Mdev = P.build_block_jacobi(P.convert_matrix(A, P.FP32), 1)
    rep2 = P.gmres_ir(A, b, precond_fp32=Mdev)
    assert rep2.total_iters == rep.total_iters and np.array_equal(rep2.x, rep.x)
    rep3 = P.gmres_ir(A, b, precond_fp32=P.build_block_jacobi(P.convert_matrix(A, P.FP32), 4))
    assert rep3.converged

    Ao = O.stencil_csr("laplace3d", 20)
    A, b = dev(Ao), np.ones(Ao.n_rows)
    for deg, key in ((5, "laplace3d:20/ir+poly5/m50"), (25, "laplace3d:20/ir+poly25/m50")):
        Mo = O.poly_build(Ao.astype(np.float32), deg, seed=0)
        rep = P.gmres_ir(A, b, precond_fp32=Mo)
        g = golden_runs[key]
        assert rep.converged
        assert abs(rep.total_iters - g["total_iters"]) <= max(1, int(0.02 * g["total_iters"])), (deg, rep.total_iters)
        orep = O.solve_ir(Ao, b, precond32=Mo)
        assert rel_err(rep.x, orep.x) <= 1e-8
    # fp32 polynomial inside an fp64 solve: cast_apply path, false convergence flagged
    Mo = O.poly_build(Ao.astype(np.float32), 25, seed=0)
    rep = P.gmres_restarted(A, b, precond=Mo)
    assert rep.loss_of_accuracy == golden_runs["laplace3d:20/fp64+poly25_32/m50"]["loss_of_accuracy"]


def test_divergence_is_raised():
    d = np.eye(4)
    d[2, 2] = np.inf
    A = P.CsrMatrix.from_dense(d)
    with pytest.raises(P.DivergenceError):
        P.gmres_restarted(A, np.ones(4))


def test_native_code_launched():
    before = _lib.launch_count()
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE2D, 30))
    P.gmres_ir(A, np.ones(A.n_rows))
    assert _lib.launch_count() - before > 100


@pytest.mark.parametrize("solver", ["fp64", "ir", "fd"])
def test_stencil_storage_solves_same_iterate_as_csr(solver):
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 24))
    b = np.ones(A.n_rows)
    kw = {"criteria": P.StopCriteria(m=30)}
    f = {"fp64": P.gmres_restarted, "ir": P.gmres_ir,
         "fd": lambda A, b, **k: P.gmres_fd(A, b, switch_iter=60, **k)}[solver]
    with P.solvers.step_kernel("split"):     # the same Arnoldi kernels for both storages
        r_csr = f(A, b, storage="csr", **kw)
        r_st = f(A, b, storage="stencil", **kw)
    assert r_csr.total_iters == r_st.total_iters
    # the SpMV is bit-identical and every Arnoldi reduction runs in the same
    # kernels on the same grid, so the iterate is bitwise the same; only the
    # explicit-residual norm is summed in a storage-dependent row order
    # (CSR 512-row tiles vs stencil 16-byte row groups), so history norms may
    # differ in the last bits
    assert np.array_equal(r_csr.x, r_st.x)
    assert len(r_csr.residual_history) == len(r_st.residual_history)
    for a, b_ in zip(r_csr.residual_history, r_st.residual_history):
        assert a.iteration == b_.iteration and a.phase == b_.phase
        assert abs(a.implicit - b_.implicit) <= 1e-12 * abs(a.implicit)
        if a.explicit is None:
            assert b_.explicit is None
        else:
            assert abs(a.explicit - b_.explicit) <= 1e-12 * abs(a.explicit)


def test_stencil_storage_with_preconditioners():
    Ao = O.stencil_csr("laplace3d", 16)
    A, b = dev(Ao), np.ones(Ao.n_rows)
    for M in (O.poly_build(Ao.astype(np.float32), 12, seed=0), O.jacobi_build(Ao.astype(np.float32), 1)):
        with P.solvers.step_kernel("split"):
            r1 = P.gmres_ir(A, b, precond_fp32=M, storage="csr")
            r2 = P.gmres_ir(A, b, precond_fp32=M, storage="stencil")
        assert r1.total_iters == r2.total_iters and np.array_equal(r1.x, r2.x)
        # the persistent step (Jacobi(1) folded into its scaling phase) agrees to rounding
        r3 = P.gmres_ir(A, b, precond_fp32=M, storage="stencil")
        assert abs(r3.total_iters - r1.total_iters) <= 1 and np.linalg.norm(r3.x - r1.x) <= 1e-9 * np.linalg.norm(r1.x)


@pytest.fixture(scope="module")
def cfg2_reference():
    from conftest import load_json
    return load_json("reference_cfg2.json")["runs"]


@pytest.mark.parametrize("solver", ["ir", "fp64", "fd1000"])
def test_cfg2_laplace3d150_full_solve_vs_reference(solver, cfg2_reference):
    """BASELINE configs[1] at full size against the reference's own runs
    (tests/golden/reference_cfg2.json: 2387 fp64 / 2400 IR / 2316 GMRES-FD
    switching at 1000 iterations; ~20 / ~13 / ~10 CPU-minutes): same count (+-2 %), every restart-boundary
    residual within 2x, final fp64 residual <= 1e-10, solution within 1e-8
    relative on a 4101-point strided sample."""
    g = cfg2_reference[f"laplace3d:150/{solver}/m50"]
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 150))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50)
    if solver == "ir":
        rep = P.gmres_ir(A, b, criteria=crit)
    elif solver == "fp64":
        rep = P.gmres_restarted(A, b, criteria=crit)
    else:
        rep = P.gmres_fd(A, b, criteria=crit, switch_iter=int(solver[2:]))
    assert rep.converged
    assert iters_match(rep, g, 50, name=f"laplace3d:150/{solver}/m50"), (rep.total_iters, g["total_iters"],
                                                                         rep.iters_fp32, g["iters_fp32"])
    # residual trajectory: within 2x of the reference at every restart boundary
    # while it is well above the tolerance; in the last cycles the per-cycle
    # reduction swings with the summation order (e.g. cfg3 IR: 6.1e-10 ->
    # 3.5e-10 -> 8.2e-11), so there only the count rule above applies
    ours = {e.iteration: e.explicit for e in rep.residual_history if e.explicit is not None}
    for it, _, ref_exp, _ in g["boundaries"]:
        if it in ours and it > 0 and ref_exp > 100 * 1e-10:
            assert 0.5 <= ours[it] / ref_exp <= 2.0, (it, ours[it], ref_exp)
    nr, _ = P.explicit_residual(A, b, rep.x)
    assert nr / float(torch.linalg.norm(b)) <= 1e-10
    x = rep.x.cpu().numpy()[:: g["x_stride"]]
    ref = np.asarray(g["x_sample"])
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-8
    assert abs(float(torch.linalg.norm(rep.x)) - g["x_norm"]) / g["x_norm"] <= 1e-8


@pytest.fixture(scope="module")
def cfg3_reference():
    from conftest import load_json
    return load_json("reference_cfg3.json")["runs"]


@pytest.mark.parametrize("solver", ["ir+jacobi1", "fp64"])
def test_cfg3_convdiff1500_full_solve_vs_reference(solver, cfg3_reference):
    """BASELINE configs[2] at full size (UniFlow2D = convdiff2d:1500 with
    convection 1501, 2.25M rows, nonsymmetric) against the reference's own run
    (tests/golden/reference_cfg3.json: 2744 fp64 / 3100 IR + fp32 Jacobi(1)
    iterations, ~14 CPU-minutes each): same count (+-2 % or the marginal-cycle
    rule), boundary residuals within 2x, final fp64 residual <= 1e-10,
    solution within 1e-8 relative on the strided sample."""
    g = cfg3_reference[f"convdiff2d:1500:c1501/{solver}/m50"]
    A = P.generate(P.StencilSpec(P.StencilKind.CONVDIFF2D, 1500, convection=1501.0))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50)
    if solver == "fp64":
        rep = P.gmres_restarted(A, b, criteria=crit)
    else:
        M = P.build_block_jacobi(P.convert_matrix(A, P.FP32), 1)
        rep = P.gmres_ir(A, b, criteria=crit, precond_fp32=M)
    assert rep.converged
    assert iters_match(rep, g, 50), (rep.total_iters, g["total_iters"], g["boundaries"][-3:])
    # residual trajectory: within 2x of the reference at every restart boundary
    # while it is well above the tolerance; in the last cycles the per-cycle
    # reduction swings with the summation order (e.g. cfg3 IR: 6.1e-10 ->
    # 3.5e-10 -> 8.2e-11), so there only the count rule above applies
    ours = {e.iteration: e.explicit for e in rep.residual_history if e.explicit is not None}
    for it, _, ref_exp, _ in g["boundaries"]:
        if it in ours and it > 0 and ref_exp > 100 * 1e-10:
            assert 0.5 <= ours[it] / ref_exp <= 2.0, (it, ours[it], ref_exp)
    nr, _ = P.explicit_residual(A, b, rep.x)
    assert nr / float(torch.linalg.norm(b)) <= 1e-10
    x = rep.x.cpu().numpy()[:: g["x_stride"]]
    ref = np.asarray(g["x_sample"])
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-8


@pytest.mark.parametrize("name,kind,nx,kw,solver", [
    ("laplace3d:40/ir/m50", "laplace3d", 40, {}, "ir"), ("laplace3d:40/fp64/m50", "laplace3d", 40, {}, "fp64"),
    ("laplace2d:100/ir/m50", "laplace2d", 100, {}, "ir"),
    ("convdiff2d:100:c100/fp64/m50", "convdiff2d", 100, {"convection": 100.0}, "fp64")])
def test_persistent_step_kernel_matches_split_step(name, kind, nx, kw, solver, golden_runs):
    """The persistent per-step kernel (csrc/step_kernel.cu) and the four-launch
    step compute the same CGS2 step with differently ordered reductions.  Both
    must converge at the reference's count (iters_match) -- or, for the
    order-sensitive laplace3d:40 GMRES-IR, at the device-order count, the
    persistent one bit for bit -- with solutions within 1e-9 of each other and
    final fp64 residuals <= rtol."""
    A = P.generate(P.StencilSpec(P.StencilKind(kind), nx, **kw))
    b = np.ones(A.n_rows)
    crit = P.StopCriteria(rtol=1e-10, m=50)
    f = P.gmres_ir if solver == "ir" else P.gmres_restarted
    with P.solvers.step_kernel("split"):
        r1 = f(A, b, criteria=crit)
    with P.solvers.step_kernel("persistent"):
        r2 = f(A, b, criteria=crit)
    g = golden_runs[name]
    assert r1.converged and r2.converged
    if name in ORDER_SENSITIVE:
        from oracle import devorder as D
        Ao = O.stencil_csr(kind, nx, **kw)
        dv = D.solve_ir(Ao, b, m=50, nsm=_nsm())
        assert r2.total_iters == dv.total_iters and np.array_equal(r2.x, dv.x)
        assert r1.total_iters == dv.total_iters, (r1.total_iters, dv.total_iters)
    else:
        assert iters_match(r1, g, 50), (r1.total_iters, g["total_iters"])
        assert iters_match(r2, g, 50), (r2.total_iters, g["total_iters"])
    assert rel_err(r2.x, r1.x) <= 1e-9
    for r in (r1, r2):
        rn, _ = P.explicit_residual(A, b, r.x)
        assert rn / np.linalg.norm(b) <= 1e-10


@pytest.fixture(scope="module")
def cfg4_reference():
    from conftest import load_json
    return {d: load_json(f"reference_cfg4_poly{d}.json")["runs"][f"laplace3d:200/ir+poly{d}/m50"] for d in (25, 40)}


def _cycle_lengths(history):
    b = [e.iteration for e in history if e.explicit is not None]
    return [y - x for x, y in zip(b, b[1:])]


@pytest.mark.parametrize("degree", [25, 40])
@pytest.mark.parametrize("build", ["oracle", "device"])
def test_cfg4_laplace3d200_ir_poly_vs_reference(degree, build, cfg4_reference):
    """BASELINE configs[3] at full size: GMRES-IR + GMRES-polynomial(25 / 40)
    on Laplace3D 200^3 (8M rows) against the reference's own runs
    (tests/golden/reference_cfg4_poly*.json: 131 / 85 iterations in 3 restart
    cycles, ~30 CPU-minutes each).  The inner cycles end early at the implicit
    threshold, so each cycle's length is the step at which the implicit
    residual crosses rtol*||r32||; a crossing that lands one step apart is the
    same quantisation as an IR restart boundary.  Bar: the same number of
    cycles, the first cycle (identical start) within +-1 step of the
    reference's, the total within +-2 % or +-1 per cycle, final fp64 residual
    <= rtol, solution within 1e-8.
    'oracle' applies the reference-identical preconditioner (oracle
    poly_build); 'device' builds it with device Arnoldi steps."""
    g = cfg4_reference[degree]
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 200))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    if build == "oracle":
        rp, ci, v = A.host_arrays()
        M = O.poly_build(O.Csr(A.n_rows, A.n_cols, rp, ci, v.astype(np.float32)), degree, seed=0)
    else:
        M = P.build_poly_precond(P.convert_matrix(A, P.FP32), degree, seed=0)
    rep = P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50), precond_fp32=M)
    assert rep.converged
    ours, ref = _cycle_lengths(rep.residual_history), _cycle_lengths(
        [P.HistoryEntry(it, imp, exp, ph) for it, imp, exp, ph in g["boundaries"]])
    assert len(ours) == len(ref), (ours, ref)
    assert abs(ours[0] - ref[0]) <= 1, (ours, ref)
    assert abs(rep.total_iters - g["total_iters"]) <= max(0.02 * g["total_iters"], len(ref))
    nr, _ = P.explicit_residual(A, b, rep.x)
    assert nr / float(torch.linalg.norm(b)) <= 1e-10
    x = rep.x.cpu().numpy()[:: g["x_stride"]]
    sample = np.asarray(g["x_sample"])
    assert np.linalg.norm(x - sample) / np.linalg.norm(sample) <= 1e-8
    print(f"cfg4 poly{degree} ({build} build): {rep.total_iters} it {ours} vs reference "
          f"{g['total_iters']} {ref}")


def test_cfg5_laplace3d400_assembly_and_first_ir_cycle_vs_reference():
    """BASELINE configs[4] (Laplace3D 400^3, 64M rows, 447M nonzeros) on one
    B200.  A full reference solve is ~40 CPU-hours, so the reference pinned
    (tests/golden/reference_cfg5.json) the assembly, its first GMRES-IR cycle
    and its first fp64 GMRES(50) cycle.  Here: device assembly bit-exact by
    sha256; the first IR cycle's explicit residual within 0.1 % of the
    reference's; and the iterate against the fp64 cycle, which in exact
    arithmetic is the same Krylov iterate (x0 = 0, same b): ours within 1e-4.
    The reference's own fp32 cycle is 0.9 % away from it -- its sequential
    single-precision BLAS dot products over 64M entries lose the smooth-mode
    coefficient (kappa ~ 6.5e4), which our tree reductions keep; the test
    records that too."""
    import hashlib
    from conftest import load_json
    g = load_json("reference_cfg5.json")
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 400))
    asm = g["assembly"]
    assert (A.n_rows, A.nnz) == (asm["n"], asm["nnz"])
    for name, t in (("row_ptr", A.row_ptr), ("col_idx", A.col_idx), ("values", A.values)):
        assert hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest() == asm[name], name
    ref_ir = g["runs"]["laplace3d:400/ir/m50/max50"]
    ref64 = g["runs"]["laplace3d:400/fp64/m50/max50"]
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    rep = P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=50))
    assert rep.total_iters == ref_ir["total_iters"] == 50
    ours = [e.explicit for e in rep.residual_history if e.explicit is not None]
    theirs = [bd[2] for bd in ref_ir["boundaries"]]
    assert len(ours) == len(theirs) and abs(ours[-1] / theirs[-1] - 1) <= 1e-3, (ours, theirs)
    stride = ref_ir["x_stride"]
    x = rep.x.cpu().numpy()[::stride]
    x64 = np.asarray(ref64["x_sample"])
    xir = np.asarray(ref_ir["x_sample"])
    ours_err = np.linalg.norm(x - x64) / np.linalg.norm(x64)
    ref_err = np.linalg.norm(xir - x64) / np.linalg.norm(x64)
    assert ours_err <= 1e-4, ours_err
    assert ref_err > 10 * ours_err, (ref_err, ours_err)


@pytest.mark.parametrize("kind,nx,kw,const", [("laplace3d", 33, {}, True), ("laplace2d", 61, {}, True),
                                              ("convdiff2d", 101, {"convection": 1501.0}, True),
                                              ("recirc2d", 49, {"convection": 0.5}, False)])
def test_constant_coefficient_stencil_path_is_bitwise_the_packed_path(kind, nx, kw, const):
    """Stencils with one coefficient per slot (Laplace, uniform convection) take
    the coefficient-stream SpMV (csrc/spmv.cuh StencilConst: x only, presence
    from grid coordinates); the iterate and history equal the packed-values
    path bit for bit.  Position-dependent stencils (Recirc2D) keep the values."""
    spec = P.StencilSpec(P.StencilKind(kind), nx, **kw)
    reps, flags = [], []
    for on in (True, False):
        prev, P.core.STENCIL_CONST = P.core.STENCIL_CONST, on
        try:
            A = P.generate(spec)
            b = np.ones(A.n_rows)
            flags.append(P.convert_matrix(A, P.FP32).stencil_const())
            reps.append(P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=30, max_iters=600)))
        finally:
            P.core.STENCIL_CONST = prev
    assert flags == [const, False]
    a, b_ = reps
    assert a.total_iters == b_.total_iters
    assert np.array_equal(a.x, b_.x)
    assert [(e.iteration, e.implicit, e.explicit) for e in a.residual_history] == \
           [(e.iteration, e.implicit, e.explicit) for e in b_.residual_history]


@pytest.mark.timeout(600)
def test_persistent_step_barrier_reuse_across_grids():
    """The persistent step's grid barrier counts arrivals on a monotonic
    per-solver counter (csrc/step_kernel.cu grid_barrier_mono): interleave
    solvers whose step grids differ (G = 13 ... 148 CTAs, fp32 and fp64, cycles
    ending early at convergence) and repeat each solve -- every repeat must be
    bitwise identical to the first and no launch may hang."""
    crit = P.StopCriteria(rtol=1e-10, m=50)
    cases = [(P.StencilKind.LAPLACE2D, 40), (P.StencilKind.LAPLACE3D, 30), (P.StencilKind.LAPLACE2D, 120),
             (P.StencilKind.LAPLACE3D, 14)]
    mats = [P.generate(P.StencilSpec(k, nx)) for k, nx in cases]
    first = {}
    with P.solvers.step_kernel("persistent"):
        for rep in range(2):
            for ci, A in enumerate(mats):
                b = np.ones(A.n_rows)
                for name, f in (("ir", P.gmres_ir), ("fp64", P.gmres_restarted)):
                    r = f(A, b, criteria=crit)
                    assert r.converged
                    key = (ci, name)
                    if rep == 0:
                        first[key] = (r.total_iters, np.asarray(r.x).copy())
                    else:
                        assert r.total_iters == first[key][0]
                        assert np.array_equal(np.asarray(r.x), first[key][1])
