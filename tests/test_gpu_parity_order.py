"""GPU parity beyond iteration counts.

1. Bitwise: the single-GPU solves (persistent step kernel) equal the
   device-order oracle (oracle/devorder.c: the reference's algorithm with
   the kernels' association of every reduction) bit for bit -- iterate and
   every history entry.  With test_oracle.py (the same oracle code with the
   reference's association reproduces the reference's counts and solution
   sha256) this pins any count difference from the reference on the
   reduction order alone: laplace3d:40 GMRES-IR takes 250 iterations in the
   reference's sequential-BLAS order and 200 in the device's.
2. The reference's CGS2 acceptance criterion 03 (tests/test_acceptance.py:
   97-126, tests/test_krylov.py:59-71) on the basis the DEVICE built: ||V^T V
   - I||_max <= 100 u m and ||A V_m - V_{m+1} H||_F <= 100 u ||A||_F m, fp32 and
   fp64, for both step kernels.
3. Criterion 02 (GMRES optimality, tests/test_acceptance.py:72-94) on native
   device cycles: implicit residuals equal the brute-force Krylov minima.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import _lib
from paper_2109_01232_b200.krylov import HessenbergLS
from paper_2109_01232_b200.solvers import NativeSolve
from oracle import cpu_gmres as O
from oracle import devorder as D


def _nsm():
    return torch.cuda.get_device_properties(0).multi_processor_count


BITWISE_CASES = [
    # name, kind, nx, kwargs, solver, extra
    ("laplace2d:50/fp64", "laplace2d", 50, {}, "fp64", {}),
    ("laplace2d:50/ir", "laplace2d", 50, {}, "ir", {}),
    ("laplace2d:100/ir", "laplace2d", 100, {}, "ir", {}),
    ("laplace2d:100/fd200", "laplace2d", 100, {}, "fd", {"switch_iter": 200}),
    ("laplace2d:100/fp32/max300", "laplace2d", 100, {}, "fp32", {"max_iters": 300}),
    ("laplace3d:30/fd100", "laplace3d", 30, {}, "fd", {"switch_iter": 100}),
    ("laplace3d:40/ir", "laplace3d", 40, {}, "ir", {}),
    ("laplace3d:40/fp64", "laplace3d", 40, {}, "fp64", {}),
    ("convdiff2d:100:c100/fp64", "convdiff2d", 100, {"convection": 100.0}, "fp64", {}),
    ("convdiff2d:100:c100/ir", "convdiff2d", 100, {"convection": 100.0}, "ir", {}),
    ("recirc2d:40:c0.5/ir", "recirc2d", 40, {"convection": 0.5}, "ir", {}),
]


@pytest.mark.parametrize("case", BITWISE_CASES, ids=[c[0] for c in BITWISE_CASES])
def test_gpu_solve_is_bitwise_the_device_order_oracle(case):
    name, kind, nx, kw, solver, extra = case
    Ao = O.stencil_csr(kind, nx, **kw)
    b = O.ones_rhs(Ao.n_rows)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    mi = extra.get("max_iters", 100_000)
    crit = P.StopCriteria(rtol=1e-10, m=50, max_iters=mi)
    nsm = _nsm()
    with P.solvers.step_kernel("persistent"):
        if solver == "ir":
            rep = P.gmres_ir(A, b, criteria=crit)
            dv = D.solve_ir(Ao, b, m=50, max_iters=mi, nsm=nsm)
        elif solver == "fd":
            rep = P.gmres_fd(A, b, criteria=crit, switch_iter=extra["switch_iter"])
            dv = D.solve_fd(Ao, b, m=50, max_iters=mi, switch_iter=extra["switch_iter"], nsm=nsm)
        else:
            prec = P.FP32 if solver == "fp32" else P.FP64
            rep = P.gmres_restarted(A, b, criteria=crit, precision=prec)
            dv = D.solve_restarted(Ao, b, m=50, max_iters=mi, nsm=nsm,
                                   dtype=np.float32 if solver == "fp32" else np.float64)
    assert (rep.total_iters, rep.iters_fp32, rep.iters_fp64) == (dv.total_iters, dv.iters_fp32, dv.iters_fp64)
    assert rep.converged == dv.converged
    ours = [(e.iteration, e.implicit, e.explicit, e.phase) for e in rep.residual_history]
    assert ours == dv.history
    assert np.array_equal(rep.x, dv.x)


def test_order_sensitive_case_counts():
    """laplace3d:40 GMRES-IR: the reference-order oracle (pinned to the
    reference) needs 250 iterations, the device-order oracle 200 -- the same
    algorithm, only the association of the fp32 reductions differs -- and
    the GPU (bitwise equal to the device-order oracle above) needs 200."""
    Ao = O.stencil_csr("laplace3d", 40)
    b = O.ones_rhs(Ao.n_rows)
    assert O.solve_ir(Ao, b, m=50).total_iters == 250
    assert D.solve_ir(Ao, b, m=50, nsm=_nsm()).total_iters == 200
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 40))
    assert P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50)).total_iters == 200


# ----------------------------------------------------------------- CGS2 acceptance


def _device_cycle(A, prec, b, m, mode):
    """One native restart cycle of m steps from x0 = 0 (no early stop); returns
    (V as n x (k+1) fp64, H (k+1) x k fp64, steps)."""
    Ap = A if A.precision is prec else P.convert_matrix(A, prec)
    n = A.n_rows
    bd = P.solvers.padded_copy(P.convert_vector(b, prec) if prec is P.FP32 else b, prec)
    xd = P.solvers.dvec(n, prec)
    with P.solvers.step_kernel(mode):
        ns = NativeSolve(_lib.MODE_RESTARTED, prec, Ap, None, bd, xd, m, 1e-300)
    try:
        ns.begin()
        hdr, _ = ns.cycle(m)
        k = int(hdr.steps)
        V = ns.V.view(m + 1, ns.ldv)[: k + 1, :n].double().cpu().numpy().T
        H = HessenbergLS(ns.state).H[: k + 1, :k].astype(np.float64)
        storage = ns.storage
    finally:
        ns.close()
    return V, H, k, storage


def _random_csr(n, seed):
    r = np.random.default_rng(seed)
    d = r.standard_normal((n, n)) * (r.random((n, n)) < 0.02)
    d += 5.0 * np.eye(n)
    return P.CsrMatrix.from_dense(d), d


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("mode", ["persistent", "split"])
@pytest.mark.parametrize("matrix", ["laplace2d:50", "laplace3d:24", "convdiff2d:60:c61", "random-csr:500"])
def test_cgs2_orthogonality_and_arnoldi_relation_on_device_basis(prec, mode, matrix):
    """Criterion 03 of the reference (tests/test_acceptance.py:97-126) on V and
    H read back from the device after a 50-step cycle."""
    m = 50
    prec = P.FP32 if prec == "fp32" else P.FP64
    if matrix.startswith("random"):
        if mode == "persistent":
            pytest.skip("the persistent step kernel runs on stencil storage only")
        A, _ = _random_csr(500, 3)
    else:
        kind, nx, *rest = matrix.split(":")
        kw = {"convection": float(rest[0][1:])} if rest else {}
        A = P.generate(P.StencilSpec(P.StencilKind(kind), int(nx), **kw))
    b = np.random.default_rng(3).standard_normal(A.n_rows)
    V, H, k, storage = _device_cycle(A, prec, b, m, mode)
    assert k == m
    if not matrix.startswith("random"):
        assert storage.startswith("stencil")
    u = prec.unit_roundoff
    gram = np.abs(V.T @ V - np.eye(m + 1)).max()
    assert gram <= 100 * u * m, gram
    Ap = A if A.precision is prec else P.convert_matrix(A, prec)
    rp, ci, vals = Ap.host_arrays()
    Ao = O.Csr(A.n_rows, A.n_cols, rp, ci, vals)
    AV = np.column_stack([O.spmv(Ao, V[:, j].astype(prec.dtype)) for j in range(m)]).astype(np.float64)
    frob = np.linalg.norm(AV - V @ H, "fro")
    a_frob = float(np.linalg.norm(vals.astype(np.float64)))
    assert frob <= 100 * u * a_frob * m, (frob, 100 * u * a_frob * m)


def test_native_cycle_gmres_optimality():
    """Criterion 02 (tests/test_acceptance.py:72-94) on native device cycles:
    each implicit residual equals the brute-force minimum over the Krylov space
    (dense QR basis + dense least squares) to 1e-8 relative."""
    rng = np.random.default_rng(20260811)
    worst = 0.0
    for _ in range(6):
        n = int(rng.integers(60, 201))
        Ad = np.eye(n) * 1.2 + rng.standard_normal((n, n)) / np.sqrt(n)
        b = rng.standard_normal(n)
        A = P.CsrMatrix.from_dense(Ad)
        jmax = min(n, 30)
        xd = P.solvers.dvec(n, P.FP64)
        ns = NativeSolve(_lib.MODE_RESTARTED, P.FP64, A, None, P.solvers.padded_copy(b, P.FP64), xd, jmax, 1e-300)
        try:
            bn, _ = ns.begin()
            hdr, imp = ns.cycle(jmax)
        finally:
            ns.close()
        assert hdr.steps == jmax
        K = np.zeros((n, jmax))
        K[:, 0] = b
        for j in range(1, jmax + 1):
            Q, _ = np.linalg.qr(K[:, :j])
            if j < jmax:
                K[:, j] = Ad @ Q[:, j - 1]
            M = Ad @ Q
            c, *_ = np.linalg.lstsq(M, b, rcond=None)
            best = np.linalg.norm(b - M @ c)
            worst = max(worst, abs(imp[j - 1] - best) / best)
    assert worst <= 1e-8, worst
