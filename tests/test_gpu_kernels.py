"""GPU parity of the L1 kernels against the oracle / reference fixtures.

Bit-exact: SpMV (numpy add.reduceat order), explicit residual vector,
stencil assembly (pattern + value bits, also at the config sizes via the
reference's sha256), casts, Jacobi(1) apply, polynomial apply.
Tolerance-based: reductions (norms, multi-dots), whose order differs from
OpenBLAS by design.
"""

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2109_01232_b200 as P
from oracle import cpu_gmres as O
from paper_2109_01232_b200 import _lib


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def dev_csr(c):
    return P.CsrMatrix(len(c["row_ptr"]) - 1, len(c["x"]), c["row_ptr"], c["col_idx"], c["values"])


def test_spmv_bitexact_on_reference_fixtures(spmv_cases):
    assert len(spmv_cases) >= 16
    for (name, prec), c in sorted(spmv_cases.items()):
        A = dev_csr(c)
        y = P.spmv(A, torch.from_numpy(c["x"]).cuda()).cpu().numpy()
        assert bits_equal(y, c["y"]), (name, prec)
        # numpy in -> numpy out through the same kernel
        assert bits_equal(P.spmv(A, c["x"]), c["y"])


@pytest.mark.parametrize("kind,nx,kw", [("laplace3d", 33, {}), ("convdiff2d", 101, {"convection": 1501.0}),
                                        ("recirc2d", 77, {"convection": 40.1}), ("laplace2d", 129, {})])
def test_spmv_bitexact_vs_oracle_multi_tile(kind, nx, kw, rng):
    Ao = O.stencil_csr(kind, nx, **kw)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    for dt in (np.float64, np.float32):
        Ad = A if dt == np.float64 else P.convert_matrix(A, P.FP32)
        x = rng.standard_normal(Ao.n_cols).astype(dt)
        y = P.spmv(Ad, x)
        assert bits_equal(y, O.spmv(Ao.astype(dt), x)), (kind, dt)


def test_spmv_edge_cases():
    # empty rows, empty matrix rows at the end, single row, identity
    d = np.zeros((5, 5)); d[1, 2] = 3.0; d[3, 0] = -1.0
    A = P.CsrMatrix.from_dense(d)
    assert np.array_equal(P.spmv(A, np.ones(5)), [0.0, 3.0, 0.0, -1.0, 0.0])
    A = P.CsrMatrix.from_dense(np.eye(3))
    assert np.array_equal(P.spmv(A, np.array([1.0, 2.0, 3.0])), [1.0, 2.0, 3.0])
    t = np.diag(np.full(4, 2.0)) + np.diag(np.full(3, -1.0), 1) + np.diag(np.full(3, -1.0), -1)
    assert np.array_equal(P.spmv(P.CsrMatrix.from_dense(t), np.ones(4)), [1.0, 0.0, 0.0, 1.0])
    with pytest.raises(P.ShapeError):
        P.spmv(A, np.ones(4))
    with pytest.raises(P.PrecisionError):
        P.spmv(A, np.ones(3, dtype=np.float32))


def test_explicit_residual_bitexact_vector(rng):
    Ao = O.stencil_csr("laplace3d", 21)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    b = rng.standard_normal(Ao.n_rows)
    x = rng.standard_normal(Ao.n_rows)
    nr, r = P.explicit_residual(A, b, x)
    nr_o, r_o = O.residual(Ao, b, x)
    assert bits_equal(r, r_o)
    assert nr == pytest.approx(nr_o, rel=1e-13)


def test_norm2_and_gemv(rng):
    for dt, tol in ((np.float64, 1e-13), (np.float32, 2e-6)):
        x = rng.standard_normal(100_003).astype(dt)
        assert P.norm2(x) == pytest.approx(float(np.linalg.norm(x.astype(np.float64))), rel=tol)
        V = np.asfortranarray(rng.standard_normal((5000, 37)).astype(dt))
        w = rng.standard_normal(5000).astype(dt)
        c = P.gemv(V, w, transpose=True)
        ref = V.astype(np.float64).T @ w.astype(np.float64)
        assert np.allclose(c, ref, rtol=tol * 50, atol=tol * 50 * np.abs(V).sum(0).max())
        d = rng.standard_normal(37).astype(dt)
        y = rng.standard_normal(5000).astype(dt)
        out = P.gemv(V, d, y.copy(), alpha=-1.0, beta=1.0)
        ref = y.astype(np.float64) - V.astype(np.float64) @ d.astype(np.float64)
        assert np.allclose(out, ref, rtol=tol * 50, atol=tol * 100 * 37)
    assert P.norm2(np.array([3.0, 4.0])) == 5.0
    assert P.norm2(np.zeros(0)) == 0.0


def test_convert_bitexact_and_overflow(rng):
    x = rng.standard_normal(10_001) * 1e3
    y = P.convert_vector(x, P.FP32)
    assert bits_equal(y, x.astype(np.float32))
    assert bits_equal(P.convert_vector(y, P.FP64), y.astype(np.float64))
    bad = np.ones(100); bad[37] = 1e300; bad[80] = -1e300
    with pytest.raises(P.PrecisionOverflowError, match="entry 37"):
        P.convert_vector(bad, P.FP32)
    Ao = O.stencil_csr("recirc2d", 31, convection=7.0)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    A32 = P.convert_matrix(A, P.FP32)
    assert bits_equal(A32.values.cpu().numpy(), Ao.values.astype(np.float32))
    assert A32.row_ptr.data_ptr() == A.row_ptr.data_ptr()   # pattern shared


@pytest.mark.parametrize("kind", list(_lib.STENCIL_KIND))
def test_generator_bitexact_small(kind):
    kw = {"convection": 40.1} if kind in ("convdiff2d", "recirc2d") else {}
    for nx in (2, 3, 9, 31):
        Ao = O.stencil_csr(kind, nx, **kw)
        A = P.generate(P.StencilSpec(P.StencilKind(kind), nx, **kw))
        rp, ci, v = A.host_arrays()
        assert bits_equal(rp, Ao.row_ptr) and bits_equal(ci, Ao.col_idx) and bits_equal(v, Ao.values), (kind, nx)


def test_generator_row_slices():
    spec = P.StencilSpec(P.StencilKind.LAPLACE3D, 19)
    Ao = O.stencil_csr("laplace3d", 19)
    for a, b in ((0, 361), (361, 5000), (5000, 6859), (1234, 1235)):
        rp, ci, v = P.gen.generate_rows(spec, a, b)
        base = Ao.row_ptr[a]
        assert np.array_equal(rp.cpu().numpy(), Ao.row_ptr[a:b + 1] - base)
        assert np.array_equal(ci.cpu().numpy(), Ao.col_idx[Ao.row_ptr[a]:Ao.row_ptr[b]])
        assert bits_equal(v.cpu().numpy(), Ao.values[Ao.row_ptr[a]:Ao.row_ptr[b]])


def test_generator_config_sizes_match_reference_sha256(golden_assembly):
    for key, g in golden_assembly.items():
        A = P.generate(P.StencilSpec(P.StencilKind(g["kind"]), g["nx"], **g["kwargs"]))
        assert (A.n_rows, A.nnz) == (g["n"], g["nnz"]), key
        rp, ci, v = A.host_arrays()
        assert sha(rp) == g["row_ptr"], key
        assert sha(ci) == g["col_idx"], key
        assert sha(v) == g["values"], key
        del A


def test_jacobi_build_and_apply(rng):
    Ao = O.stencil_csr("convdiff2d", 40, convection=31.0)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    A32 = P.convert_matrix(A, P.FP32)
    A32o = Ao.astype(np.float32)
    x = rng.standard_normal(Ao.n_rows).astype(np.float32)
    for k in (1, 3, 4, 7):
        Mo = O.jacobi_build(A32o, k)
        M = P.build_block_jacobi(A32, k)
        assert np.array_equal(M.block_piv.cpu().numpy(), Mo.block_piv)
        assert np.allclose(M.block_lu.cpu().numpy(), Mo.block_lu, rtol=1e-5, atol=1e-6)
        y = P.apply_block_jacobi(Mo, x)       # oracle factors, device apply
        yo = O.jacobi_apply(Mo, x)
        if k == 1:
            assert bits_equal(y, yo)
        else:
            assert np.allclose(y, yo, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("degree", [0, 3, 10, 12, 25])
def test_poly_apply_matches_oracle(degree, rng):
    Ao = O.stencil_csr("laplace3d", 12)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    for dt in (np.float32, np.float64):
        Ad = A if dt == np.float64 else P.convert_matrix(A, P.FP32)
        Mo = O.poly_build(Ao.astype(dt), degree, seed=0)
        x = rng.standard_normal(Ao.n_rows).astype(dt)
        before = _lib.launch_count()
        y = P.apply_poly(Mo, Ad, x)
        yo = O.poly_apply(Mo, Ao.astype(dt), x)
        assert bits_equal(y, yo), (degree, dt)


def test_poly_build_on_device_close_to_oracle():
    Ao = O.stencil_csr("laplace2d", 20)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
    x = np.random.default_rng(5).standard_normal(Ao.n_rows)
    for deg, basis in ((5, P.PolyBasis.POWER), (15, P.PolyBasis.NEWTON_ROOTS)):
        M = P.build_poly_precond(A, deg, seed=0)
        Mo = O.poly_build(Ao, deg, seed=0)
        assert M.basis is basis and M.degree == Mo.degree == deg
        # same polynomial up to the (different) reduction order of the build's dots
        y, yo = P.apply_poly(M, A, x), O.poly_apply(Mo, Ao, x)
        assert np.linalg.norm(y - yo) <= 1e-7 * np.linalg.norm(yo)


@pytest.mark.parametrize("kind,nx,kw", [("laplace3d", 23, {}), ("laplace2d", 37, {}),
                                        ("convdiff2d", 41, {"convection": 1501.0}),
                                        ("recirc2d", 33, {"convection": 40.1}),
                                        ("stretched2d", 17, {}), ("laplace3d", 2, {})])
def test_stencil_storage_bitexact(kind, nx, kw, rng):
    """The stencil-specialised SpMV (packed values, no col_idx) equals the CSR
    kernel and the oracle bit for bit, in both precisions."""
    import ctypes as C
    from paper_2109_01232_b200.core import ctx, padded_length, stream_handle
    Ao = O.stencil_csr(kind, nx, **kw)
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)   # uploaded, not tagged
    dims, nxd = A.stencil_shape()
    assert (dims, nxd) == ((3 if kind == "laplace3d" else 2), nx)
    for dt in (np.float64, np.float32):
        Ad = A if dt == np.float64 else P.convert_matrix(A, P.FP32)
        dia = Ad.dia()
        x = rng.standard_normal(Ao.n_cols).astype(dt)
        xd = torch.from_numpy(x).cuda()
        y = torch.empty_like(xd)
        _lib.call("mpg_spmv_dia", Ad.precision.code, dims, nx, Ao.n_rows, dia.data_ptr(),
                  padded_length(Ao.n_rows), xd.data_ptr(), y.data_ptr(), ctx().ws.data_ptr(),
                  stream_handle())
        assert bits_equal(y.cpu().numpy(), O.spmv(Ao.astype(dt), x)), (kind, dt)


def test_stencil_detection_rejects_non_stencils():
    d = np.diag(np.full(64, 2.0)) + np.diag(np.full(63, -1.0), 1)
    assert P.CsrMatrix.from_dense(d).stencil_shape() is None
    Ao = O.stencil_csr("star2d", 8)
    assert P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values).stencil_shape() is None
    # same sizes as a 5-point stencil but one entry moved: the device check rejects it
    Ao = O.stencil_csr("laplace2d", 8)
    ci = Ao.col_idx.copy()
    ci[10] = ci[10] + 1 if ci[10] + 1 < ci[11] else ci[10]
    A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, np.where(np.arange(len(ci)) == 3, ci[3] + 1, ci),
                    Ao.values)
    assert A.stencil_shape() is None
