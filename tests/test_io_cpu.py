"""Matrix Market ingestion and reverse Cuthill-McKee: the
host cores against the reference's own outputs (tests/golden/reference_io.json,
made by tests/golden/make_golden.py --io from mpgmres.io / mpgmres.precond)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2109_01232_b200 import io as mio

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ref():
    with open(os.path.join(GOLD, "reference_io.json")) as f:
        return json.load(f)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canonical(n_rows, r, c, v):
    """coo_to_csr(sum_duplicates=True) on the host, as core.coo_to_csr does."""
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    new = np.concatenate([[True], (np.diff(r) != 0) | (np.diff(c) != 0)])
    s = np.flatnonzero(new)
    v = np.add.reduceat(v, s)
    r, c = r[s], c[s]
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n_rows))]).astype(np.int32)
    return rp, c.astype(np.int32), v


@pytest.mark.parametrize("name", ["general_dups.mtx", "symmetric.mtx", "integer_rect.mtx"])
def test_matrix_market_arrays_match_reference(name, ref):
    n_rows, n_cols, r, c, v = mio.read_matrix_market_arrays(os.path.join(GOLD, "mm", name))
    rp, ci, vals = canonical(n_rows, r, c, v)
    g = ref["mm"][name]
    assert (n_rows, n_cols, len(ci)) == (g["n_rows"], g["n_cols"], g["nnz"])
    assert sha(rp) == g["row_ptr"] and sha(ci) == g["col_idx"] and sha(vals) == g["values"]


def test_matrix_market_rejects_bad_files(tmp_path):
    p = tmp_path / "x.mtx"
    for text in ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
                 "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
                 "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
                 "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
                 "hello\n"):
        p.write_text(text)
        with pytest.raises(mio.MatrixMarketError):
            mio.read_matrix_market_arrays(str(p))


@pytest.mark.parametrize("name", ["laplace2d:12", "convdiff2d:9", "symmetric.mtx", "general_dups.mtx",
                                  "laplace2d:12:shuffled", "blocks12"])
def test_rcm_order_matches_reference(name, ref):
    g = ref["rcm"][name]
    perm = mio.rcm_order(g["n"], np.asarray(g["row_ptr"]), np.asarray(g["col_idx"]))
    assert perm.tolist() == g["perm"]
    P = mio.Permutation(perm)
    x = np.arange(g["n"], dtype=float) * 1.5
    assert np.array_equal(P.invert_apply(P.apply(x)), x)
