"""Matrix Market ingestion and reverse Cuthill-McKee ordering.

Host-side preprocessing that puts SuiteSparse-style inputs on the device path:

* ``load_matrix_market`` / ``write_matrix_market`` follow io.py:59-131:
  coordinate real/integer, general or symmetric; 1-based indices to 0-based;
  symmetric storage mirrored; duplicates summed (in file order, numpy
  ``add.reduceat``); canonical sorted CSR.  Pattern, complex and array files
  are rejected.  The result is a device ``CsrMatrix`` (fp64).
* ``rcm_reorder`` / ``permute_csr`` / ``Permutation`` follow precond.py:421-515:
  reverse Cuthill-McKee on the symmetrised pattern, one component at a time
  from a pseudo-peripheral vertex (repeated BFS sweeps; candidates from the
  last level ordered by degree, then index), children in ascending (degree,
  index); the concatenated order reversed; ``P A P^T`` in canonical form.

The numpy cores (``read_matrix_market_arrays``, ``rcm_order``) need no GPU and
are what the CPU tests pin against the reference's outputs.
"""

from __future__ import annotations

import csv
from collections import deque
from dataclasses import dataclass

import numpy as np

__all__ = ["MatrixMarketError", "load_matrix_market", "write_matrix_market", "read_matrix_market_arrays",
           "Permutation", "rcm_order", "rcm_reorder", "permute_csr", "write_convergence_csv",
           "read_convergence_csv", "write_summary_csv", "SUMMARY_FIELDS"]


class MatrixMarketError(ValueError):
    """Malformed or unsupported Matrix Market input (io.py:51)."""


def read_matrix_market_arrays(path) -> tuple[int, int, np.ndarray, np.ndarray, np.ndarray]:
    """(n_rows, n_cols, rows, cols, values) as 0-based int64 / fp64 triplets,
    symmetric storage mirrored, duplicates not yet summed."""
    with open(path, "r", encoding="utf-8") as fh:
        tok = fh.readline().lower().split()
        if len(tok) < 4 or tok[0] != "%%matrixmarket" or tok[1] != "matrix":
            raise MatrixMarketError(f"{path}: not a Matrix Market matrix file")
        layout, field = tok[2], tok[3]
        symmetry = tok[4] if len(tok) > 4 else "general"
        if layout != "coordinate" or field not in ("real", "integer"):
            raise MatrixMarketError(f"{path}: unsupported format '{layout} {field}' "
                                    "(only coordinate real/integer is supported)")
        if symmetry not in ("general", "symmetric"):
            raise MatrixMarketError(f"{path}: unsupported symmetry '{symmetry}' (only general or symmetric)")
        body = [(no, ln.split()) for no, ln in enumerate(fh, start=2)
                if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MatrixMarketError(f"{path}: missing size line")
    no, size = body[0]
    try:
        n_rows, n_cols, nnz = int(size[0]), int(size[1]), int(size[2])
    except (ValueError, IndexError):
        raise MatrixMarketError(f"{path}:{no}: malformed size line") from None
    entries = body[1:]
    if len(entries) != nnz:
        raise MatrixMarketError(f"{path}: header declares {nnz} entries, found {len(entries)}")
    r = np.empty(nnz, dtype=np.int64)
    c = np.empty(nnz, dtype=np.int64)
    v = np.empty(nnz, dtype=np.float64)
    for i, (no, parts) in enumerate(entries):
        try:
            r[i], c[i], v[i] = int(parts[0]), int(parts[1]), float(parts[2])
        except (ValueError, IndexError):
            raise MatrixMarketError(f"{path}:{no}: malformed entry") from None
        if not (1 <= r[i] <= n_rows and 1 <= c[i] <= n_cols):
            raise MatrixMarketError(f"{path}:{no}: index ({r[i]}, {c[i]}) out of range "
                                    f"for a {n_rows}x{n_cols} matrix")
    r -= 1
    c -= 1
    if symmetry == "symmetric":
        mirror = r != c
        r, c, v = np.concatenate([r, c[mirror]]), np.concatenate([c, r[mirror]]), np.concatenate([v, v[mirror]])
    return n_rows, n_cols, r, c, v


def load_matrix_market(path):
    """fp64 device CsrMatrix from a Matrix Market file (io.py:59-121)."""
    from .core import coo_to_csr, validate_csr
    n_rows, n_cols, r, c, v = read_matrix_market_arrays(path)
    A = coo_to_csr(n_rows, n_cols, r, c, v, sum_duplicates=True)
    validate_csr(A)
    return A


def write_matrix_market(A, path) -> None:
    """Coordinate real general, 1-based, fp64 round-trip safe (io.py:124-131)."""
    rp, ci, vals = (np.asarray(t.cpu()) if hasattr(t, "cpu") else np.asarray(t)
                    for t in (A.row_ptr, A.col_idx, A.values))
    rows = np.repeat(np.arange(A.n_rows), np.diff(rp))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{A.n_rows} {A.n_cols} {len(ci)}\n")
        fh.writelines(f"{r + 1} {c + 1} {float(x):.17g}\n" for r, c, x in zip(rows, ci, vals))


# ---------------------------------------------------------------------------
# reverse Cuthill-McKee (precond.py:421-515)

@dataclass(frozen=True)
class Permutation:
    """A bijection on [0, n); ``perm[new] = old`` (precond.py:114-141)."""

    perm: np.ndarray

    def __post_init__(self) -> None:
        p = np.asarray(self.perm, dtype=np.int64)
        object.__setattr__(self, "perm", p)
        if not np.array_equal(np.sort(p), np.arange(len(p))):
            raise ValueError("not a permutation of 0..n-1")

    def __len__(self) -> int:
        return len(self.perm)

    def inverse_array(self) -> np.ndarray:
        inv = np.empty_like(self.perm)
        inv[self.perm] = np.arange(len(self.perm))
        return inv

    def apply(self, x):
        """Reordered copy: result[new] = x[old]."""
        return x[self.perm] if hasattr(x, "cpu") else np.ascontiguousarray(np.asarray(x)[self.perm])

    def invert_apply(self, x):
        """Undo :meth:`apply`."""
        if hasattr(x, "cpu"):
            import torch
            out = torch.empty_like(x)
            out[torch.as_tensor(self.perm, device=x.device)] = x
            return out
        out = np.empty_like(np.asarray(x))
        out[self.perm] = x
        return out


def _undirected(n: int, row_ptr: np.ndarray, col_idx: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Adjacency (CSR, sorted, no self-loops, no duplicates) of the pattern of A + A^T."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    cols = np.asarray(col_idx, dtype=np.int64)
    a = np.concatenate([rows, cols])
    b = np.concatenate([cols, rows])
    off = a != b
    key = np.unique(a[off] * n + b[off])
    return np.searchsorted(key // n, np.arange(n + 1)), key % n


def _levels(ptr: np.ndarray, adj: np.ndarray, root: int) -> np.ndarray:
    """BFS level of every vertex from root (-1 if unreachable)."""
    lev = np.full(len(ptr) - 1, -1, dtype=np.int64)
    lev[root] = 0
    front = np.array([root], dtype=np.int64)
    d = 0
    while front.size:
        d += 1
        nb = np.concatenate([adj[ptr[u]:ptr[u + 1]] for u in front])
        nb = np.unique(nb[lev[nb] < 0])
        lev[nb] = d
        front = nb
    return lev


def _by_degree(vs: np.ndarray, deg: np.ndarray) -> np.ndarray:
    """vs ordered by (degree, index)."""
    return vs[np.lexsort((vs, deg[vs]))]


def _start_vertex(ptr, adj, deg, seed: int) -> int:
    """Pseudo-peripheral vertex of seed's component: BFS from the current
    vertex, take the lowest-(degree, index) vertex of the deepest level, and
    repeat while that deepens the level structure; the last candidate wins."""
    lev = _levels(ptr, adj, seed)
    depth = int(lev.max())
    while True:
        cand = int(_by_degree(np.flatnonzero(lev == depth), deg)[0])
        clev = _levels(ptr, adj, cand)
        cdepth = int(clev.max())
        if cdepth <= depth:
            return cand
        lev, depth = clev, cdepth


def rcm_order(n: int, row_ptr, col_idx) -> np.ndarray:
    """perm[new] = old of the reverse Cuthill-McKee ordering (host, numpy)."""
    ptr, adj = _undirected(n, np.asarray(row_ptr), np.asarray(col_idx))
    deg = np.diff(ptr)
    seen = np.zeros(n, dtype=bool)
    order: list[int] = []
    for seed in range(n):
        if seen[seed]:
            continue
        root = _start_vertex(ptr, adj, deg, seed)
        seen[root] = True
        q = deque([root])
        while q:
            u = q.popleft()
            order.append(u)
            nb = adj[ptr[u]:ptr[u + 1]]
            nb = _by_degree(nb[~seen[nb]], deg)
            seen[nb] = True
            q.extend(int(x) for x in nb)
    return np.asarray(order[::-1], dtype=np.int64)


def permute_csr(A, perm: Permutation):
    """P A P^T with result[i, j] = A[perm[i], perm[j]] (precond.py:445-450), device CsrMatrix."""
    from .core import coo_to_csr
    rp, ci, vals = (np.asarray(t.cpu()) for t in (A.row_ptr, A.col_idx, A.values))
    inv = perm.inverse_array()
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(rp))
    return coo_to_csr(A.n_rows, A.n_cols, inv[rows], inv[ci.astype(np.int64)], vals.copy())


def rcm_reorder(A):
    """(Permutation, P A P^T) for a square device CsrMatrix (precond.py:421-442)."""
    from .core import CsrMatrix, ShapeError
    A = CsrMatrix.from_any(A)
    if A.n_rows != A.n_cols:
        raise ShapeError("reordering needs a square matrix")
    perm = Permutation(rcm_order(A.n_rows, A.row_ptr.cpu().numpy(), A.col_idx.cpu().numpy()))
    return perm, permute_csr(A, perm)


# ---------------------------------------------------------------------------
# result CSVs (io.py:165-201): the same artefacts the reference writes

def write_convergence_csv(report, path) -> None:
    """Per-iteration residual history; explicit entries blank off the restart boundaries."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["iteration", "implicit_relres", "explicit_relres", "phase"])
        w.writerows([e.iteration, repr(e.implicit), "" if e.explicit is None else repr(e.explicit), e.phase]
                    for e in report.residual_history)


def read_convergence_csv(path) -> list:
    from .solvers import HistoryEntry
    with open(path, "r", encoding="utf-8", newline="") as fh:
        rows = list(csv.reader(fh))[1:]
    return [HistoryEntry(int(r[0]), float(r[1]), None if r[2] == "" else float(r[2]), r[3]) for r in rows]


SUMMARY_FIELDS = ["name", "n", "nnz", "solver", "precond", "time_s", "iters", "converged", "loss_of_accuracy"]


def write_summary_csv(rows: list[dict], path) -> None:
    """Solver-comparison summary, one solve per row."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=SUMMARY_FIELDS)
        w.writeheader()
        w.writerows({k: row.get(k, "") for k in SUMMARY_FIELDS} for row in rows)
