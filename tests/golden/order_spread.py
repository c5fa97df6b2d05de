"""Reduction-order sensitivity of GMRES-FD and GMRES-IR iteration counts (test evidence).

GMRES-FD switches from fp32 to fp64 at `switch_iter`.  When the switch
comes after the fp32 leg has reached its attainable accuracy (explicit
residual ~1e-5 here), the fp64 leg starts from an iterate whose error is the
fp32 leg's accumulated rounding, and its length depends on the ORDER of the
fp32 dot-product / norm / update summations, not on the algorithm.  This
script re-runs the CPU oracle (bit-identical to the reference, see
test_oracle.py) with the fp32 reductions re-associated in ways any valid
implementation might use (reversed, blocked, pairwise, column-sequential, ...)
and records the spread of total iteration counts.  tests/test_gpu_solvers.py
records that spread next to the count of the device-order oracle
(oracle/devorder.c: the association the GPU kernels use), so an order-sensitive
case's reference count, its spread and the GPU's own order sit side by side.
GMRES-IR on Laplace3D(40) is the case SURVEY.md A.5 flags: the reference
needs 250 iterations, blocked / pairwise reductions 200.  The tests do NOT
widen any parity band with this spread: order-sensitive cases are asserted
bit for bit against the device-order oracle (tests/test_gpu_parity_order.py).

    python tests/golden/order_spread.py      # writes order_spread.json
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import cpu_gmres as O  # noqa: E402
from oracle import devorder as D  # noqa: E402

CASES = [("laplace3d", 30, "fd", 100), ("laplace2d", 100, "fd", 200), ("laplace3d", 40, "ir", 0)]


def _blocked(B, rev=False):
    def dots(V, w):
        n = w.shape[0]
        starts = list(range(0, n, B))
        if rev:
            starts = starts[::-1]
        out = np.zeros(V.shape[1], dtype=w.dtype)
        for s in starts:
            out = (out + (V[s:s + B].T @ w[s:s + B]).astype(w.dtype)).astype(w.dtype)
        return out
    return dots


def _blocked_nrm(B):
    def nrm(x):
        acc = x.dtype.type(0)
        for s in range(0, x.shape[0], B):
            acc = x.dtype.type(acc + np.dot(x[s:s + B], x[s:s + B]))
        return float(np.sqrt(acc))
    return nrm


def pw_dots(V, w):
    return (V * w[:, None]).sum(axis=0, dtype=w.dtype)


def pw_nrm(x):
    return float(np.sqrt((x * x).sum(dtype=x.dtype)))


def rev_dots(V, w):
    return np.array([np.dot(V[::-1, i], w[::-1]) for i in range(V.shape[1])], dtype=w.dtype)


def strided_dots(S):
    """S interleaved partial sums (a grid-stride kernel), then a sequential total."""
    def dots(V, w):
        n = w.shape[0]
        out = np.zeros(V.shape[1], dtype=w.dtype)
        for p in range(S):
            out = (out + (V[p:n:S].T @ w[p:n:S]).astype(w.dtype)).astype(w.dtype)
        return out
    return dots


def sep_update(V, c, w):
    for i in range(V.shape[1]):
        w -= V[:, i] * c[i]
    return w


def variants():
    v = {"reference": {}}
    v["pairwise_dots"] = dict(d=pw_dots)
    v["pairwise_dots_norm"] = dict(d=pw_dots, n=pw_nrm)
    v["reversed_dots"] = dict(d=rev_dots)
    v["reversed_dots_pairwise_norm"] = dict(d=rev_dots, n=pw_nrm)
    v["column_update"] = dict(u=sep_update)
    v["pairwise_column_update"] = dict(d=pw_dots, n=pw_nrm, u=sep_update)
    for B in (128, 512, 1024, 4096):
        v[f"blocked{B}"] = dict(d=_blocked(B), n=_blocked_nrm(B))
        v[f"blocked{B}_rev"] = dict(d=_blocked(B, rev=True))
    for S in (32, 256, 1024):
        v[f"strided{S}"] = dict(d=strided_dots(S))
    return v


def main():
    orig = (O.basis_dots, O.basis_update, O.nrm2)
    out = {}
    try:
        for kind, nx, solver, sw in CASES:
            A = O.stencil_csr(kind, nx)
            b = O.ones_rhs(A.n_rows)
            counts = {}
            for name, v in variants().items():
                O.basis_dots = v.get("d", orig[0])
                O.basis_update = v.get("u", orig[1])
                O.nrm2 = v.get("n", orig[2])
                run = (lambda: O.solve_fd(A, b, m=50, switch_iter=sw)) if solver == "fd" else \
                    (lambda: O.solve_ir(A, b, m=50))
                counts[name] = int(run().total_iters)
                print(kind, nx, solver, sw, name, counts[name], flush=True)
            O.basis_dots, O.basis_update, O.nrm2 = orig
            dev = D.solve_fd(A, b, m=50, switch_iter=sw) if solver == "fd" else D.solve_ir(A, b, m=50)
            vals = list(counts.values())
            key = f"{kind}:{nx}/fd{sw}/m50" if solver == "fd" else f"{kind}:{nx}/ir/m50"
            out[key] = {"counts": counts, "min": min(vals), "max": max(vals),
                        "device_order": int(dev.total_iters)}
    finally:
        O.basis_dots, O.basis_update, O.nrm2 = orig
    with open(os.path.join(HERE, "order_spread.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
