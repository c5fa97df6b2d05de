"""One eager GMRES cycle at a bench configuration, for ncu.

    python tools/profile_cycle.py [--nx 150] [--mode ir|fp64] [--m 50]

Generates the matrix on the device, runs the initial residual and one warm
cycle (graph), then one eager cycle whose kernels ncu can attribute one by
one.  Prints the per-class device times of the eager cycle.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import _lib
from paper_2109_01232_b200.core import FP32, FP64, convert_matrix, dvec, padded_copy
from paper_2109_01232_b200.solvers import NativeSolve


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=150)
    ap.add_argument("--mode", default="ir", choices=["ir", "fp64", "fp32"])
    ap.add_argument("--m", type=int, default=50)
    ap.add_argument("--kind", default="laplace3d")
    a = ap.parse_args()
    A = P.generate(P.StencilSpec(P.StencilKind(a.kind), a.nx))
    n = A.n_rows
    b = padded_copy(torch.ones(n, dtype=torch.float64, device="cuda"), FP64)
    if a.mode == "ir":
        ns = NativeSolve(_lib.MODE_IR, FP32, convert_matrix(A, FP32), A, b, dvec(n, FP64), a.m, 1e-10)
    elif a.mode == "fp64":
        ns = NativeSolve(_lib.MODE_RESTARTED, FP64, A, None, b, dvec(n, FP64), a.m, 1e-10)
    else:
        A32 = convert_matrix(A, FP32)
        ns = NativeSolve(_lib.MODE_RESTARTED, FP32, A32, None, padded_copy(torch.ones(n, device="cuda"), FP32),
                         dvec(n, FP32), a.m, 1e-10)
    ns.begin()
    ns.cycle(a.m)
    torch.cuda.synchronize()
    prof = ns.profile_cycle(a.m)
    ns.close()
    print(json.dumps({"nx": a.nx, "mode": a.mode, "n": n, "nnz": A.nnz, "profile_ms": prof}))


if __name__ == "__main__":
    main()
