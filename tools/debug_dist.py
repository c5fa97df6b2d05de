"""Phase-by-phase check of the distributed pipeline at world size 1 (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import dist as D

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 10
spec = P.StencilSpec(P.StencilKind.LAPLACE3D, nx)
part = D.RowPartition.for_stencil(3, nx, 1, 0)
s = D.DistributedStencilSolver(spec, part, "ir", 5, 1e-10, D.NullCollectives())
orig = s._ph


def traced(name, j=0, m_limit=1):
    t = time.time()
    orig(name, j, m_limit)
    torch.cuda.synchronize()
    hdr, imp = s.state.read()
    print(f"{name:12s} j={j} {1e3 * (time.time() - t):7.2f} ms  done={hdr.done} steps={hdr.steps} "
          f"flags={hdr.flags} gamma={hdr.gamma:.3e} rnorm={hdr.rnorm:.3e} w0={hdr.w0:.3e} "
          f"h_sub={hdr.h_sub:.3e} red0={float(s.red[0]):.3e}", flush=True)


s._ph = traced
print(s.begin())
hdr, imp = s.cycle(5)
print("cycle", hdr.steps, list(imp[:5]), hdr.rnorm)
A = P.generate(spec)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
from paper_2109_01232_b200.solvers import NativeSolve
from paper_2109_01232_b200.core import convert_matrix, padded_copy, dvec
ns = NativeSolve(1, P.FP32, convert_matrix(A, P.FP32), A, padded_copy(b, P.FP64), dvec(A.n_rows, P.FP64), 5, 1e-10)
print("fused begin", ns.begin())
h2, i2 = ns.cycle(5)
print("fused cycle", h2.steps, list(i2[:5]), h2.rnorm)
