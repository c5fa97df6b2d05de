"""One eager IR cycle of the single-GPU solver (for ncu -k regex:<kernel>).
    python tools/cycle_probe.py [nx=150] [steps=5] [solver=ir|fp64] [storage=auto|csr|stencil] [mega=auto|split|persistent]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import _lib
from paper_2109_01232_b200.core import FP32, FP64, convert_matrix, padded_copy, dvec
from paper_2109_01232_b200.solvers import NativeSolve
a = sys.argv[1:] + [None] * 5
nx = int(a[0] or 150)
steps = int(a[1] or 5)
solver = a[2] or "ir"
storage = a[3] or "auto"
mega = a[4] or "auto"
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, nx))
n = A.n_rows
b = torch.ones(n, dtype=torch.float64, device="cuda")
with P.solvers.step_kernel(mega):
    if solver == "ir":
        ns = NativeSolve(_lib.MODE_IR, FP32, convert_matrix(A, FP32), A, padded_copy(b, FP64), dvec(n, FP64), 50,
                         1e-10, use_graph=False, storage=storage)
    else:
        ns = NativeSolve(_lib.MODE_RESTARTED, FP64, A, None, padded_copy(b, FP64), dvec(n, FP64), 50, 1e-10,
                         use_graph=False, storage=storage)
ns.begin()
ns.cycle(steps)
torch.cuda.synchronize()
print("cycle probe done", ns.storage)
