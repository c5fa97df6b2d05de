"""Small solves through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck).  Sizes are tiny: the tools replay and
instrument every access.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2109_01232_b200 as P

crit = P.StopCriteria(rtol=1e-10, m=12, max_iters=24)
A3 = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 14))
A2 = P.generate(P.StencilSpec(P.StencilKind.CONVDIFF2D, 40, convection=20.0))
Ar = P.generate(P.StencilSpec(P.StencilKind.RECIRC2D, 30, convection=3.0))
for A in (A3, A2, Ar):
    b = np.ones(A.n_rows)
    for mode in ("persistent", "split"):
        with P.solvers.step_kernel(mode):
            P.gmres_ir(A, b, criteria=crit)
            P.gmres_restarted(A, b, criteria=crit)
    P.gmres_fd(A, b, criteria=crit, switch_iter=12)
    P.gmres_ir(A, b, criteria=crit, storage="csr")                    # CSR kernels
    P.gmres_restarted(A, b, criteria=crit, storage="csr")
A32 = P.convert_matrix(A3, P.FP32)
b = np.ones(A3.n_rows)
P.gmres_ir(A3, b, criteria=crit, precond_fp32=P.build_poly_precond(A32, 5, seed=0))   # polynomial
P.gmres_ir(A3, b, criteria=crit, precond_fp32=P.build_block_jacobi(A32, 1))           # Jacobi(1)
P.gmres_restarted(A3, b, criteria=crit, precond=P.build_block_jacobi(A3, 3))          # block Jacobi
x = np.random.default_rng(0).standard_normal(A3.n_rows)
P.spmv(A3, x)
P.norm2(torch.as_tensor(x, device="cuda"))
torch.cuda.synchronize()
print("sanitize probe done")
