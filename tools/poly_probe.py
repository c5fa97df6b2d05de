"""One short GMRES-IR + poly(25) solve at laplace3d:200 (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01232_b200 as P
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 200
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 25
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, nx))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
M = P.build_poly_precond(P.convert_matrix(A, P.FP32), deg, seed=0)
rep = P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=3), precond_fp32=M, use_graph=False)
print(rep.total_iters)
