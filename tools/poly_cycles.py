"""Cycle structure and timing of GMRES-IR + poly(d) at laplace3d:nx."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01232_b200 as P
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 200
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 25
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, nx))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
M = P.build_poly_precond(P.convert_matrix(A, P.FP32), deg, seed=0)
crit = P.StopCriteria(rtol=1e-10, m=50)
for ug in (True, False):
    P.gmres_ir(A, b, criteria=crit, precond_fp32=M, use_graph=ug)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rep = P.gmres_ir(A, b, criteria=crit, precond_fp32=M, use_graph=ug); e1.record(); e1.synchronize()
    bounds = [e.iteration for e in rep.residual_history if e.explicit is not None]
    print(json.dumps({"graph": ug, "iters": rep.total_iters, "s": e0.elapsed_time(e1) / 1e3,
                      "cycles": len(bounds) - 1, "cycle_lengths": [b1 - b0 for b0, b1 in zip(bounds, bounds[1:])]}))
