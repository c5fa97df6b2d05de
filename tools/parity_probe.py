"""Iteration counts of the order-sensitive parity cases under both step kernels
(debug aid): laplace3d:40 GMRES-IR (reference 250) and laplace3d:30 GMRES-FD
switching at 100 (reference 196), with each run's restart-boundary residuals."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2109_01232_b200 as P

CASES = [("laplace3d", 40, "ir", 0), ("laplace3d", 30, "fd", 100), ("laplace3d", 40, "fp64", 0),
         ("laplace2d", 100, "ir", 0), ("laplace2d", 100, "fd", 200)]
for kind, nx, solver, sw in CASES:
    A = P.generate(P.StencilSpec(P.StencilKind(kind), nx))
    b = np.ones(A.n_rows)
    crit = P.StopCriteria(rtol=1e-10, m=50)
    for mode in ("split", "persistent"):
        with P.solvers.step_kernel(mode):
            if solver == "ir":
                rep = P.gmres_ir(A, b, criteria=crit)
            elif solver == "fd":
                rep = P.gmres_fd(A, b, criteria=crit, switch_iter=sw)
            else:
                rep = P.gmres_restarted(A, b, criteria=crit)
        marks = [(e.iteration, f"{e.explicit:.3e}") for e in rep.residual_history if e.explicit is not None]
        print(f"{kind}:{nx}/{solver}{sw or ''} {mode}: {rep.total_iters} ({rep.iters_fp32}+{rep.iters_fp64}) "
              f"{marks[-4:]}", flush=True)
