"""Print the restart-boundary record of a GPU solve next to the oracle's (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2109_01232_b200 as P
from oracle import cpu_gmres as O

kind, nx, sw = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ("laplace3d", 30, 100)
Ao = O.stencil_csr(kind, nx)
b = O.ones_rhs(Ao.n_rows)
A = P.CsrMatrix(Ao.n_rows, Ao.n_cols, Ao.row_ptr, Ao.col_idx, Ao.values)
crit = P.StopCriteria(rtol=1e-10, m=50)
for st in ("csr", "stencil"):
    rep = P.gmres_fd(A, b, criteria=crit, switch_iter=sw) if st == "csr" else None
    if rep is None:
        continue
    print(st, rep.total_iters, rep.iters_fp32, rep.iters_fp64,
          [(e.iteration, f"{e.explicit:.3e}", e.phase) for e in rep.residual_history if e.explicit is not None])
r32 = P.gmres_restarted(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=sw), precision=P.FP32)
print("fp32 leg", [(e.iteration, f"{e.implicit:.3e}", f"{e.explicit:.3e}") for e in r32.residual_history if e.explicit is not None])
o = O.solve_fd(Ao, b, m=50, switch_iter=sw)
print("oracle", o.total_iters, [(h[0], f"{h[2]:.3e}", h[3]) for h in o.history if h[2] is not None])
