"""sha256 of a solve's iterate and history (A/B bitwise-equality helper).

    MPG_LIB_PATH=tools/variants/x.so python tools/hash_solve.py [kind] [nx] [ir|fp64]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2109_01232_b200 as P

kind, nx, solver = (sys.argv[1:] + ["laplace3d", "60", "ir"][len(sys.argv) - 1:])[:3]
A = P.generate(P.StencilSpec(P.StencilKind(kind), int(nx)))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
crit = P.StopCriteria(rtol=1e-10, m=50)
rep = (P.gmres_ir if solver == "ir" else P.gmres_restarted)(A, b, criteria=crit)
x = rep.x.cpu().numpy() if torch.is_tensor(rep.x) else np.asarray(rep.x)
h = hashlib.sha256(x.tobytes()).hexdigest()[:16]
hist = hashlib.sha256(repr([(e.iteration, e.implicit, e.explicit) for e in rep.residual_history]).encode()).hexdigest()[:16]
print(kind, nx, solver, rep.total_iters, "x", h, "history", hist, os.environ.get("MPG_LIB_PATH", "default"))
