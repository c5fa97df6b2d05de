"""Where the end-to-end (host numpy in / out) GMRES-IR call spends its time at cfg2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_01232_b200 as P
from paper_2109_01232_b200.core import CsrMatrix, convert_matrix, FP32

A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 150))
rp, ci, v = A.host_arrays()
class H: pass
Ah = H(); Ah.n_rows = Ah.n_cols = A.n_rows; Ah.row_ptr, Ah.col_idx, Ah.values = rp, ci, v
bh = np.ones(A.n_rows)
crit = P.StopCriteria(rtol=1e-10, m=50)
P.gmres_ir(Ah, bh, criteria=crit)      # warm (graph capture etc.)
def t(label, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0):8.1f} ms", flush=True); return r
Ad = t("upload CSR (from_any)", lambda: CsrMatrix.from_any(Ah))
t("stencil detect + pack fp64", lambda: Ad.stencil_shape())
A32 = t("convert_matrix fp32", lambda: convert_matrix(Ad, FP32))
t("pack fp32", lambda: A32.dia())
t("gmres_ir device inputs", lambda: P.gmres_ir(Ad, torch.from_numpy(bh).cuda(), criteria=crit))
t("gmres_ir host inputs (e2e)", lambda: P.gmres_ir(Ah, bh, criteria=crit))
