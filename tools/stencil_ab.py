"""Stencil-SpMV A/B (MPG_LIB_PATH selects a build): per-class device time of
one eager four-launch IR cycle at laplace3d:400 and :150, and the cfg4
GMRES-IR + poly(25) solve time at laplace3d:200 (25 stencil SpMVs per step)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import _lib
from paper_2109_01232_b200.core import FP32, FP64, convert_matrix, padded_copy, dvec
from paper_2109_01232_b200.solvers import NativeSolve
tag = os.path.basename(os.environ.get("MPG_LIB_PATH", "default"))
for nx in (400, 150):
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, nx))
    n = A.n_rows
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    with P.solvers.step_kernel("split"):
        ns = NativeSolve(_lib.MODE_IR, FP32, convert_matrix(A, FP32), A, padded_copy(b, FP64), dvec(n, FP64), 50, 1e-10)
    ns.begin(); ns.cycle(50)
    prof = ns.profile_cycle(50)
    ns.close()
    sp = prof["spmv_dot1"]
    res = prof["residual"]
    print(json.dumps({"lib": tag, "nx": nx, "spmv_us": round(sp[0] / sp[1] * 1e3, 2),
                      "spmv_TBs": round(2 * n * 4 / (sp[0] / sp[1] * 1e-3) / 1e12, 3),
                      "resid64_us": round(res[0] * 1e3, 1), "resid64_TBs": round(3 * n * 8 / (res[0] * 1e-3) / 1e12, 3)}))
    with P.solvers.step_kernel("split"):
        ns = NativeSolve(_lib.MODE_RESTARTED, FP64, A, None, padded_copy(b, FP64), dvec(n, FP64), 50, 1e-10)
    ns.begin(); ns.cycle(50)
    prof = ns.profile_cycle(50)
    ns.close()
    sp = prof["spmv_dot1"]
    print(json.dumps({"lib": tag, "nx": nx, "fp64_spmv_us": round(sp[0] / sp[1] * 1e3, 2),
                      "fp64_spmv_TBs": round(2 * n * 8 / (sp[0] / sp[1] * 1e-3) / 1e12, 3),
                      "fp64_resid_us": round(prof["residual"][0] * 1e3, 1)}))
    del A, b
    torch.cuda.empty_cache()
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, 200))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
M = P.build_poly_precond(P.convert_matrix(A, P.FP32), 25, seed=0)
crit = P.StopCriteria(rtol=1e-10, m=50)
P.gmres_ir(A, b, criteria=crit, precond_fp32=M)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); rep = P.gmres_ir(A, b, criteria=crit, precond_fp32=M); e1.record(); e1.synchronize()
print(json.dumps({"lib": tag, "cfg4_poly25_s": round(e0.elapsed_time(e1) / 1e3, 4), "iters": rep.total_iters,
                  "kernel_times": {k: round(v, 4) for k, v in rep.kernel_times.items()}}))
