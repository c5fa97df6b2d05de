"""Phase timeline of the persistent step kernel (build: tools/build_variant.sh
mt -DMPG_MEGA_TIMING=26; run with MPG_LIB_PATH=tools/variants/mt.so)."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import _lib
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, int(sys.argv[1]) if len(sys.argv) > 1 else 150))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
solver = sys.argv[2] if len(sys.argv) > 2 else "ir"
crit = P.StopCriteria(rtol=1e-10, m=50, max_iters=50)
if solver == "ir":
    P.gmres_ir(A, b, criteria=crit, use_graph=False)
else:   # fp64 GMRES: force the persistent step (MPG_MEGA=1 or step_kernel("persistent"))
    with P.solvers.step_kernel("persistent"):
        P.gmres_restarted(A, b, criteria=crit, use_graph=False)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (296 * 10))()
_lib.load().mpg_debug_mega_times(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(296, 10)[:148].astype(np.int64)
t0 = t[:, 0].min()
names = ["start", "P1 SpMV done", "P1b dots done", "B1 released", "P2 done", "B2 released", "P3 done",
         "B3 released", "P4 done"]
for i, nm in enumerate(names):
    col = t[:, i] - t0
    print(f"{nm:16s} min {col.min() / 1e3:8.1f} us  median {np.median(col) / 1e3:8.1f}  max {col.max() / 1e3:8.1f}")
if os.environ.get("MPG_PHASE_CTAS"):
    # which CTAs finish each phase last (skew attribution): rank by phase end relative to its start
    nblk = -(-A.n_rows // 128)
    nb = np.array([(nblk - 1 - c) // 148 + 1 for c in range(148)])
    for i, nm in [(2, "P1b"), (4, "P2"), (6, "P3")]:
        dur = t[:, i] - t[:, i - 1]
        order = np.argsort(-dur)[:12]
        print(f"{nm} slowest CTAs (dur us, nb):", [(int(c), round(dur[c] / 1e3, 1), int(nb[c])) for c in order])
        print(f"{nm} dur: min {dur.min()/1e3:.1f} med {np.median(dur)/1e3:.1f} max {dur.max()/1e3:.1f}; "
              f"end spread {(t[:, i].max() - np.median(t[:, i]))/1e3:.1f} us")
    np.save(os.path.join("gpurun_out", "mega_times.npy"), t)
