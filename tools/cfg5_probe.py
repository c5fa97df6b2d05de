"""First GMRES-IR cycle at laplace3d:400 vs the reference's recorded iterate (debug aid)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_01232_b200 as P
g = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/reference_cfg5.json")))
ref = g["runs"]["laplace3d:400/ir/m50/max50"]
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, int(sys.argv[1]) if len(sys.argv) > 1 else 400))
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
for mode in ("split", "auto"):
    with P.solvers.step_kernel(mode):
        rep = P.gmres_ir(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=50))
    x = rep.x.cpu().numpy()[:: ref["x_stride"]]
    s = np.asarray(ref["x_sample"])
    d = x - s
    print(mode, "res", [e.explicit for e in rep.residual_history if e.explicit is not None], ref["boundaries"][-1][2])
    print(" rel", np.linalg.norm(d) / np.linalg.norm(s), "max idx", int(np.argmax(abs(d))), "x", x[:4], "ref", s[:4])
    print(" d[::512]", d[::512])
rep64 = P.gmres_restarted(A, b, criteria=P.StopCriteria(rtol=1e-10, m=50, max_iters=50))
x64 = rep64.x.cpu().numpy()[:: ref["x_stride"]]
xs = rep.x.cpu().numpy()[:: ref["x_stride"]]
s = np.asarray(ref["x_sample"])
print("fp64 GMRES(50) first cycle as the exact-arithmetic Krylov iterate:")
print(" ours(fp32 IR) vs fp64:", np.linalg.norm(xs - x64) / np.linalg.norm(x64))
print(" reference(fp32 IR) vs fp64:", np.linalg.norm(s - x64) / np.linalg.norm(x64))
