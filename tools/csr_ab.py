"""CSR SpMV A/B under the reference's spmv_bench protocol (bench.py:82-119):
Laplace3D 150 / ConvDiff2D 1500 / Laplace3D 200, fp64 and fp32, algorithmic
TB/s = (nnz (s+4) + 4 (n+1) + 2 n s) / t.  MPG_LIB_PATH selects a variant."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import bench as B
cases = [("laplace3d:150", P.StencilSpec(P.StencilKind.LAPLACE3D, 150)),
         ("convdiff2d:1500", P.StencilSpec(P.StencilKind.CONVDIFF2D, 1500, convection=1501.0)),
         ("laplace3d:200", P.StencilSpec(P.StencilKind.LAPLACE3D, 200))]
tag = os.environ.get("MPG_LIB_PATH", "default")
for name, spec in cases:
    A = P.generate(spec)
    r = B.spmv_bench(A, reps=200, trials=3, warmup=20)
    out = {"lib": os.path.basename(tag), "case": name}
    for key, t, s in (("fp64", r.t_fp64, 8), ("fp32", r.t_fp32, 4)):
        by = A.nnz * (s + 4) + 4 * (A.n_rows + 1) + 2 * A.n_rows * s
        out[key + "_us"] = round(t / 200 * 1e6, 2)
        out[key + "_TBs"] = round(by / (t / 200) / 1e12, 3)
    print(json.dumps(out), flush=True)
