"""A few CSR SpMV launches (for ncu): spmv_bench with 2 warm-up pairs, then 5
fp64 and 5 fp32 products.  ncu -s 4 -c 1 picks an fp64 launch, -s 9 -c 1 fp32.
    python tools/spmv_probe.py [laplace3d:150 | convdiff2d:1500:1501 | laplace3d:200]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import bench as B
arg = sys.argv[1] if len(sys.argv) > 1 else "laplace3d:150"
parts = arg.split(":")
if parts[0].isdigit():            # old form: nx of laplace3d
    parts = ["laplace3d", parts[0]]
kind, nx = parts[0], int(parts[1])
kw = {"convection": float(parts[2])} if len(parts) > 2 else {}
A = P.generate(P.StencilSpec(P.StencilKind(kind), nx, **kw))
r = B.spmv_bench(A, reps=5, trials=1, warmup=2)
print(r)
