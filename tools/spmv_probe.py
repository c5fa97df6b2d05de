"""A few CSR SpMV launches at laplace3d:nx (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import bench as B
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 150
A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, nx))
r = B.spmv_bench(A, reps=5, trials=1, warmup=2)
print(r)
