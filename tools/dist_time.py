"""Time the row-partitioned path at world size 1 over NCCL -- the phase path
(graph vs eager) and the distributed persistent step (graph) -- against the
fused single-GPU solve at cfg2 (overhead of the distributed machinery)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2109_01232_b200 as P
from paper_2109_01232_b200.dist import Collectives, DistributedStencilSolver, RowPartition, _dist_solve

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 150
spec = P.StencilSpec(P.StencilKind.LAPLACE3D, nx)
crit = P.StopCriteria(rtol=1e-10, m=50)
part = RowPartition.for_stencil(3, nx, 1, 0)
out = {}
for ug, pers in ((True, False), (False, False), (True, True)):
    s = DistributedStencilSolver(spec, part, "ir", 50, 1e-10, Collectives(), use_graph=ug, persistent=pers)
    def solve():
        s.x_buf.zero_()
        return _dist_solve(s, crit, True, None)
    solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rep = solve(); e1.record(); e1.synchronize()
    key = "dist_persistent_graph" if pers else ("dist_graph" if ug else "dist_eager")
    out[key] = (round(e0.elapsed_time(e1) / 1e3, 4), rep.total_iters)
    s.close()
A = P.generate(spec)
b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
P.gmres_ir(A, b, criteria=crit)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); rep = P.gmres_ir(A, b, criteria=crit); e1.record(); e1.synchronize()
out["fused"] = (round(e0.elapsed_time(e1) / 1e3, 4), rep.total_iters)
print(json.dumps(out))
dist.destroy_process_group()
