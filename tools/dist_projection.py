"""Per-rank work of the row-partitioned cfg2 / cfg5 solve, measured on ONE GPU:
rank 0's plane block of an N-way partition, solved as a stand-alone subdomain
(no neighbours: the cut planes read the zero guard rows) with the distributed
solver at world size 1 -- the same kernels (persistent step or phase path,
"auto" rule) on n/N rows.  This is the compute part of an N-GPU step; the
N-GPU run adds the in-kernel exchanges (three peer-memory sums and one halo
plane per step) on top.  A projection input, not a multi-GPU measurement.

    python tools/dist_projection.py [nx=150] [cycles=2]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2109_01232_b200 as P
from paper_2109_01232_b200.dist import (Collectives, DistributedStencilSolver, RowPartition, _dist_solve,
                                        plane_partition)

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 150
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = P.StencilSpec(P.StencilKind.LAPLACE3D, nx)
plane = nx * nx
for N in [int(a) for a in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "2", "4", "8"])]:
    p0, p1 = plane_partition(nx, N)[0]
    part = RowPartition(3, nx, 1, 0, p0 * plane, p1 * plane, plane)
    crit = P.StopCriteria(rtol=1e-10, m=50, max_iters=50 * cycles)
    s = DistributedStencilSolver(spec, part, "ir", 50, 1e-10, Collectives(), persistent="auto")
    s.x_buf.zero_()
    _dist_solve(s, crit, True, None)
    s.x_buf.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = _dist_solve(s, crit, True, None)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(json.dumps({"nx": nx, "N": N, "n_local": part.n_local, "persistent": s.persistent,
                      "iters": rep.total_iters, "s": round(t, 5), "us_per_iter": round(t / rep.total_iters * 1e6, 2)}),
          flush=True)
    s.close()
dist.destroy_process_group()
