"""Time full solves at a bench configuration (A/B helper; not the bench).

    python tools/solve_time.py [--kind laplace3d] [--nx 150] [--solver ir|fp64] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2109_01232_b200 as P


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="laplace3d")
    ap.add_argument("--nx", type=int, default=150)
    ap.add_argument("--solver", default="ir")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-iters", type=int, default=100_000)
    a = ap.parse_args()
    A = P.generate(P.StencilSpec(P.StencilKind(a.kind), a.nx))
    b = torch.ones(A.n_rows, dtype=torch.float64, device="cuda")
    crit = P.StopCriteria(rtol=1e-10, m=50, max_iters=a.max_iters)
    f = (lambda: P.gmres_ir(A, b, criteria=crit)) if a.solver == "ir" else \
        (lambda: P.gmres_restarted(A, b, criteria=crit))
    f()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    print(json.dumps({"kind": a.kind, "nx": a.nx, "solver": a.solver, "iters": rep.total_iters,
                      "s": [round(t, 4) for t in ts], "env": {k: v for k, v in os.environ.items() if k.startswith("MPG_")}}))


if __name__ == "__main__":
    main()
