"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container, where the read-only reference exists:

    python tests/golden/make_golden.py            # small + assembly hashes
    python tests/golden/make_golden.py --cfg2     # + full Laplace3D(150) runs (~35 min)
    python tests/golden/make_golden.py --skip-small --cfg3   # ConvDiff2D(1500) runs (~28 min)
    python tests/golden/make_golden.py --skip-small --cfg4 25  # Laplace3D(200) IR+poly(25) (~1 h)
    python tests/golden/make_golden.py --skip-small --cfg5     # Laplace3D(400): assembly + 1 IR cycle

Nothing on the GPU box reads /root/reference: the tests only read the
committed JSON/NPZ written here.  The reference is imported read-only from
``/root/reference/pkg/src`` (mpgmres 0.1.0, numpy 2.3.5, scipy 1.18.1,
OpenBLAS 0.3.30 SkylakeX, BLAS pinned to one thread by the reference).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import mpgmres
    return mpgmres


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def report_dict(rep) -> dict:
    return {
        "converged": bool(rep.converged),
        "total_iters": int(rep.total_iters),
        "iters_fp32": int(rep.iters_fp32),
        "iters_fp64": int(rep.iters_fp64),
        "loss_of_accuracy": bool(rep.loss_of_accuracy),
        "stalled_at": rep.stalled_at,
        # explicit residuals at restart boundaries (the per-cycle record)
        "boundaries": [[int(e.iteration), float(e.implicit), float(e.explicit), e.phase]
                       for e in rep.residual_history if e.explicit is not None],
        "history_len": len(rep.residual_history),
        "x_sha256": sha(rep.x),
        "x_norm": float(np.linalg.norm(rep.x)),
        "x_head": [float(v) for v in rep.x[:4]],
        # strided sample of the solution (full x is too large to commit at cfg2)
        "x_stride": max(1, len(rep.x) // 4096),
        "x_sample": [float(v) for v in rep.x[:: max(1, len(rep.x) // 4096)]],
        "total_time_s": float(rep.total_time),
    }


SMALL_RUNS = [
    # (name, spec, solver, kwargs)
    ("laplace2d:50/fp64/m50", ("laplace2d", 50, {}), "fp64", {"m": 50}),
    ("laplace2d:50/ir/m50", ("laplace2d", 50, {}), "ir", {"m": 50}),
    ("laplace2d:100/fp64/m50", ("laplace2d", 100, {}), "fp64", {"m": 50}),
    ("laplace2d:100/ir/m50", ("laplace2d", 100, {}), "ir", {"m": 50}),
    ("laplace2d:100/fd200/m50", ("laplace2d", 100, {}), "fd", {"m": 50, "switch_iter": 200}),
    ("laplace2d:100/fp64/m25", ("laplace2d", 100, {}), "fp64", {"m": 25}),
    ("laplace2d:100/ir/m25", ("laplace2d", 100, {}), "ir", {"m": 25}),
    ("laplace2d:100/fp64/m100", ("laplace2d", 100, {}), "fp64", {"m": 100}),
    ("laplace2d:100/ir/m100", ("laplace2d", 100, {}), "ir", {"m": 100}),
    ("laplace2d:100/fp32/m50/max5000", ("laplace2d", 100, {}), "fp32", {"m": 50, "max_iters": 5000}),
    ("laplace3d:40/fp64/m50", ("laplace3d", 40, {}), "fp64", {"m": 50}),
    ("laplace3d:40/ir/m50", ("laplace3d", 40, {}), "ir", {"m": 50}),
    ("laplace3d:30/fd100/m50", ("laplace3d", 30, {}), "fd", {"m": 50, "switch_iter": 100}),
    ("convdiff2d:100:c100/fp64/m50", ("convdiff2d", 100, {"convection": 100.0}), "fp64", {"m": 50}),
    ("convdiff2d:100:c100/ir/m50", ("convdiff2d", 100, {"convection": 100.0}), "ir", {"m": 50}),
    ("convdiff2d:60:c61/ir+jacobi1/m50", ("convdiff2d", 60, {"convection": 61.0}), "ir+jacobi1", {"m": 50}),
    ("recirc2d:40:c0.5/ir/m50", ("recirc2d", 40, {"convection": 0.5}), "ir", {"m": 50}),
    ("laplace3d:20/ir+poly5/m50", ("laplace3d", 20, {}), "ir+poly5", {"m": 50}),
    ("laplace3d:20/ir+poly25/m50", ("laplace3d", 20, {}), "ir+poly25", {"m": 50}),
    ("laplace3d:20/fp64+poly25_32/m50", ("laplace3d", 20, {}), "fp64+poly25_32", {"m": 50}),
    ("laplace2d:20/fp64/m10/max15", ("laplace2d", 20, {}), "fp64", {"m": 10, "max_iters": 15}),
]

CFG2_RUNS = [
    ("laplace3d:150/fp64/m50", ("laplace3d", 150, {}), "fp64", {"m": 50}),
    ("laplace3d:150/ir/m50", ("laplace3d", 150, {}), "ir", {"m": 50}),
]

CFG3_RUNS = [  # BASELINE configs[2]: UniFlow2D 1500^2 (convection=1501, dx_term 0.5)
    ("convdiff2d:1500:c1501/fp64/m50", ("convdiff2d", 1500, {"convection": 1501.0}), "fp64", {"m": 50}),
    ("convdiff2d:1500:c1501/ir+jacobi1/m50", ("convdiff2d", 1500, {"convection": 1501.0}), "ir+jacobi1",
     {"m": 50}),
]


CFG4_RUNS = {  # BASELINE configs[3]: GMRES-IR + GMRES-polynomial(d) on Laplace3D 200^3
    d: (f"laplace3d:200/ir+poly{d}/m50", ("laplace3d", 200, {}), f"ir+poly{d}", {"m": 50}) for d in (25, 40)
}


def run_one(mp, spec, solver, kw):
    kind, nx, sk = spec
    A = mp.generate(mp.StencilSpec(mp.StencilKind(kind), nx, **sk))
    b = np.ones(A.n_rows)
    crit = mp.StopCriteria(rtol=kw.get("rtol", 1e-10), m=kw["m"],
                           max_iters=kw.get("max_iters", 100_000))
    if solver == "fp64":
        return mp.gmres_restarted(A, b, criteria=crit)
    if solver == "fp32":
        return mp.gmres_restarted(A, b, criteria=crit, precision=mp.FP32)
    if solver == "ir":
        return mp.gmres_ir(A, b, criteria=crit)
    if solver == "fd":
        return mp.gmres_fd(A, b, criteria=crit, switch_iter=kw["switch_iter"])
    A32 = mp.convert_matrix(A, mp.FP32)
    if solver == "ir+jacobi1":
        return mp.gmres_ir(A, b, criteria=crit, precond_fp32=mp.build_block_jacobi(A32, 1))
    if solver.startswith("ir+poly"):
        M = mp.build_poly_precond(A32, int(solver[7:]), seed=0)
        return mp.gmres_ir(A, b, criteria=crit, precond_fp32=M)
    if solver == "fp64+poly25_32":
        M = mp.build_poly_precond(A32, 25, seed=0)
        return mp.gmres_restarted(A, b, criteria=crit, precond=M)
    raise ValueError(solver)


ASSEMBLY = [  # (kind, nx, kwargs): sha256 of row_ptr / col_idx / values
    ("laplace2d", 100, {}),
    ("laplace3d", 150, {}),
    ("convdiff2d", 1500, {"convection": 1501.0}),
    ("recirc2d", 1500, {"convection": 1.0}),
    ("laplace3d", 200, {}),
    ("recirc2d", 77, {"convection": 40.1}),
    ("stretched2d", 60, {}),
    ("biharmonic2d", 33, {}),
    ("star2d", 31, {}),
]


def spmv_fixtures(mp):
    """Small SpMV cases: matrices, x, and the reference's y, both precisions."""
    rng = np.random.default_rng(20260101)
    out = {}
    cases = [("laplace3d", 7, {}), ("laplace2d", 17, {}), ("convdiff2d", 15, {"convection": 1501.0}),
             ("recirc2d", 19, {"convection": 40.1}), ("biharmonic2d", 14, {}), ("star2d", 16, {})]
    mats = [(f"{k}:{nx}", mp.generate(mp.StencilSpec(mp.StencilKind(k), nx, **kw)))
            for k, nx, kw in cases]
    # long rows (numpy pairwise sum with 8-way unrolling and recursive split)
    for n, dens in ((64, 0.5), (300, 0.6)):
        d = rng.standard_normal((n, n)) * (rng.random((n, n)) < dens)
        d[5, :] = 0.0  # an empty row
        mats.append((f"dense{n}", mp.CsrMatrix.from_dense(d)))
    for name, A in mats:
        for prec in ("fp64", "fp32"):
            Ap = A if prec == "fp64" else mp.convert_matrix(A, mp.FP32)
            x = rng.standard_normal(A.n_cols).astype(Ap.values.dtype)
            y = mp.spmv(Ap, x)
            key = f"{name}/{prec}"
            out[key + "/row_ptr"] = Ap.row_ptr
            out[key + "/col_idx"] = Ap.col_idx
            out[key + "/values"] = Ap.values
            out[key + "/x"] = x
            out[key + "/y"] = y
    return out


def io_fixtures(mp, meta):
    """Matrix Market files (written here as text) loaded by the reference, and
    its reverse Cuthill-McKee permutations (io.py:59-121, precond.py:421-515)."""
    from mpgmres import io as mio
    from mpgmres import precond as mpc
    rng = np.random.default_rng(7)
    d = os.path.join(HERE, "mm")
    os.makedirs(d, exist_ok=True)
    files = {}
    # general real with duplicates (summed) and comments
    n = 40
    r = rng.integers(1, n + 1, 300); c = rng.integers(1, n + 1, 300); v = rng.standard_normal(300)
    lines = ["%%MatrixMarket matrix coordinate real general", "% a comment", f"{n} {n} 300"]
    lines += [f"{a} {b} {x:.17g}" for a, b, x in zip(r, c, v)]
    files["general_dups.mtx"] = "\n".join(lines) + "\n"
    # symmetric (lower triangle stored, diagonal once)
    ent = {(i, i): 4.0 + i for i in range(1, 31)}
    for _ in range(80):
        a, b = sorted(rng.integers(1, 31, 2))
        if a != b:
            ent[(b, a)] = float(rng.standard_normal())
    lines = ["%%MatrixMarket matrix coordinate real symmetric", f"30 30 {len(ent)}"]
    lines += [f"{a} {b} {x:.17g}" for (a, b), x in ent.items()]
    files["symmetric.mtx"] = "\n".join(lines) + "\n"
    # integer field, rectangular
    lines = ["%%MatrixMarket matrix coordinate integer general", "5 7 6",
             "1 1 3", "2 7 -1", "5 2 8", "3 3 1", "4 6 2", "1 1 4"]
    files["integer_rect.mtx"] = "\n".join(lines) + "\n"
    out = {"meta": meta, "mm": {}, "rcm": {}}
    for name, text in files.items():
        path = os.path.join(d, name)
        with open(path, "w") as f:
            f.write(text)
        A = mio.load_matrix_market(path)
        out["mm"][name] = {"n_rows": A.n_rows, "n_cols": A.n_cols, "nnz": A.nnz, "row_ptr": sha(A.row_ptr),
                           "col_idx": sha(A.col_idx), "values": sha(A.values)}
    # RCM permutations
    mats = {"laplace2d:12": mp.generate(mp.StencilSpec(mp.StencilKind("laplace2d"), 12)),
            "convdiff2d:9": mp.generate(mp.StencilSpec(mp.StencilKind("convdiff2d"), 9, convection=3.0)),
            "symmetric.mtx": mio.load_matrix_market(os.path.join(d, "symmetric.mtx")),
            "general_dups.mtx": mio.load_matrix_market(os.path.join(d, "general_dups.mtx"))}
    # a shuffled stencil (RCM recovers a banded order) and a disconnected block matrix
    L = mats["laplace2d:12"]
    p = rng.permutation(L.n_rows)
    mats["laplace2d:12:shuffled"] = mpc.permute_csr(L, mpc.Permutation(p))
    blk = np.zeros((12, 12)); blk[:5, :5] = rng.standard_normal((5, 5)); blk[7:, 7:] = rng.standard_normal((5, 5))
    blk[5, 5] = blk[6, 6] = 1.0
    mats["blocks12"] = mp.CsrMatrix.from_dense(blk)
    for name, A in mats.items():
        perm, B = mpc.rcm_reorder(A)
        out["rcm"][name] = {"n": A.n_rows, "row_ptr": A.row_ptr.tolist(), "col_idx": A.col_idx.tolist(),
                            "perm": perm.perm.tolist(), "permuted_row_ptr": sha(B.row_ptr),
                            "permuted_col_idx": sha(B.col_idx), "permuted_values": sha(B.values),
                            "values": A.values.tolist()}
    with open(os.path.join(HERE, "reference_io.json"), "w") as f:
        json.dump(out, f)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--cfg3", action="store_true")
    ap.add_argument("--cfg4", type=int, choices=[25, 40], default=None)
    ap.add_argument("--cfg5", action="store_true")
    ap.add_argument("--cfg2-fd", type=int, default=None, metavar="SWITCH")
    ap.add_argument("--io", action="store_true")
    ap.add_argument("--cfg5-fp64", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    mp = _ref()
    meta = {"reference": "mpgmres " + mp.__version__, "numpy": np.__version__,
            "generated": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    if not args.skip_small:
        runs = {}
        for name, spec, solver, kw in SMALL_RUNS:
            t = time.time()
            runs[name] = report_dict(run_one(mp, spec, solver, kw))
            print(f"{name}: {runs[name]['total_iters']} it ({time.time() - t:.1f}s)", flush=True)
        with open(os.path.join(HERE, "reference_runs.json"), "w") as f:
            json.dump({"meta": meta, "runs": runs}, f, indent=1)
        asm = {}
        for kind, nx, kw in ASSEMBLY:
            A = mp.generate(mp.StencilSpec(mp.StencilKind(kind), nx, **kw))
            asm[f"{kind}:{nx}:" + ",".join(f"{k}={v}" for k, v in kw.items())] = {
                "kind": kind, "nx": nx, "kwargs": kw, "n": A.n_rows, "nnz": A.nnz,
                "row_ptr": sha(A.row_ptr), "col_idx": sha(A.col_idx), "values": sha(A.values)}
            print("assembly", kind, nx, flush=True)
            del A
        with open(os.path.join(HERE, "assembly_sha256.json"), "w") as f:
            json.dump({"meta": meta, "matrices": asm}, f, indent=1)
        np.savez_compressed(os.path.join(HERE, "spmv_cases.npz"), **spmv_fixtures(mp))
    if args.cfg2:
        runs = {}
        for name, spec, solver, kw in CFG2_RUNS:
            t = time.time()
            runs[name] = report_dict(run_one(mp, spec, solver, kw))
            print(f"{name}: {runs[name]['total_iters']} it ({time.time() - t:.1f}s)", flush=True)
        with open(os.path.join(HERE, "reference_cfg2.json"), "w") as f:
            json.dump({"meta": meta, "runs": runs}, f, indent=1)
    if args.cfg3:
        runs = {}
        for name, spec, solver, kw in CFG3_RUNS:
            t = time.time()
            runs[name] = report_dict(run_one(mp, spec, solver, kw))
            print(f"{name}: {runs[name]['total_iters']} it ({time.time() - t:.1f}s)", flush=True)
        with open(os.path.join(HERE, "reference_cfg3.json"), "w") as f:
            json.dump({"meta": meta, "runs": runs}, f, indent=1)
    if args.cfg5:
        # BASELINE configs[4] (64M rows): a full reference solve is ~40 CPU-hours,
        # so pin the assembly (sha256) and the first GMRES-IR cycle (50 fp32
        # iterations + the fp64 residual) at full size
        t = time.time()
        A = mp.generate(mp.StencilSpec(mp.StencilKind("laplace3d"), 400))
        asm = {"n": A.n_rows, "nnz": A.nnz, "row_ptr": sha(A.row_ptr), "col_idx": sha(A.col_idx),
               "values": sha(A.values)}
        print("cfg5 assembly", asm, f"({time.time() - t:.1f}s)", flush=True)
        b = np.ones(A.n_rows)
        rep = mp.gmres_ir(A, b, criteria=mp.StopCriteria(rtol=1e-10, m=50, max_iters=50))
        runs = {"laplace3d:400/ir/m50/max50": report_dict(rep)}
        print("cfg5 one IR cycle", runs["laplace3d:400/ir/m50/max50"]["boundaries"],
              f"({time.time() - t:.1f}s)", flush=True)
        with open(os.path.join(HERE, "reference_cfg5.json"), "w") as f:
            json.dump({"meta": meta, "assembly": asm, "runs": runs}, f, indent=1)
    if args.cfg2_fd is not None:
        # BASELINE configs[1] lists GMRES-FD beside fp64 and IR: one switch point
        name = f"laplace3d:150/fd{args.cfg2_fd}/m50"
        t = time.time()
        rep = run_one(mp, ("laplace3d", 150, {}), "fd", {"m": 50, "switch_iter": args.cfg2_fd})
        path = os.path.join(HERE, "reference_cfg2.json")
        with open(path) as f:
            d = json.load(f)
        d["runs"][name] = report_dict(rep)
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(f"{name}: {rep.total_iters} it ({time.time() - t:.1f}s)", flush=True)
    if args.io:
        io_fixtures(mp, meta)
    if args.cfg5_fp64:
        # the fp64 GMRES(50) first cycle at 400^3: the Krylov iterate to ~1e-12, against
        # which the fp32 inner cycles' accuracy is judged (test_gpu_solvers cfg5 test)
        t = time.time()
        A = mp.generate(mp.StencilSpec(mp.StencilKind("laplace3d"), 400))
        rep = mp.gmres_restarted(A, np.ones(A.n_rows), criteria=mp.StopCriteria(rtol=1e-10, m=50, max_iters=50))
        path = os.path.join(HERE, "reference_cfg5.json")
        with open(path) as f:
            d = json.load(f)
        d["runs"]["laplace3d:400/fp64/m50/max50"] = report_dict(rep)
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print("cfg5 fp64 cycle", d["runs"]["laplace3d:400/fp64/m50/max50"]["boundaries"],
              f"({time.time() - t:.1f}s)", flush=True)
    if args.cfg4:
        name, spec, solver, kw = CFG4_RUNS[args.cfg4]
        t = time.time()
        runs = {name: report_dict(run_one(mp, spec, solver, kw))}
        print(f"{name}: {runs[name]['total_iters']} it ({time.time() - t:.1f}s)", flush=True)
        with open(os.path.join(HERE, f"reference_cfg4_poly{args.cfg4}.json"), "w") as f:
            json.dump({"meta": meta, "runs": runs}, f, indent=1)


if __name__ == "__main__":
    main()
