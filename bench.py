"""Benchmark: GMRES-IR solve time to 1e-10 on 3D Laplace 150^3 (BASELINE.json
configs[1]; n = 3,375,000, nnz = 23,490,000), GMRES(50), b = ones, x0 = 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

One "step" = one complete GMRES-IR solve from x0 = 0 to rel. residual 1e-10
(~2400 fp32 inner iterations).  The matrix, right-hand side and fp32 copy
are resident in HBM before the timed region (the reference also excludes
the fp32 copy, solvers.py:321); the working set (A64 + A32 + V32 ~ 1.2 GB)
is ~10x the 126 MB L2, so no L2 flush is needed between steps.

Prints ONE JSON line (rank 0).  Extra keys: fp64 GMRES(50) solve time and
the IR speedup on the same GPU, iteration counts, the per-kernel-class
device time of one profiled cycle, the roofline of the dominant kernel,
the CPU oracle timed on this host (cpu_baseline), and the end-to-end time
through the public API with host (numpy) inputs (e2e).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES-IR solve time to 1e-10 rel residual; speedup vs fp64 GMRES; HBM GB/s"
PUBLISHED_V100_IR_S = 11.75      # Laplace3D150 GMRES-IR on V100
REFERENCE_IR_ITERS = 2400        # reference/paper iteration count at this config
NX = 150
M = 50
RTOL = 1e-10


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int = 0):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# algorithmic byte model

def cycle_bytes(n: int, nnz: int, m: int, s: int, storage: str = "csr") -> dict[str, float]:
    """Algorithmic bytes per cycle for each fused kernel class, s = value size.
    CSR: values + col_idx + row_ptr; stencil: the present values only."""
    if storage == "stencil-const":
        spmv = 2 * n * s                                      # coefficients in registers: x once + y once
    elif storage == "stencil":
        spmv = nnz * s + 2 * n * s                            # values + x once + y once
    else:
        spmv = nnz * (s + 4) + 4 * (n + 1) + 2 * n * s       # CSR + x once + y once
    ks = range(1, m + 1)
    return {
        "spmv_dot1": sum(spmv + k * n * s for k in ks),       # + read V[0..k) for pass-1 dots
        "update_dot": sum((k + 2) * n * s for k in ks),       # read V[0..k) + w, write w
        "update_norm_givens": sum((k + 2) * n * s for k in ks),
        "scale": m * 2 * n * s,
        # persistent per-step kernel: matrix + v_j once, V[0..k) three sweeps, v_{j+1}
        # written; w never leaves shared memory
        "step": sum(spmv + 3 * k * n * s for k in ks),
    }


def split_cycle_bytes(model: dict, n: int, nnz: int, m: int, s: int, storage: str) -> dict:
    """K_A split into two launches (the default): the SpMV class moves the
    matrix, x once and w once; the pass-1 dot kernel reads V[0..k) and w.
    Kernel-level algorithmic bytes: each launch's inputs and outputs once."""
    mat = {"stencil-const": 0, "stencil": nnz * s}.get(storage, nnz * (s + 4) + 4 * (n + 1))
    spmv = mat + 2 * n * s
    out = dict(model)
    out["spmv_dot1"] = m * spmv
    out["dot1"] = sum((k + 1) * n * s for k in range(1, m + 1))
    return out


def native_arm(args, rank: int, world: int):
    import numpy as np
    import torch

    import paper_2109_01232_b200 as P
    from paper_2109_01232_b200 import _lib
    from paper_2109_01232_b200.core import FP32, FP64, convert_matrix, padded_copy, dvec
    from paper_2109_01232_b200.solvers import NativeSolve, StopCriteria, gmres_ir

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    spec = P.StencilSpec(P.StencilKind.LAPLACE3D, NX)
    A = P.generate(spec)
    n, nnz = A.n_rows, A.nnz
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    crit = StopCriteria(rtol=RTOL, m=M)
    # warm-up (also builds + caches the CUDA graphs' kernels/attributes)
    for _ in range(args.warmup):
        rep = gmres_ir(A, b, criteria=crit)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    l0 = _lib.launch_count()
    times, iters = [], []
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        for _ in range(args.steps):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            if _ == 0:
                e0.record()
            rep = gmres_ir(A, b, criteria=crit)
            s1.record()
            s1.synchronize()
            times.append(s0.elapsed_time(s1) / 1e3)
            iters.append(rep.total_iters)
        e1.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - l0
    total_s = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([total_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_s = float(t.item())
    solve_s = total_s / args.steps
    x_ir = rep.x
    res_ir, _ = P.explicit_residual(A, b, x_ir)
    # fp64 GMRES(50) on the same GPU (speedup denominator): warmed up like the
    # IR solve, then the mean of two timed solves
    P.gmres_restarted(A, b, criteria=crit)
    f64 = []
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rep64 = P.gmres_restarted(A, b, criteria=crit)
        e1.record()
        e1.synchronize()
        f64.append(e0.elapsed_time(e1) / 1e3)
    fp64_s = sum(f64) / len(f64)
    sol_diff = float(torch.linalg.norm(rep64.x - x_ir) / torch.linalg.norm(rep64.x))

    # the same two solves with BOTH forced onto one Arnoldi-step implementation
    # (the default picks the persistent step for the 13.5 MB fp32 vectors and the
    # four-launch step for the 27 MB fp64 ones): the IR speedup without any
    # kernel asymmetry
    def timed(f):
        f()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        r = f()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3, r.total_iters
    same_kernel = {}
    for mode in ("persistent", "split"):
        with P.solvers.step_kernel(mode):
            t_ir, it_ir = timed(lambda: gmres_ir(A, b, criteria=crit))
            t_64, it_64 = timed(lambda: P.gmres_restarted(A, b, criteria=crit))
        same_kernel[mode] = {"ir_s": round(t_ir, 5), "ir_iters": it_ir, "fp64_s": round(t_64, 5),
                             "fp64_iters": it_64, "speedup": round(t_64 / t_ir, 3)}

    # one profiled (eager) IR cycle per storage: per-kernel-class device time
    A32 = convert_matrix(A, FP32)
    bd = padded_copy(b, FP64)
    profiles = {}
    for storage in ("stencil", "csr"):
        ns = NativeSolve(_lib.MODE_IR, FP32, A32, A, bd, dvec(n, FP64), M, RTOL, storage=storage)
        ns.begin()
        ns.cycle(M)                                   # warm
        prof = ns.profile_cycle(M)
        used = ns.storage
        ns.close()
        model = cycle_bytes(n, nnz, M, 4, used)
        if prof.get("dot1", (0.0, 0))[1] > 0:
            model = split_cycle_bytes(model, n, nnz, M, 4, used)
        # only the classes this cycle actually launched
        model = {k: v for k, v in model.items() if prof.get(k, (0.0, 0))[1] > 0}
        # (K_S fused into K_C: "scale" has no launches and drops out above; the fused
        # kernel's read V + w', write v = (k+2) n s is update_norm_givens' count)
        kernels = {}
        for k, (ms, cnt) in prof.items():
            kernels[k] = {"ms_per_cycle": round(ms, 4), "launches": cnt}
            if k in model and ms > 0:
                kernels[k]["GBps"] = round(model[k] / (ms / 1e3) / 1e9, 1)
        cyc_ms = sum(v[0] for v in prof.values())
        profiles[storage] = {"storage": used, "ms": round(cyc_ms, 4),
                             "GBps_algorithmic": round(sum(model.values()) / (cyc_ms / 1e3) / 1e9, 1),
                             "kernels": kernels, "_prof": prof, "_model": model}
    peak, peak_kind = _peaks()
    main = profiles["stencil"]
    prof, model = main.pop("_prof"), main.pop("_model")
    profiles["csr"].pop("_prof"), profiles["csr"].pop("_model")
    dom = max((k for k in model if k in prof), key=lambda k: prof[k][0])
    dom_gbs = model[dom] / (prof[dom][0] / 1e3) / 1e9

    # BASELINE configs[4] (64M rows) on this GPU: two restart cycles (north_star's
    # per-kernel GB/s at the 400^3 size); skipped with --no-cfg5
    cfg5 = None if args.no_cfg5 else cfg5_segment_single()

    # end to end through the public API with HOST inputs (numpy CSR + b)
    rp, ci, v = A.host_arrays()

    class HostCsr:  # the reference's CsrMatrix shape (numpy arrays)
        pass
    def pinned(a):   # host inputs in page-locked memory (numpy views)
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    Ah = HostCsr()
    Ah.n_rows = Ah.n_cols = n
    Ah.row_ptr, Ah.col_idx, Ah.values = pinned(rp), pinned(ci), pinned(v)
    bh = pinned(np.ones(n))
    # one untimed call (allocator pools, first-touch), then K timed steps; each
    # step uploads A and b, solves, and returns x as numpy (device -> host)
    gmres_ir(Ah, bh, criteria=crit)
    e2e_times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep_h = gmres_ir(Ah, bh, criteria=crit)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times) / len(e2e_times)
    h2d = rp.nbytes + ci.nbytes + v.nbytes + bh.nbytes
    d2h = rep_h.x.nbytes

    out = {
        "metric": METRIC,
        "value": round(solve_s, 5),
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(solve_s * 1e3, 3),
        "higher_is_better": False,
        "scaling": "replicas" if world > 1 else "strong",
        "vs_baseline": round(solve_s / PUBLISHED_V100_IR_S, 5),
        "vs_baseline_note": "value / published V100 GMRES-IR time 11.75 s (PAPER.md:461)",
        "dtype": "f32 inner / f64 outer",
        "data": "synthetic (reference generator, on device); b = ones, x0 = 0",
        "config": {"workload": "gmres_ir laplace3d:150 GMRES(50) rtol=1e-10 (BASELINE configs[1])",
                   "n": n, "nnz": nnz, "m": M, "rtol": RTOL,
                   "l2": "working set ~1.2 GB >> 126 MB L2; no flush needed"},
        "iters": iters[-1],
        "iters_reference": REFERENCE_IR_ITERS,
        "final_rel_residual": res_ir / float(torch.linalg.norm(b)),
        "fp64_solve_s": round(fp64_s, 5),
        "fp64_iters": rep64.total_iters,
        "speedup_vs_fp64": round(fp64_s / solve_s, 3),
        "speedup_same_step_kernel": same_kernel,
        "solution_rel_diff_ir_vs_fp64": sol_diff,
        "step_times_s": [round(t, 5) for t in times],
        "kernel_times_s": {k: round(v, 5) for k, v in rep.kernel_times.items()},
        "storage": main["storage"],
        "profile_cycle": main,
        "profile_cycle_csr": profiles["csr"],
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(dom_gbs, 1), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(dom_gbs / peak, 4),
                     "algorithmic_bytes_per_launch": round(model[dom] / prof[dom][1]),
                     "launches_per_cycle": prof[dom][1],
                     **_traffic(dom)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cfg5_segment": cfg5,
        "e2e": {"value": round(e2e_s, 5), "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "iters": rep_h.total_iters,
                "step_times_s": [round(t, 5) for t in e2e_times],
                "note": "gmres_ir on host (pinned numpy) CSR arrays + b, x returned as numpy; "
                        "wall clock per call, mean of the timed steps after one untimed call"},
    }
    return out



def _max_over_ranks_profile(prof: dict) -> dict:
    """Per-class device ms of one rank's profiled cycle -> max over ranks (the
    slowest rank sets the pace), with this rank's bytes (ranks hold equal
    plane counts up to one plane) and the communication share."""
    import torch
    keys = sorted(prof)
    t = torch.tensor([prof[k]["ms"] for k in keys], dtype=torch.float64, device="cuda")
    if torch.distributed.is_initialized():
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    out = {}
    for i, k in enumerate(keys):
        d = dict(prof[k])
        d["ms"] = round(float(t[i]), 4)
        if d.get("bytes") and d["ms"] > 0:
            d["GBps"] = round(d["bytes"] / (d["ms"] / 1e3) / 1e9, 1)
        out[k] = d
    total = sum(d["ms"] for d in out.values())
    comm = sum(out[k]["ms"] for k in ("allreduce", "halo", "post") if k in out)
    out["_summary"] = {"cycle_ms": round(total, 4), "comm_ms": round(comm, 4),
                       "comm_share": round(comm / total, 4) if total else None,
                       "note": "per rank, max over ranks; comm = allreduce + halo exchange + post kernels"}
    return out


def _dist_roofline(prof: dict) -> dict | None:
    """Roofline of the dominant phase kernel class of a distributed cycle
    (algorithmic bytes of this rank's rows / device time, max over ranks)."""
    cls = [k for k in ("step", "spmv_dot", "update_dot", "update_norm", "scale") if k in prof and prof[k].get("GBps")]
    if not cls:
        return None
    dom = max(cls, key=lambda k: prof[k]["ms"])
    peak, kind = _peaks()
    a = prof[dom]["GBps"]
    return {"bound": "hbm", "kernel": dom, "achieved": a, "peak": peak, "peak_kind": kind, "unit": "GB/s",
            "frac": round(a / peak, 4), "algorithmic_bytes_per_cycle": prof[dom]["bytes"],
            "launches_per_cycle": prof[dom]["launches"], "traffic": None,
            "note": "per rank; ncu is not run on multi-rank commands (B200_PROFILING.md)"}


CFG5_NX = 400          # BASELINE configs[4]: Laplace3D 400^3, 64M rows
CFG5_ITERS = 100       # two restart cycles (time 1-2 cycles, report s/iteration)


def cfg5_segment_single() -> dict:
    """BASELINE configs[4] on one GPU: GMRES-IR and fp64 GMRES(50) for a fixed
    two restart cycles of Laplace3D 400^3 (64M rows; the full solve needs
    ~15k iterations), s/iteration, the per-kernel-class GB/s of one profiled
    IR cycle and the explicit residual reached."""
    import torch
    import paper_2109_01232_b200 as P
    from paper_2109_01232_b200 import _lib
    from paper_2109_01232_b200.core import FP32, FP64, convert_matrix, padded_copy, dvec
    from paper_2109_01232_b200.solvers import NativeSolve, StopCriteria, gmres_ir
    A = P.generate(P.StencilSpec(P.StencilKind.LAPLACE3D, CFG5_NX))
    n, nnz = A.n_rows, A.nnz
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    crit = StopCriteria(rtol=RTOL, m=M, max_iters=CFG5_ITERS)
    out = {"workload": f"laplace3d:{CFG5_NX} (BASELINE configs[4]), GMRES(50), {CFG5_ITERS} iterations",
           "n": n, "nnz": nnz}
    for name, f in (("ir", lambda: gmres_ir(A, b, criteria=crit)),
                    ("fp64", lambda: P.gmres_restarted(A, b, criteria=crit))):
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = f()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        out[name] = {"s": round(t, 4), "iters": rep.total_iters, "s_per_iter": round(t / rep.total_iters, 6),
                     "explicit_rel_residual": rep.residual_history[-1].explicit}
    out["speedup_ir_vs_fp64"] = round(out["fp64"]["s"] / out["ir"]["s"], 3)
    A32 = convert_matrix(A, FP32)
    ns = NativeSolve(_lib.MODE_IR, FP32, A32, A, padded_copy(b, FP64), dvec(n, FP64), M, RTOL)
    ns.begin()
    ns.cycle(M)
    prof = ns.profile_cycle(M)
    used = ns.storage
    ns.close()
    model = cycle_bytes(n, nnz, M, 4, used)
    if prof.get("dot1", (0.0, 0))[1] > 0:
        model = split_cycle_bytes(model, n, nnz, M, 4, used)
    kern = {}
    for k, (ms, cnt) in prof.items():
        if cnt:
            kern[k] = {"ms_per_cycle": round(ms, 4), "launches": cnt}
            if k in model and ms > 0:
                kern[k]["GBps"] = round(model[k] / (ms / 1e3) / 1e9, 1)
    out["profile_cycle"] = {"storage": used, "kernels": kern}
    del A, A32, b
    torch.cuda.empty_cache()
    return out


def cfg5_segment_dist(world: int, rank: int, coll, peer: bool, persistent="auto") -> dict:
    """BASELINE configs[4] row-partitioned over the ranks: GMRES-IR for a fixed
    two restart cycles of Laplace3D 400^3, s/iteration (max over ranks), the
    profiled cycle's per-phase GB/s and communication share."""
    import torch
    import paper_2109_01232_b200 as P
    from paper_2109_01232_b200.dist import DistributedStencilSolver, RowPartition, _dist_solve
    from paper_2109_01232_b200.solvers import StopCriteria
    spec = P.StencilSpec(P.StencilKind.LAPLACE3D, CFG5_NX)
    part = RowPartition.for_stencil(3, CFG5_NX, world, rank)
    crit = StopCriteria(rtol=RTOL, m=M, max_iters=CFG5_ITERS)
    solver = DistributedStencilSolver(spec, part, "ir", M, RTOL, coll, peer_halo=peer, persistent=persistent)
    try:
        solver.x_buf.zero_()
        _dist_solve(solver, crit, True, None)                 # warm (graphs captured)
        solver.x_buf.zero_()
        torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = _dist_solve(solver, crit, True, None)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        solver.x_buf.zero_()
        solver.begin()
        prof = _max_over_ranks_profile(solver.profile_cycle(M))
    finally:
        solver.close()
    ts = float(t.item())
    return {"workload": f"laplace3d:{CFG5_NX} (BASELINE configs[4]) row-partitioned over {world} ranks, "
                        f"GMRES-IR GMRES(50), {CFG5_ITERS} iterations",
            "n": CFG5_NX ** 3, "n_local": part.n_local, "s": round(ts, 4), "iters": rep.total_iters,
            "s_per_iter": round(ts / max(rep.total_iters, 1), 6),
            "explicit_rel_residual": rep.residual_history[-1].explicit,
            "profile_cycle": prof, "roofline": _dist_roofline(prof)}


def _traffic(cls: str) -> dict:
    """DRAM bytes per launch of kernel class `cls` from the committed ncu capture
    of one cfg2 IR cycle (tools/traffic_from_ncu.py; L2 flushed per launch)."""
    path = os.path.join(ROOT, "profiles", "r2_traffic_ir_cycle.json")
    try:
        with open(path) as f:
            c = json.load(f)["classes"][cls]
        return {"traffic": round(c["dram_bytes_per_launch"]),
                "traffic_source": "profiles/r2_traffic_ir_cycle.json (ncu dram__bytes_read+write, "
                                  "mean over the cycle's launches)"}
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def _backend() -> str:
    """NCCL with one GPU per rank; gloo (host-staged collectives, a smoke run of
    the same path) when ranks outnumber the visible GPUs.  MPG_BENCH_BACKEND
    overrides."""
    import torch
    env = os.environ.get("MPG_BENCH_BACKEND")
    if env:
        return env
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return "gloo" if world > max(1, torch.cuda.device_count()) else "nccl"


def dist_arm(args, rank: int, world: int):
    """--gpus N > 1: the same cfg2 GMRES-IR solve row-partitioned over N GPUs
    (one process per GPU, NCCL halo exchange + allreduces), strong scaling."""
    import numpy as np
    import torch

    import paper_2109_01232_b200 as P
    from paper_2109_01232_b200 import _lib
    from paper_2109_01232_b200.dist import Collectives, DistributedStencilSolver, RowPartition, _dist_solve
    from paper_2109_01232_b200.solvers import StopCriteria

    from paper_2109_01232_b200.dist import HostStagedCollectives
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    spec = P.StencilSpec(P.StencilKind.LAPLACE3D, NX)
    part = RowPartition.for_stencil(3, NX, world, rank)
    # NCCL (device collectives) on the multi-GPU box; gloo only for smoke runs
    # of this path with several ranks sharing one GPU (MPG_BENCH_BACKEND=gloo)
    coll = HostStagedCollectives() if _backend() == "gloo" else Collectives()
    crit = StopCriteria(rtol=RTOL, m=M)
    # NVLink peer-memory halos written by the SCALE phase (MPG_PEER_HALO=0: NCCL send/recv)
    peer = os.environ.get("MPG_PEER_HALO", "1") != "0"
    # one cooperative kernel per Arnoldi step with the cross-rank sums done
    # in-kernel over peer memory (MPG_DIST_PERSISTENT=0: the phase path, NCCL
    # allreduces between per-phase kernels)
    pers = "auto" if os.environ.get("MPG_DIST_PERSISTENT", "1") != "0" else False
    solver = DistributedStencilSolver(spec, part, "ir", M, RTOL, coll, peer_halo=peer, persistent=pers)

    def solve():
        solver.x_buf.zero_()
        return _dist_solve(solver, crit, True, None)

    for _ in range(args.warmup):
        rep = solve()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    l0 = _lib.launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            rep = solve()
        e1.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - l0
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    solve_s = float(t.item()) / args.steps
    # one eager profiled cycle: per-phase device time, GB/s, communication share
    solver.x_buf.zero_()
    solver.begin()
    prof = _max_over_ranks_profile(solver.profile_cycle(M))
    cfg5 = cfg5_segment_dist(world, rank, coll, peer, pers)
    # e2e: the public distributed API with a host right-hand side slice, x
    # downloaded; every call assembles this rank's rows, maps the peers and
    # captures the cycle graph (what a user's call costs).  One untimed call,
    # then the mean of `steps` timed calls, max over ranks.
    b_host = np.ones(part.n_local)
    from paper_2109_01232_b200.dist import dist_gmres_ir

    def e2e_call():
        r = dist_gmres_ir(spec, part, coll, crit, b_local=b_host, peer_halo=peer, persistent=pers)
        return r, r.x.cpu().numpy()
    e2e_call()
    e2e_t = []
    for _ in range(args.steps):
        torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep_h, x_host = e2e_call()
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e = torch.tensor([sum(e2e_t) / len(e2e_t)], device="cuda")
    torch.distributed.all_reduce(e2e, op=torch.distributed.ReduceOp.MAX)
    solver.close()
    return {
        "metric": METRIC, "value": round(solve_s, 5), "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(solve_s * 1e3, 3),
        "higher_is_better": False, "scaling": "strong",
        "vs_baseline": round(solve_s / PUBLISHED_V100_IR_S, 5),
        "vs_baseline_note": "value / published V100 GMRES-IR time 11.75 s (PAPER.md:461)",
        "dtype": "f32 inner / f64 outer", "data": "synthetic (per-rank device assembly); b = ones, x0 = 0",
        "config": {"workload": "gmres_ir laplace3d:150 GMRES(50) rtol=1e-10 (BASELINE configs[1]), "
                               "row-partitioned by z-planes",
                   "n": NX ** 3, "m": M, "rtol": RTOL, "parallelism": f"rows{world}",
                   "collectives": ("one cooperative kernel per Arnoldi step per rank: the three cross-rank "
                                   "sums done in-kernel over peer-memory exchange boxes (release/acquire "
                                   "sequence numbers), halo planes stored into the neighbours by the kernel; "
                                   "NCCL only for the per-cycle start/residual sums" if solver.persistent else
                                   ("peer-memory halo stores fused into the basis scaling + " if solver.peer
                                    else "NCCL halo send/recv + ") + "3 NCCL allreduces per Arnoldi step")
                                  + "; whole cycles replayed as CUDA graphs",
                   "l2": "working set >> L2 per rank at N<=8; no flush needed"},
        "iters": rep.total_iters, "iters_reference": REFERENCE_IR_ITERS,
        "storage": "stencil", "gpu_launches": launches, "clocks": clk.summary(),
        "profile_cycle": prof,
        "roofline": _dist_roofline(prof),
        "cfg5_segment": cfg5,
        "e2e": {"value": round(float(e2e.item()), 5), "unit": "s",
                "h2d_bytes_per_step": int(b_host.nbytes) * world, "d2h_bytes_per_step": int(x_host.nbytes) * world,
                "iters": rep_h.total_iters,
                "note": "dist_gmres_ir per call (per-rank assembly, peer mappings, graph capture, solve, x to host); "
                        "mean of the timed calls after one untimed call, max over ranks"},
        "smoke": _backend() == "gloo",
        "smoke_note": ("ranks share one GPU (gloo, time-sliced): a functional run of the multi-GPU path, "
                       "not a performance number") if _backend() == "gloo" else None,
    }


def _stock_reference():
    """The unmodified reference package staged by `pip install --target
    baseline/_ref /root/reference/pkg`, or None when it is not
    staged (then the bit-identical oracle port stands in, kind "port")."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "mpgmres")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import mpgmres
    except Exception:
        return None
    return mpgmres


_REF_CACHE = {}


def cpu_sample(threads: int | None, iters: int = M):
    """The reference's GMRES-IR at the bench config, bounded to its first
    `iters` fp32 inner iterations (one 50-step restart cycle + the fp64
    refinement residual): the stock `mpgmres.gmres_ir` through its public API
    (its own `deterministic_kernels()` pins BLAS to one thread, core.py:51-67),
    timed by its own SolveReport.total_time (perf_counter around the solve,
    solvers.py:327-383).  Returns a dict with the extrapolated full-solve
    seconds (x 2400 / iters: every cycle of the reference solve runs the same
    50 steps) and the measured sample."""
    ref = _stock_reference()
    if ref is not None:
        if "A" not in _REF_CACHE:
            import numpy as np
            A = ref.generate(ref.StencilSpec(ref.StencilKind.LAPLACE3D, NX))
            _REF_CACHE["A"] = (A, np.ones(A.n_rows))
        A, b = _REF_CACHE["A"]
        rep = ref.gmres_ir(A, b, criteria=ref.StopCriteria(rtol=RTOL, m=M, max_iters=iters))
        dt, it, kind, cores = rep.total_time, rep.total_iters, "reference", 1
        what = "baseline/_ref mpgmres.gmres_ir (stock, 1 BLAS thread as its deterministic_kernels pins)"
        kt = {k: round(v, 4) for k, v in rep.kernel_times.items()}
    else:
        from oracle import cpu_gmres as O
        if "Ao" not in _REF_CACHE:
            Ao = O.stencil_csr("laplace3d", NX)
            _REF_CACHE["Ao"] = (Ao, O.ones_rhs(Ao.n_rows))
        A, b = _REF_CACHE["Ao"]
        t0 = time.perf_counter()
        rep = O.solve_ir(A, b, m=M, max_iters=iters, threads=threads)
        dt, it, kind, cores = time.perf_counter() - t0, rep.total_iters, "port", threads or 1
        what = "oracle/cpu_gmres.py solve_ir (port; the reference is not staged in baseline/_ref)"
        kt = None
    factor = REFERENCE_IR_ITERS / it
    return {"value": dt * factor, "sample_s": dt, "sample_iters": it, "extrapolation_factor": factor,
            "kind": kind, "cores": cores, "what": what, "kernel_times": kt}


def reference_arm(args, rank: int, world: int):
    """--impl reference: the reference's own CPU solver on this host (rank 0
    only).  Each step is one bounded sample -- the first 50-iteration restart
    cycle of the cfg2 GMRES-IR solve (~13 s on one core) -- extrapolated to the
    reference's 2400 iterations; warm-up steps run a 1-iteration solve (page-in
    and first-call costs only)."""
    if rank != 0:
        return None
    samples = []
    for i in range(args.warmup + args.steps):
        s = cpu_sample(None, iters=1 if i < args.warmup else M)
        if i >= args.warmup:
            samples.append(s)
    val = statistics.mean(s["value"] for s in samples)
    meas = sum(s["sample_s"] for s in samples)
    last = samples[-1]
    cb = {"value": round(val, 3), "unit": "s", "cores": last["cores"], "kind": last["kind"],
          "sample": f"{last['what']}: each step the first {last['sample_iters']}-iteration IR cycle "
                    f"(+ fp64 residual) of the cfg2 solve, extrapolated x{last['extrapolation_factor']:g} "
                    f"to 2400 iterations",
          "sample_s_per_step": round(meas / len(samples), 3),
          "sample_iters_per_step": last["sample_iters"],
          "extrapolation_factor": last["extrapolation_factor"],
          "measured_region_s": round(meas, 2),
          "kernel_times_last_sample_s": last["kernel_times"]}
    return {
        "metric": METRIC, "impl": "reference", "value": round(val, 3), "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(val * 1e3, 1), "higher_is_better": False, "scaling": "strong",
        "value_is_extrapolated": True,
        "vs_baseline": round(val / PUBLISHED_V100_IR_S, 3), "dtype": "f32 inner / f64 outer",
        "data": "synthetic; b = ones, x0 = 0",
        "config": {"workload": "gmres_ir laplace3d:150 GMRES(50) rtol=1e-10 (BASELINE configs[1])"},
        "cpu_baseline": cb,
        "e2e": {"value": round(val, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the 400^3 (configs[4]) segment")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        out = reference_arm(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        torch.distributed.init_process_group(_backend())
        out = dist_arm(args, rank, world)
    else:
        out = native_arm(args, rank, world)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:   # the CPU baseline rides on the N=1 line only
            cs = cpu_sample(1)
            out["cpu_baseline"] = {
                "value": round(cs["value"], 3), "unit": "s", "cores": cs["cores"], "kind": cs["kind"],
                "sample": f"{cs['what']}: the first {cs['sample_iters']}-iteration IR cycle "
                          f"({cs['sample_s']:.1f} s), extrapolated x{cs['extrapolation_factor']:g} to 2400 iterations",
                "sample_s": round(cs["sample_s"], 3), "sample_iters": cs["sample_iters"],
                "extrapolation_factor": cs["extrapolation_factor"]}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
