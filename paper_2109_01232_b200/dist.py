"""Row-partitioned multi-GPU GMRES (the reference is single-process).

One process per GPU.  Rank r owns a contiguous block of whole grid planes
(z-planes for the 7-point 3-D stencil, y-lines for 5-point 2-D stencils), so
its halo is exactly one plane on each side.  Every vector the SpMV reads
(each Krylov basis vector and the iterate) is stored with its halo planes
right around the owned block, so the stencil kernel reads neighbours in
place — no pack/unpack copies.

Per Arnoldi step the path has exactly the exchanges the algorithm needs:
one halo exchange before the SpMV and one sum-allreduce after each of the
three reduction phases (pass-1 dots + ||w||^2 + non-finite flag, pass-2
dots, ||w''||^2).  The kernels run in "dist" mode (raw local sums), the
allreduce sums them across ranks, and a 1-CTA post kernel finishes the phase
identically on every rank (the Hessenberg/Givens state is replicated
bit-identically, because every rank post-processes the same reduced bits).

Collectives go through ``torch.distributed`` (NCCL over NVLink on the B200
box: device tensors, graph-capturable; gloo for CPU tests and single-GPU
multi-process checks, host-staged).  The host loop is the reference's
restart bookkeeping (solvers.py:177-227 / :297-384).
"""

from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, timing
from .core import DIA_TAIL, FP32, FP64, Precision, PrecisionError, device, padded_length, ptr, stream_handle
from .solvers import (LOSS_OF_ACCURACY_FACTOR, STALL_IMPROVEMENT, STALL_RESTARTS, HistoryEntry,
                      SolveReport, StopCriteria, _raise_flags, _relative)

__all__ = ["RowPartition", "plane_partition", "Collectives", "HostStagedCollectives",
           "NullCollectives", "DistributedStencilSolver", "dist_gmres_ir", "dist_gmres_restarted"]

PH = {name: i for i, name in enumerate(
    ["BNORM", "POST_BNORM", "RESID", "POST_RESID", "START", "POST_START", "START_SCALE",
     "SPMV_DOT", "POST_DOT1", "UPDATE_DOT", "POST_DOT2", "UPDATE_NORM", "POST_NORM", "SCALE",
     "FINISH", "STEP"])}
MEGA_MAX_K = 56   # csrc/state.cuh kMegaMaxK: the persistent step covers k <= 56 basis vectors


def plane_partition(n_planes: int, world: int) -> list[tuple[int, int]]:
    """Contiguous plane blocks [floor(r*P/W), floor((r+1)*P/W))."""
    if n_planes < world:
        raise ValueError(f"{world} ranks need at least {world} grid planes, got {n_planes}")
    return [((r * n_planes) // world, ((r + 1) * n_planes) // world) for r in range(world)]


@dataclass(frozen=True)
class RowPartition:
    """This rank's rows of a row-partitioned stencil matrix."""

    dims: int
    nx: int
    world: int
    rank: int
    row0: int
    row1: int
    halo: int

    @classmethod
    def for_stencil(cls, dims: int, nx: int, world: int, rank: int) -> "RowPartition":
        plane = nx ** (dims - 1)
        p0, p1 = plane_partition(nx, world)[rank]
        return cls(dims, nx, world, rank, p0 * plane, p1 * plane, plane)

    @property
    def n_local(self) -> int:
        return self.row1 - self.row0

    @property
    def n_global(self) -> int:
        return self.nx ** self.dims

    @property
    def prev(self) -> int | None:
        return self.rank - 1 if self.rank > 0 else None

    @property
    def next(self) -> int | None:
        return self.rank + 1 if self.rank + 1 < self.world else None

    @property
    def own_offset(self) -> int:
        """Offset of the owned block inside each padded vector row."""
        return padded_length(self.halo)

    @property
    def ld(self) -> int:
        """Row stride of the basis: each padded row holds its own lower halo,
        owned block and upper halo (so consecutive rows never overlap)."""
        return padded_length(self.own_offset + self.n_local + self.halo)


# ---------------------------------------------------------------------------
# collectives

class Collectives:
    """Sum-allreduce and halo exchange over torch.distributed (NCCL: device
    tensors, in stream order, capturable in a CUDA graph)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        # NCCL collectives are stream-ordered device work: a cycle can be graph-captured
        try:
            self.capturable = dist.get_backend(group) == "nccl"
        except Exception:  # pragma: no cover
            self.capturable = False

    def allreduce_(self, t: torch.Tensor) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def halo_(self, row: torch.Tensor, part: RowPartition) -> None:
        """row: one padded vector (halo | owned | halo around own_offset).
        Sends the first/last `halo` owned values to the previous/next rank,
        receives theirs into this row's lower/upper halo."""
        d, o, n, h = self.dist, part.own_offset, part.n_local, part.halo
        ops = []
        if part.prev is not None:
            ops.append(d.P2POp(d.isend, row[o:o + h], part.prev, self.group))
            ops.append(d.P2POp(d.irecv, row[o - h:o], part.prev, self.group))
        if part.next is not None:
            ops.append(d.P2POp(d.isend, row[o + n - h:o + n], part.next, self.group))
            ops.append(d.P2POp(d.irecv, row[o + n:o + n + h], part.next, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()


class HostStagedCollectives(Collectives):
    """Collectives for a gloo group with device tensors (host-staged copies):
    lets several ranks share one GPU in tests, and runs on CPU tensors too."""

    capturable = False

    def __init__(self, group=None):
        super().__init__(group)
        self.capturable = False

    def allreduce_(self, t: torch.Tensor) -> None:
        h = t.detach().to("cpu", copy=True)
        super().allreduce_(h)
        t.copy_(h)

    def halo_(self, row: torch.Tensor, part: RowPartition) -> None:
        h = row.detach().to("cpu", copy=True)
        super().halo_(h, part)
        o, n, hh = part.own_offset, part.n_local, part.halo
        if part.prev is not None:
            row[o - hh:o].copy_(h[o - hh:o])
        if part.next is not None:
            row[o + n:o + n + hh].copy_(h[o + n:o + n + hh])


class NullCollectives:
    """World size 1: the sum over one rank is the identity, no neighbours."""

    capturable = True

    def allreduce_(self, t: torch.Tensor) -> None:
        return None

    def halo_(self, row: torch.Tensor, part: RowPartition) -> None:
        return None


def _enable_peer(dev: torch.device) -> None:
    """IPC mappings of another GPU's memory are opened in that GPU's context;
    our kernels on this GPU store into them, which needs peer access from
    this device (a no-op when the ranks share a device, as in the tests)."""
    if dev.index is None or dev.index == torch.cuda.current_device():
        return
    rc = _lib.load().mpg_enable_peer(int(dev.index))
    if rc:
        raise RuntimeError(f"peer access {torch.cuda.current_device()} -> {dev.index} unavailable (rc {rc})")


# ---------------------------------------------------------------------------
# the per-rank native solver

class DistributedStencilSolver:
    """One rank of a row-partitioned GMRES-IR / GMRES(m) solve on a 5/7-point
    stencil matrix assembled per rank on the device (mpg_generate_stencil
    for the rank's rows, packed with mpg_stencil_pack_rows)."""

    def __init__(self, spec, part: RowPartition, mode: str, m: int, rtol: float,
                 collectives, precision: Precision = FP64, b_local=None, use_graph: bool = True,
                 peer_halo: bool = False, group=None, persistent: bool | str = False):
        from .gen import generate_rows
        if mode not in ("ir", "restarted"):
            raise ValueError("mode must be 'ir' or 'restarted'")
        self.spec, self.part, self.m, self.rtol, self.coll = spec, part, m, rtol, collectives
        # CUDA-graph replay of whole cycles needs stream-ordered device collectives
        self.use_graph = bool(getattr(collectives, "capturable", False)) and use_graph
        self._graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self._eager_cycles: dict[int, int] = {}
        self.mode = _lib.MODE_IR if mode == "ir" else _lib.MODE_RESTARTED
        self.prec = FP32 if mode == "ir" else precision
        outer = FP64 if mode == "ir" else precision
        self.outer = outer
        n, o, ld = part.n_local, part.own_offset, part.ld
        dev = device()
        lib = _lib.load()
        # local rows of the fp64 matrix, packed into the stencil storage
        rp, ci, v64 = generate_rows(spec, part.row0, part.row1)
        S = 7 if part.dims == 3 else 5
        self._dia = {}
        for p in {FP64, self.prec}:
            vals = v64 if p is FP64 else v64.to(torch.float32)
            # slot stride = the descriptor's ldv (the kernels index both with it)
            dia = torch.zeros(S * ld + DIA_TAIL, dtype=p.torch_dtype, device=dev)   # + header tail
            bad = torch.zeros(1, dtype=torch.int32, device=dev)
            _lib.call("mpg_stencil_pack_rows", p.code, part.dims, part.nx, part.row0, n, ptr(rp),
                      ptr(ci), ptr(vals), ptr(dia), ld, ptr(bad), stream_handle())
            if int(bad.item()):
                raise ValueError("the partition's rows are not a 5/7-point stencil")
            self._dia[p] = dia
        self._csr = (rp, ci, v64, v64.to(torch.float32) if self.prec is FP32 else v64)
        # vectors: x (outer, with halos), b, r (outer), r_in (IR fp32), V rows with halos
        self.x_buf = torch.zeros(ld, dtype=outer.torch_dtype, device=dev)
        self.b = torch.zeros(padded_length(n), dtype=outer.torch_dtype, device=dev)
        if b_local is None:
            self.b[:n] = 1.0
        else:
            self.b[:n].copy_(torch.as_tensor(b_local, dtype=outer.torch_dtype))
        self.r = torch.zeros(padded_length(n), dtype=outer.torch_dtype, device=dev)
        self.r_in = torch.zeros(padded_length(n), dtype=torch.float32, device=dev) \
            if self.mode == _lib.MODE_IR else None
        self.V_buf = torch.zeros((m + 1) * ld + o, dtype=self.prec.torch_dtype, device=dev)
        self.w = torch.zeros(padded_length(n), dtype=self.prec.torch_dtype, device=dev)
        self.u = torch.zeros(padded_length(n), dtype=self.prec.torch_dtype, device=dev)
        from .krylov import DeviceState
        self.state = DeviceState(m, self.prec)
        self.ws = torch.zeros(int(lib.mpg_workspace_bytes()), dtype=torch.uint8, device=dev)
        s = self.prec.dtype.itemsize
        red_off = int(lib.mpg_state_offset(self.prec.code, m, 9))
        self.red = self.state.buf[red_off: red_off + s * (m + 8)].view(self.prec.torch_dtype)
        res_off = _lib.StateHeader.reserved.offset             # header reserved[0]
        self.reserved0 = self.state.buf[res_off: res_off + 8].view(torch.float64)
        d = _lib.SolverDesc()
        d.mode, d.prec, d.m, d.use_graph = self.mode, self.prec.code, m, 0
        d.n, d.ldv, d.rtol = n, ld, float(rtol)
        d.breakdown_tol = 10.0 * self.prec.unit_roundoff
        d.row_ptr, d.col_idx = ptr(rp), ptr(ci)
        d.values = ptr(self._csr[3])
        d.values64 = ptr(v64) if self.mode == _lib.MODE_IR else None
        d.x, d.b, d.r = ptr(self.x_buf) + o * outer.dtype.itemsize, ptr(self.b), ptr(self.r)
        d.r_in = ptr(self.r_in) if self.r_in is not None else None
        d.V = ptr(self.V_buf) + o * s
        d.w, d.u = ptr(self.w), ptr(self.u)
        d.state, d.ws = ptr(self.state.buf), ptr(self.ws)
        d.stencil_dims, d.stencil_nx = part.dims, part.nx
        d.dia = ptr(self._dia[self.prec])
        d.dia64 = ptr(self._dia[FP64]) if self.mode == _lib.MODE_IR else None
        d.dist, d.row0, d.halo = 1, part.row0, part.halo
        # distributed persistent step: one cooperative kernel per Arnoldi step,
        # its three cross-rank sums over peer-memory exchange boxes (needs the
        # peer halo across ranks, and every step inside the kernel's k range)
        # "auto": the same rule as the single-GPU solver (csrc/solver.cu): the
        # persistent step while a basis vector is <= 20 MB (at 8M+ rows the
        # four-launch kernels measured 8-13 % faster: IR 100 iterations at
        # 400^3 0.357 vs 0.403 s, 200^3 0.048 vs 0.052 s)
        if persistent == "auto":
            persistent = part.n_local * self.prec.dtype.itemsize <= 20e6
        self.persistent = bool(persistent) and m <= MEGA_MAX_K
        if self.persistent and part.world > 1:
            peer_halo = True
        self.peer = bool(peer_halo) and part.world > 1
        if self.peer:
            try:
                self._setup_peer_halo(d, group)
            except Exception as exc:  # pragma: no cover - depends on the node's IPC/P2P support
                import warnings
                warnings.warn(f"peer-memory halo unavailable ({exc}); using collective halo exchange",
                              stacklevel=2)
                self.peer = False
                d.peer_prev_V = d.peer_next_V = d.halo_flags = None
                d.peer_prev_flag = d.peer_next_flag = None
        if self.persistent:
            try:
                self._setup_xbox(d, group)
            except Exception as exc:  # pragma: no cover - depends on the node's IPC/P2P support
                import warnings
                warnings.warn(f"exchange boxes unavailable ({exc}); using the phase path", stacklevel=2)
                self.persistent = False
                d.xworld = 0
        h = C.c_void_p()
        _lib.call("mpg_solver_create", C.byref(d), C.byref(h))
        self.handle, self.desc = h, d

    def _setup_xbox(self, d, group) -> None:
        """Allocate this rank's exchange box (the persistent step's mailbox for
        the three per-step cross-rank sums) and map every rank's box into this
        process (CUDA IPC over the process group; NVLink peer memory on one
        node)."""
        part = self.part
        self.xbox = torch.zeros(int(_lib.load().mpg_xbox_bytes()), dtype=torch.uint8, device=self.V_buf.device)
        d.xworld, d.xrank = part.world, part.rank
        if part.world == 1:
            d.xbox[0] = ptr(self.xbox)
            return
        import torch.distributed as dist
        from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor
        infos = [None] * part.world
        dist.all_gather_object(infos, reduce_tensor(self.xbox)[1], group=group)
        self._xmaps = []
        for r in range(part.world):
            if r == part.rank:
                d.xbox[r] = ptr(self.xbox)
            else:
                t = rebuild_cuda_tensor(*infos[r])
                _enable_peer(t.device)
                self._xmaps.append(t)
                d.xbox[r] = t.data_ptr()

    def _setup_peer_halo(self, d, group) -> None:
        """Map the neighbours' basis buffers and halo flags into this process
        (CUDA IPC handles exchanged over the process group; on one node the
        mappings are NVLink peer memory) so the SCALE phase can store the
        boundary planes of each new basis vector straight into their halos."""
        import torch.distributed as dist
        from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor
        part, s = self.part, self.prec.dtype.itemsize
        self.halo_flags = torch.zeros(2, dtype=torch.int32, device=self.V_buf.device)
        info = {"V": reduce_tensor(self.V_buf)[1], "flags": reduce_tensor(self.halo_flags)[1],
                "ld": part.ld, "n": part.n_local, "o": part.own_offset}
        infos = [None] * part.world
        dist.all_gather_object(infos, info, group=group)
        self._peer_maps = []

        def open_peer(r):
            v = rebuild_cuda_tensor(*infos[r]["V"])
            f = rebuild_cuda_tensor(*infos[r]["flags"])
            _enable_peer(v.device)
            self._peer_maps += [v, f]
            return v.data_ptr() + infos[r]["o"] * s, f.data_ptr(), infos[r]
        d.halo_flags = ptr(self.halo_flags)
        if part.prev is not None:
            vp, fp, inf = open_peer(part.prev)
            d.peer_prev_V, d.peer_prev_ld, d.peer_prev_off = vp, inf["ld"], inf["n"]   # its upper halo
            d.peer_prev_flag = fp + 4                                                   # its flags[1]
        if part.next is not None:
            vp, fp, inf = open_peer(part.next)
            d.peer_next_V, d.peer_next_ld, d.peer_next_off = vp, inf["ld"], -part.halo  # its lower halo
            d.peer_next_flag = fp                                                       # its flags[0]

    # --- helpers
    def close(self):
        if self.handle:
            _lib.load().mpg_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def V_row(self, j: int) -> torch.Tensor:
        """Padded row j of the basis (halo | owned | halo around own_offset)."""
        ld = self.part.ld
        return self.V_buf[j * ld: j * ld + ld]

    @property
    def x_local(self) -> torch.Tensor:
        o = self.part.own_offset
        return self.x_buf[o:o + self.part.n_local]

    def _ph(self, name: str, j: int = 0, m_limit: int = 1) -> None:
        prof = getattr(self, "_prof", None)
        if prof is not None:
            with prof.scope(_PHASE_CLASS.get(name, "cycle"), j):
                _lib.call("mpg_solver_phase", self.handle, PH[name], j, max(1, m_limit), stream_handle())
            return
        _lib.call("mpg_solver_phase", self.handle, PH[name], j, max(1, m_limit), stream_handle())

    def _allreduce(self, t: torch.Tensor) -> None:
        prof = getattr(self, "_prof", None)
        if prof is not None:
            with prof.scope("allreduce", 0):
                self.coll.allreduce_(t)
            return
        self.coll.allreduce_(t)

    def _halo(self, row: torch.Tensor) -> None:
        prof = getattr(self, "_prof", None)
        if prof is not None:
            with prof.scope("halo", 0):
                self.coll.halo_(row, self.part)
            return
        self.coll.halo_(row, self.part)

    def profile_cycle(self, m_limit: int) -> dict:
        """One eager cycle with CUDA events around every phase and collective:
        {class: {"ms", "launches", "bytes"}} with this rank's algorithmic bytes
        per class (local rows)."""
        self._prof = _CycleProfile()
        try:
            self._enqueue_cycle(m_limit)
            torch.cuda.synchronize()
        finally:
            prof, self._prof = self._prof, None
        return prof.result(self.part.n_local, self.prec.dtype.itemsize)

    # --- the distributed cycle
    def begin(self) -> tuple[float, float]:
        self._ph("BNORM")
        self._allreduce(self.reserved0)
        self._ph("POST_BNORM")
        self._residual()
        hdr, _ = self.state.read()
        return float(hdr.outer_b_norm), float(hdr.rnorm)

    def _residual(self) -> None:
        self._halo(self.x_buf)
        self._ph("RESID")
        self._allreduce(self.reserved0)
        self._ph("POST_RESID")

    def cycle(self, m_limit: int):
        """One restart cycle.  With device collectives (NCCL) the whole cycle —
        phase kernels, halo exchanges and allreduces — is captured once per
        m_limit into a CUDA graph (after one eager cycle has initialised every
        kernel and communicator) and replayed, so the host issues one launch
        per cycle instead of ~16 calls per Arnoldi step."""
        if self.use_graph:
            g = self._graphs.get(m_limit)
            if g is None and self._eager_cycles.get(m_limit, 0) >= 1:
                g = self._capture(m_limit)
            if g is not None:
                g.replay()
                return self.state.read()
            self._eager_cycles[m_limit] = self._eager_cycles.get(m_limit, 0) + 1
        self._enqueue_cycle(m_limit)
        return self.state.read()

    def _capture(self, m_limit: int):
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._enqueue_cycle(m_limit)
            torch.cuda.synchronize()
        except Exception as exc:  # pragma: no cover - depends on the backend's capture support
            import warnings
            warnings.warn(f"distributed cycle capture failed ({exc}); running eagerly", stacklevel=2)
            self.use_graph = False
            torch.cuda.synchronize()
            return None
        self._graphs[m_limit] = g
        return g

    def _enqueue_cycle(self, m_limit: int) -> None:
        self._ph("START", 0, m_limit)
        self._allreduce(self.red[:2])
        self._ph("POST_START", 0, m_limit)
        self._ph("START_SCALE", 0, m_limit)
        if self.persistent:
            # one cooperative kernel per step: SpMV, CGS2, the three cross-rank
            # sums (in-kernel over the exchange boxes), Givens, scaling, and the
            # next halo planes stored into the neighbours
            self._halo(self.V_row(0))
            for j in range(m_limit):
                self._ph("STEP", j, m_limit)
            self._ph("FINISH", 0, m_limit)
            self._residual()
            return
        for j in range(m_limit):
            if j == 0 or not self.peer:      # with peer halos SCALE has already written them
                self._halo(self.V_row(j))
            self._ph("SPMV_DOT", j, m_limit)
            self._allreduce(self.red[: j + 3])
            self._ph("POST_DOT1", j, m_limit)
            self._ph("UPDATE_DOT", j, m_limit)
            self._allreduce(self.red[: j + 1])
            self._ph("POST_DOT2", j, m_limit)
            self._ph("UPDATE_NORM", j, m_limit)
            self._allreduce(self.red[:1])
            self._ph("POST_NORM", j, m_limit)
            self._ph("SCALE", j, m_limit)
        self._ph("FINISH", 0, m_limit)
        self._residual()


# phase -> profile class (DistributedStencilSolver.profile_cycle)
_PHASE_CLASS = {"SPMV_DOT": "spmv_dot", "UPDATE_DOT": "update_dot", "UPDATE_NORM": "update_norm",
                "SCALE": "scale", "POST_DOT1": "post", "POST_DOT2": "post", "POST_NORM": "post",
                "STEP": "step"}


class _CycleProfile:
    """Event pairs per (class, Arnoldi step) of one eager distributed cycle."""

    def __init__(self):
        self.ev: list = []

    @contextmanager
    def scope(self, cls: str, j: int):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            yield
        finally:
            e1.record()
            self.ev.append((cls, j, e0, e1))

    def result(self, n: int, s: int) -> dict:
        # algorithmic bytes per launch of each class at step j (k = j + 1 basis
        # vectors), this rank's rows: the constant-coefficient SpMV streams x once
        # and writes w; the pass-1 dots read V[0..k) and w
        def nbytes(cls, j):
            k = j + 1
            return {"spmv_dot": (2 + k + 1) * n * s, "update_dot": (k + 2) * n * s,
                    "update_norm": (k + 2) * n * s, "scale": 2 * n * s,
                    "step": 2 * n * s + 3 * k * n * s}.get(cls, 0)
        out: dict = {}
        for cls, j, e0, e1 in self.ev:
            ms = e0.elapsed_time(e1)
            d = out.setdefault(cls, {"ms": 0.0, "launches": 0, "bytes": 0})
            d["ms"] += ms
            d["launches"] += 1
            d["bytes"] += nbytes(cls, j)
        for d in out.values():
            d["ms"] = round(d["ms"], 4)
            if d["bytes"] and d["ms"] > 0:
                d["GBps"] = round(d["bytes"] / (d["ms"] / 1e3) / 1e9, 1)
        return out


def _dist_solve(solver: DistributedStencilSolver, criteria: StopCriteria, ir: bool,
                timer: timing.KernelTimer | None) -> SolveReport:
    """Restart bookkeeping identical to solvers.gmres_ir / _run_restarted."""
    timer = timer if timer is not None else timing.KernelTimer()
    history: list[HistoryEntry] = []
    phase = "fp32" if (ir or solver.prec is FP32) else "fp64"
    with timing.active(timer):
        b_norm, rnorm = solver.begin()
        rel = _relative(rnorm, b_norm)
        history.append(HistoryEntry(0, rel, rel, phase))
        total, converged, loss, stalled, run, prev = 0, rel <= criteria.rtol, False, None, 0, rel
        while not converged and not loss and total < criteria.max_iters:
            rho = rnorm
            hdr, imp = solver.cycle(min(criteria.m, criteria.max_iters - total))
            _raise_flags(hdr, total, ir=ir)
            implicit = [float(v) for v in imp[: hdr.steps]]
            scale = (rho / b_norm if b_norm > 0 else 1.0) if ir else None
            for i, res in enumerate(implicit[:-1]):
                val = res * scale if ir else _relative(res, b_norm)
                history.append(HistoryEntry(total + i + 1, val, None, phase))
            total += hdr.steps
            rnorm = float(hdr.rnorm)
            rel = _relative(rnorm, b_norm)
            if implicit:
                irel = implicit[-1] * scale if ir else _relative(implicit[-1], b_norm)
            else:
                irel = rel
            history.append(HistoryEntry(total, irel, rel, phase))
            converged = rel <= criteria.rtol
            if not converged and not ir and irel <= criteria.rtol and \
                    rel > LOSS_OF_ACCURACY_FACTOR * criteria.rtol:
                loss = True
            if not converged:
                run = run + 1 if (prev > 0 and (prev - rel) < STALL_IMPROVEMENT * prev) else 0
                if run >= STALL_RESTARTS and stalled is None:
                    stalled = total
                prev = rel
    fp32 = phase == "fp32"
    return SolveReport(x=solver.x_local.clone(), converged=converged, total_iters=total,
                       iters_fp32=total if fp32 else 0, iters_fp64=0 if fp32 else total,
                       residual_history=history, kernel_times=timer.breakdown(),
                       loss_of_accuracy=loss, stalled_at=stalled, total_time=timer.total)


def dist_gmres_ir(spec, part: RowPartition, collectives, criteria: StopCriteria | None = None,
                  b_local=None, *, timer=None, use_graph: bool = True, peer_halo: bool = False,
                  persistent: bool = False) -> SolveReport:
    """Row-partitioned GMRES-IR (solvers.py:297-384); x returned as this
    rank's owned block (device tensor).  persistent: one cooperative kernel
    per Arnoldi step with in-kernel cross-rank sums (MPG_PH_STEP)."""
    criteria = criteria or StopCriteria()
    s = DistributedStencilSolver(spec, part, "ir", criteria.m, criteria.rtol, collectives,
                                 b_local=b_local, use_graph=use_graph, peer_halo=peer_halo,
                                 persistent=persistent)
    try:
        return _dist_solve(s, criteria, True, timer)
    finally:
        s.close()


def dist_gmres_restarted(spec, part: RowPartition, collectives, criteria: StopCriteria | None = None,
                         precision: Precision = FP64, b_local=None, *, timer=None,
                         use_graph: bool = True, peer_halo: bool = False,
                         persistent: bool = False) -> SolveReport:
    """Row-partitioned GMRES(m) in one precision (solvers.py:251-294)."""
    criteria = criteria or StopCriteria()
    s = DistributedStencilSolver(spec, part, "restarted", criteria.m, criteria.rtol, collectives,
                                 precision=precision, b_local=b_local, use_graph=use_graph,
                                 peer_halo=peer_halo, persistent=persistent)
    try:
        return _dist_solve(s, criteria, False, timer)
    finally:
        s.close()
