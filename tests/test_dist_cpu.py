"""Multi-process (gloo, world size 2 and 3, CPU) tests of the row-partitioned
path's host side: plane partition, the padded halo layout and its exchange,
and the sum-allreduce the distributed kernels rely on."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu_gmres as O
from paper_2109_01232_b200.dist import (Collectives, HostStagedCollectives, RowPartition,
                                        plane_partition)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plane_partition_matches_oracle_rows():
    for dims, nx, world in ((3, 400, 8), (3, 150, 3), (2, 1500, 8), (3, 5, 5), (2, 7, 2)):
        plane = nx ** (dims - 1)
        parts = [RowPartition.for_stencil(dims, nx, world, r) for r in range(world)]
        assert parts[0].row0 == 0 and parts[-1].row1 == nx ** dims
        assert all(a.row1 == b.row0 for a, b in zip(parts, parts[1:]))
        assert all(p.row0 % plane == 0 and p.halo == plane for p in parts)
        # plane blocks are the oracle's contiguous partition of the planes
        assert [(p.row0 // plane, p.row1 // plane) for p in parts] == O.row_partition(nx, world)
        for p in parts:
            assert p.own_offset >= p.halo and p.own_offset % 64 == 0
            assert p.ld % 64 == 0 and p.ld >= p.own_offset + p.n_local + p.halo
    with pytest.raises(ValueError):
        plane_partition(3, 4)


def _worker(rank, world, port, staged, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coll = HostStagedCollectives() if staged else Collectives()
        res = {}
        for dims, nx in ((3, 6), (2, 9)):
            part = RowPartition.for_stencil(dims, nx, world, rank)
            row = torch.full((part.ld,), -1.0, dtype=torch.float64)
            o, n, h = part.own_offset, part.n_local, part.halo
            row[o:o + n] = torch.arange(part.row0, part.row1, dtype=torch.float64)
            coll.halo_(row, part)
            lo = row[o - h:o].numpy().copy()
            hi = row[o + n:o + n + h].numpy().copy()
            ok_lo = np.array_equal(lo, np.arange(part.row0 - h, part.row0)) if part.prev is not None \
                else np.all(lo == -1.0)
            ok_hi = np.array_equal(hi, np.arange(part.row1, part.row1 + h)) if part.next is not None \
                else np.all(hi == -1.0)
            # owned block untouched
            ok_own = np.array_equal(row[o:o + n].numpy(), np.arange(part.row0, part.row1))
            res[(dims, nx)] = bool(ok_lo and ok_hi and ok_own)
        t = torch.tensor([float(rank + 1), 2.0 ** -30 * (rank + 1)], dtype=torch.float32)
        coll.allreduce_(t)
        res["allreduce"] = t.tolist()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,staged", [(2, False), (2, True), (3, False)])
def test_halo_exchange_and_allreduce_gloo(world, staged):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, staged, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = float(sum(range(1, world + 1)))
    for r in range(world):
        res = results[r]
        assert res[(3, 6)] and res[(2, 9)], (r, res)
        assert res["allreduce"][0] == want
        # every rank receives the identical reduced bits
        assert res["allreduce"] == results[0]["allreduce"]
