"""N > 1 host logic on CPU with torch.distributed (gloo, world size 2):

* bench.slab: the per-rank slabs of the domain are an exact cover;
* bench.transfer_fn: the rebalancing transfer moves bytes from the donor's
  buffer to the receiver's only (include/ibnb.h ib_transfer_fn contract);
* bench.exchange_fn: the per-chunk exchange of [GUB, finished flag]
  is an element-wise MIN over ranks (include/ibnb.h ib_exchange_fn contract):
  GUB = the best sample of any rank, "all finished" only when every rank is;
* partitioned search: every rank solves its slab (CPU oracle) and the
  all-reduced enclosure [min GLB, min GUB] contains the known minimum and
  matches the single-domain enclosure."""
from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        ex = bench.exchange_fn(dist)
        # rebalancing transfer: rank 1 sends the first 24 bytes of its buffer to rank 0
        tr = bench.transfer_fn(dist, rank)
        buf = torch.arange(8, dtype=torch.uint8) + (100 if rank == 1 else 0)
        tr(1, 0, buf, 3)
        out["buf"] = buf.tolist()
        # exchange: rank 0 has the better incumbent and is finished, rank 1 not
        x = torch.tensor([1.5, 0.0] if rank == 0 else [2.5, -1.0], dtype=torch.float64)
        ex(x)
        out["x1"] = x.tolist()
        x = torch.tensor([3.0, 0.0] if rank == 0 else [2.0, 0.0], dtype=torch.float64)
        ex(x)
        out["x2"] = x.tolist()
        # partitioned oracle solve of configs[0] over 2 slabs
        cfg = workloads.CONFIGS[0]
        L, U = workloads.config_bounds(cfg)
        l, u = bench.slab(L, U, rank, world)
        r = oracle.solve(cfg["fid"], l, u, eps_f=cfg["eps"], eps_x=cfg["eps"], d=2, m=2, bmax=4096)
        enc = torch.tensor([r["glb"], r["gub"]], dtype=torch.float64)
        dist.all_reduce(enc, op=dist.ReduceOp.MIN)
        out["enc"] = enc.tolist()
        out["status"] = r["status"]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_slab_partition_is_an_exact_cover():
    L, U = np.full(3, -5.12), np.full(3, 5.12)
    for world in (1, 2, 3, 8):
        slabs = [bench.slab(L, U, r, world) for r in range(world)]
        assert slabs[0][0][0] == L[0] and slabs[-1][1][0] == U[0]
        for a, b in zip(slabs, slabs[1:]):
            assert a[1][0] == b[0][0]  # shared face, no gap
        for lo, hi in slabs:
            assert np.all(lo[1:] == L[1:]) and np.all(hi[1:] == U[1:]) and lo[0] < hi[0]


def test_two_rank_exchange_and_partitioned_enclosure():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # rebalancing transfer: rank 0 received rank 1's first 3 bytes, rank 1 unchanged
    assert res[0]["buf"] == [100, 101, 102, 3, 4, 5, 6, 7]
    assert res[1]["buf"] == [100, 101, 102, 103, 104, 105, 106, 107]
    for r in (0, 1):
        # min GUB over ranks; not everybody finished (-1) in round 1
        assert res[r]["x1"] == [1.5, -1.0]
        # everybody finished in round 2
        assert res[r]["x2"] == [2.0, 0.0]
    glb, gub = res[0]["enc"]
    assert res[1]["enc"] == [glb, gub]
    assert glb <= 0.0 <= gub and gub - glb <= 1e-6
    cfg = workloads.CONFIGS[0]
    whole = oracle.solve(cfg["fid"], *workloads.config_bounds(cfg), eps_f=cfg["eps"], eps_x=cfg["eps"], d=2, m=2)
    assert math.isclose(glb, whole["glb"], abs_tol=1e-12)
