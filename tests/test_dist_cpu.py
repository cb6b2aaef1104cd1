"""World-size-2 gloo tests of the multi-GPU plumbing (dist.py) on CPU: partitions, the
sample->node transpose into slabs, and the MAX / SUM reductions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_04131_b200.dist import TorchExchange, bounds, partition


def test_partition_covers_and_balances():
    for n in (0, 1, 7, 961, 6817):
        for P in (1, 2, 3, 8):
            b = bounds(n, P)
            assert b[0] == 0 and b[-1] == n and all(b[p] <= b[p + 1] for p in range(P))
            sizes = [b[p + 1] - b[p] for p in range(P)]
            assert max(sizes) - min(sizes) <= 1
            assert [partition(n, P, p) for p in range(P)] == [(b[p], b[p + 1]) for p in range(P)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, G, Btot, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = TorchExchange()
        full = torch.arange(G * Btot, dtype=torch.float64).reshape(G, Btot)
        b0, b1 = partition(Btot, world, rank)
        u_local = full[:, b0:b1].contiguous()
        slabs, sb = ex.transpose(u_local, G, Btot)
        g0, g1 = partition(G, world, rank)
        gl = g1 - g0
        # rebuild node rows from the slab layout exactly as the FFT kernel addresses it
        rows = torch.empty((gl, Btot), dtype=torch.float64)
        for p in range(world):
            w = sb[p + 1] - sb[p]
            blk = slabs[gl * sb[p]: gl * sb[p] + gl * w].reshape(gl, w)
            rows[:, sb[p]:sb[p + 1]] = blk
        ok_t = torch.equal(rows, full[g0:g1])
        km = torch.tensor([float(rank + 1) * 0.5])
        ex.max_(km)
        v = torch.arange(10, dtype=torch.int32) * (rank + 1)
        ex.sum_(v)
        out[rank] = (bool(ok_t), float(km.item()), v.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,Btot", [(7, 13), (961, 401 * 3)])
def test_gloo_world2_exchange(G, Btot):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), G, Btot, out), nprocs=world, join=True)
    for r in range(world):
        ok, km, v = out[r]
        assert ok
        assert km == 1.0
        assert v == [3 * i for i in range(10)]


def _boot_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_04131_b200.dist import bootstrap_id
        out[rank] = bootstrap_id()
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_id_identical():
    """C0: rank 0's 128-byte communicator id (made by libusfft) reaches every rank unchanged."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_boot_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert len(out[0]) == 128 and out[0] == out[1]
