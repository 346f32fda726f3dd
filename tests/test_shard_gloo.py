"""Multi-process (world size 2, gloo, CPU) test of the scenario sharding and
the final per-scenario gather used by bench.py for N > 1."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_09307_b200.shard import gather_rows, shard


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard(total, world, rank)
    ids = torch.arange(first, first + count, dtype=torch.int64)
    # stand-ins for per-scenario results: functions of the global id only
    span = torch.stack([ids * 3, ids * 3 + 1, ids % 7], dim=1)
    bd = (ids[:, None, None] * 10 + torch.arange(5)[None, None, :]).repeat(1, 4, 1)
    out_span = torch.empty((total, 3), dtype=torch.int64) if rank == 0 else None
    out_bd = torch.empty((total, 4, 5), dtype=torch.int64) if rank == 0 else None
    gather_rows(span, world, rank, out_span)
    gather_rows(bd, world, rank, out_bd)
    if rank == 0:
        q.put((out_span.tolist(), out_bd.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges():
    assert shard(65536, 8, 3) == (24576, 8192)
    assert shard(1024, 1, 0) == (0, 1024)
    with pytest.raises(ValueError):
        shard(10, 3, 0)


def test_gather_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    total, world = 64, 2
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    span, bd = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ids = torch.arange(total)
    assert span == torch.stack([ids * 3, ids * 3 + 1, ids % 7], dim=1).tolist()
    assert bd == (ids[:, None, None] * 10 + torch.arange(5)[None, None, :]).repeat(1, 4, 1).tolist()
