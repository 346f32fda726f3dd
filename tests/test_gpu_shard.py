"""Scenario sharding on the device path: two processes (gloo)
share one GPU, each replays its shard of the global scenario ids through the
C ABI, and the per-scenario span, per-rank breakdown and per-stream busy
gathered to rank 0 must equal one process replaying the whole batch — the
property that makes results independent of the GPU count (bench.py --gpus N
gathers exactly these rows over NCCL)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPEC = dict(n_layers=96, d_model=12288, d_ffn=49152, n_heads=96, d_head=128, pp=4, dp=8,
            num_microbatches=32)
TOTAL = 5120  # 2,560 per shard: both the shards and the whole batch take the two-scenario walk


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _replay(dg, first, count):
    from paper_2504_09307_b200 import ScenarioSpec
    span = np.zeros((count, 3), np.int64)
    bd = np.zeros((count, dg.n_ranks, 5), np.int64)
    busy = np.zeros((count, dg.n_streams), np.int64)
    dg.replay_batch(ScenarioSpec(count=count, first=first, seed=250409307, jitter=0.1),
                    span=span, rank_breakdown=bd, stream_busy=busy)
    return span, bd, busy


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2504_09307_b200 import DeviceGraph
    from paper_2504_09307_b200.shard import gather_rows, shard
    from paper_2504_09307_b200.synth import SynthSpec, generate_graph
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dg = DeviceGraph(generate_graph(SynthSpec(**SPEC)).graph, device=0)
        first, count = shard(TOTAL, world, rank)
        span, bd, busy = (torch.from_numpy(a) for a in _replay(dg, first, count))
        outs = [torch.empty((TOTAL,) + tuple(a.shape[1:]), dtype=torch.int64) if rank == 0
                else None for a in (span, bd, busy)]
        for a, o in zip((span, bd, busy), outs):
            gather_rows(a, world, rank, o)
        if rank == 0:
            q.put(tuple(o.numpy() for o in outs))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_shards_equal_one_batch():
    import torch.multiprocessing as mp
    from paper_2504_09307_b200 import DeviceGraph
    from paper_2504_09307_b200.synth import SynthSpec, generate_graph
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=900)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    dg = DeviceGraph(generate_graph(SynthSpec(**SPEC)).graph, device=0)
    want = _replay(dg, 0, TOTAL)
    for name, a, b in zip(("span", "breakdown", "stream busy"), got, want):
        assert np.array_equal(a, b), name
