"""ts_result.host_async: host outputs filled by copies on the graph's copy
stream, overlapping the next call's kernels (two staging sets) — every call's
span / breakdown / stream busy must equal a synchronous call's, across more
calls than there are staging sets and with device timestamps in between."""
import numpy as np
import pytest
import torch

from paper_2504_09307_b200 import DeviceGraph, ScenarioSpec
from paper_2504_09307_b200.synth import SynthSpec, generate_graph

pytestmark = pytest.mark.gpu


def test_host_async_outputs_equal_synchronous_outputs():
    g = generate_graph(SynthSpec(pp=2, dp=2, num_microbatches=4, tp=2)).graph
    dg = DeviceGraph(g, device=0)
    tile, calls = 96, 5
    dev = torch.device("cuda", 0)
    start = torch.empty((dg.n_tasks, tile), dtype=torch.int64, device=dev)
    fin = torch.empty_like(start)
    shapes = ((tile, 3), (tile, dg.n_ranks, 5), (tile, dg.n_streams))
    got = [[torch.empty(s, dtype=torch.int64).pin_memory() for s in shapes] for _ in range(calls)]
    for k in range(calls):
        spec = ScenarioSpec(count=tile, first=k * tile, seed=9, jitter=0.2)
        dg.replay_batch(spec, start=start, fin=fin, ld=tile, span=got[k][0],
                        rank_breakdown=got[k][1], stream_busy=got[k][2], host_async=True)
    dg.wait()
    for k in range(calls):
        want = [np.zeros(s, np.int64) for s in shapes]
        spec = ScenarioSpec(count=tile, first=k * tile, seed=9, jitter=0.2)
        dg.replay_batch(spec, start=start, fin=fin, ld=tile, span=want[0],
                        rank_breakdown=want[1], stream_busy=want[2])
        for a, b in zip(got[k], want):
            assert np.array_equal(a.numpy(), b), f"call {k}"


def test_host_async_falls_back_to_synchronous_when_status_is_read(monkeypatch):
    # an event-driven graph reads its scenario status back (deadlock check):
    # host_async then stays synchronous, results unchanged
    monkeypatch.setenv("LUMOS_FORCE_DES", "1")
    g = generate_graph(SynthSpec(pp=2, dp=1, num_microbatches=2, n_layers=2)).graph
    dg = DeviceGraph(g, device=0)
    assert dg.info["des_only"] == 1
    spec = ScenarioSpec(count=16, seed=4, jitter=0.1)
    a = np.zeros((16, 3), np.int64)
    b = np.zeros((16, 3), np.int64)
    dg.replay_batch(spec, span=a, host_async=True)
    dg.wait()
    dg.replay_batch(spec, span=b)
    assert np.array_equal(a, b) and (a[:, 2] > 0).all()
