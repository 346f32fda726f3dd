"""GPU parity of the device-side what-if retime sweep:
per scenario, the graph apply_whatif returns for a width / data-parallel
change without a pipeline rebuild — change_hidden (transform.cpp:279-349) then
scale_dp (transform.cpp:219-258) with the analytical cost model
(cost.cpp:40-62) — replayed on the device, against the compiled reference
applying the same transforms and replaying (oracle/_ref).

Reference test strategy mirrored: test_transform.cpp's retime cases (scale_dp
rescales only the matching gradient collectives; change_hidden rescales GEMMs
by the dims ratio and collectives through the cost model) and its error
cases (dp 1 sources/targets, missing metadata).
"""
import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import Retime, ScenarioSpec, DeviceGraph, simulate_batch
from paper_2504_09307_b200.graph import ExecutionGraph, SimulationError

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("walk_ks")]


def _with_meta(h):
    g = h.export()
    g.rt_kind, g.rt_bytes, g.rt_group, g.rt_mnk = h.retime_meta()
    return g


def _check(h, g, spec, per_scenario, sc=None):
    """per_scenario(s) -> kwargs of RefGraphHandle.apply_retime for scenario s."""
    res = simulate_batch(g, spec, timestamps=True, breakdown=False)
    for s in range(spec.count):
        hr = h.apply_retime(**per_scenario(s))
        gr = hr.export()
        dur = None if sc is None else R.orc_durations(gr, sc, spec.first + s)
        rs, rf, rspan = hr.simulate(dur)
        assert np.array_equal(res.start[:, s], rs), f"scenario {s} start"
        assert np.array_equal(res.fin[:, s], rf), f"scenario {s} fin"
        assert np.array_equal(res.span[s], rspan), f"scenario {s} span"
    return res


def test_scale_dp_sweep():
    # dp 2 -> {2, 4, 8, 16} x alpha x beta: only the dp-2 gradient allreduces move
    h, _ = R.generate(R.synth_spec(pp=1, dp=2, m=4, layers=4))
    g = _with_meta(h)
    S = 24
    tdp = np.array([2, 4, 8, 16] * 6, np.int32)
    alpha = np.repeat([10.0, 3.5, 25.0], 8)
    bpu = np.tile([50000.0, 12345.6], 12)
    spec = ScenarioSpec(count=S, retime=Retime(alpha_us=alpha, bytes_per_us=bpu, source_dp=2,
                                               target_dp=tdp))
    _check(h, g, spec, lambda s: dict(src_dp=2, tgt_dp=int(tdp[s]), alpha=float(alpha[s]),
                                      bytes_per_us=float(bpu[s])))


def test_change_hidden_and_dp_with_jitter():
    # pp 2 (p2p send/recv present): width sweep, then dp, then jitter on top
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = _with_meta(h)
    assert (g.rt_kind == 4).any() and (g.rt_kind == 5).any() and (g.rt_kind == 1).any()
    S = 16
    src = (1024, 4096, 350_000_000)
    tgt = np.array([(1024, 4096, 350_000_000), (1536, 6144, 780_000_000),
                    (2048, 8192, 1_380_000_000), (1024, 8192, 600_000_000)] * 4, np.int64)
    tdp = np.array([2, 2, 4, 8] * 4, np.int32)
    alpha = np.full(S, 10.0)
    bpu = np.repeat([50000.0, 20000.0], 8)
    rt = Retime(alpha_us=alpha, bytes_per_us=bpu, source_dp=2, target_dp=tdp, source_model=src,
                target_model=tgt)
    spec = ScenarioSpec(count=S, first=5, seed=9, jitter=0.1, retime=rt)
    _check(h, g, spec, lambda s: dict(src_model=src, tgt_model=tuple(int(x) for x in tgt[s]),
                                      src_dp=2, tgt_dp=int(tdp[s]), alpha=float(alpha[s]),
                                      bytes_per_us=float(bpu[s])),
           sc=R.OrcScenarios(seed=9, jitter=0.1))


def test_retimed_durations_materialised():
    # ts_scenario_durations with a retime: the reference's transformed durations
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = _with_meta(h)
    src = (1024, 4096, 350_000_000)
    tgt = np.array([(1536, 6144, 780_000_000), (1024, 4096, 350_000_000)], np.int64)
    rt = Retime(alpha_us=[7.0, 7.0], bytes_per_us=[40000.0, 40000.0], source_dp=2,
                target_dp=[2, 8], source_model=src, target_model=tgt)
    dur = DeviceGraph(g).scenario_durations(ScenarioSpec(count=2, retime=rt))
    for s in range(2):
        gr = h.apply_retime(src_model=src, tgt_model=tuple(int(x) for x in tgt[s]), src_dp=2,
                            tgt_dp=[2, 8][s], alpha=7.0, bytes_per_us=40000.0).export()
        assert np.array_equal(dur[:, s], gr.duration)


def test_retime_errors_follow_the_reference():
    h, _ = R.generate(R.synth_spec(pp=1, dp=2, m=4, layers=4))
    g = _with_meta(h)
    one = dict(alpha_us=[10.0], bytes_per_us=[50000.0])
    cases = [
        (Retime(**one, source_dp=2, target_dp=[1]), "cannot drop gradient collectives"),
        (Retime(**one, source_dp=1, target_dp=[4]), "no gradient collectives to rescale"),
        (Retime(**one, source_dp=4, target_dp=[8]), "no gradient collectives sized for "
                                                    "data-parallel group 4"),
        (Retime(alpha_us=[10.0], bytes_per_us=[0.0], source_dp=2, target_dp=[4]),
         "bytes_per_us must be positive"),
        (Retime(**one, source_model=(1024, 4096, 0), target_model=[(2048, 8192, 0)]),
         "needs n_params on both models"),
    ]
    for rt, msg in cases:
        with pytest.raises(Exception, match=msg):
            simulate_batch(g, ScenarioSpec(count=1, retime=rt), breakdown=False)
        with pytest.raises(Exception):
            h.apply_retime(src_model=rt.source_model,
                           tgt_model=None if rt.target_model is None else rt.target_model[0],
                           src_dp=rt.source_dp,
                           tgt_dp=rt.source_dp if rt.target_dp is None else rt.target_dp[0],
                           alpha=10.0, bytes_per_us=rt.bytes_per_us[0])
    plain = h.export()  # no metadata
    with pytest.raises(Exception, match="no retime metadata"):
        simulate_batch(plain, ScenarioSpec(count=1, retime=Retime(**one, source_dp=2,
                                                                  target_dp=[4])))


# ------------------------------------------- retime walk vs materialised path
# The walk evaluates retimed durations itself (kModeRetime: K4v variant tables
# + per-scenario cost model); LUMOS_RT_FUSED=0 takes the materialised path
# (K4r writes every duration, an explicit-duration walk reads them back),
# which the tests above pin to the reference.  Both must agree on everything.

def _both_paths(monkeypatch, g, spec, **kw):
    out = []
    for fused in ("1", "0"):
        monkeypatch.setenv("LUMOS_RT_FUSED", fused)
        out.append(simulate_batch(g, spec, timestamps=True, breakdown=True, **kw))
    monkeypatch.delenv("LUMOS_RT_FUSED")
    return out


def _assert_same(a, b):
    for name in ("start", "fin", "span", "rank_breakdown", "stream_busy"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


def test_retime_walk_equals_materialised_on_replicated_graph(monkeypatch):
    # TP and DP replicas share one program: the walk reads the creator
    # component's metadata; many width variants, dp targets, cost models,
    # class scale and jitter at once
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4), tp=2)
    g = _with_meta(h)
    S = 200
    rng = np.random.default_rng(5)
    src = (1024, 4096, 350_000_000)
    widths = np.array([(1024, 4096, 350_000_000), (1536, 6144, 780_000_000),
                       (2048, 8192, 1_380_000_000), (1024, 8192, 600_000_000),
                       (768, 3072, 200_000_000), (1024, 4096, 999)], np.int64)
    tgt = widths[rng.integers(0, len(widths), S)]
    tdp = rng.choice([2, 4, 8, 16], S).astype(np.int32)
    alpha = rng.uniform(1.0, 40.0, S)
    bpu = rng.uniform(5e3, 9e4, S)
    rt = Retime(alpha_us=alpha, bytes_per_us=bpu, source_dp=2, target_dp=tdp, source_model=src,
                target_model=tgt)
    spec = ScenarioSpec(count=S, first=11, seed=3, jitter=0.07, scale_lo=900, scale_hi=1100,
                        scale_den=1024, retime=rt)
    a, b = _both_paths(monkeypatch, g, spec)
    _assert_same(a, b)
    # the first scenarios (no class scale: the reference has no such
    # transform) against the reference transforms
    res = _check(h, g, ScenarioSpec(count=8, first=11, seed=3, jitter=0.07,
                                    retime=Retime(alpha_us=alpha[:8], bytes_per_us=bpu[:8],
                                                  source_dp=2, target_dp=tdp[:8],
                                                  source_model=src, target_model=tgt[:8])),
                 lambda s: dict(src_model=src, tgt_model=tuple(int(x) for x in tgt[s]), src_dp=2,
                                tgt_dp=int(tdp[s]), alpha=float(alpha[s]),
                                bytes_per_us=float(bpu[s])),
                 sc=R.OrcScenarios(seed=3, jitter=0.07))
    assert res.span.shape == (8, 3)


def test_retime_walk_fixup_retimes_its_durations(monkeypatch):
    # a certificate failure sends the scenario to the event-driven kernel,
    # which must apply the same retime (GEMM kernels rescaled by the widths)
    from test_gpu_parity import _graph
    g = _graph([(1, 7, 0, 100), (1, 7, 10, 10), (0, 1, 0, 2), (0, 1, 5, 4), (0, 1, 20, 5)],
               edges=[(0, 1), (2, 3), (3, 4)], rules=[(0, 3, -1, [(0, 1, 7)])])
    g.rt_kind = np.array([1, 1, 0, 0, 0], np.uint8)
    g.rt_bytes = np.zeros(5, np.int64)
    g.rt_group = np.zeros(5, np.int32)
    g.rt_mnk = np.array([[64, 1024, 4096], [64, 4096, 1024], [0] * 3, [0] * 3, [0] * 3], np.int64)
    src = (1024, 4096, 1000)
    tgt = np.array([(1024, 4096, 1000), (2048, 8192, 4000), (512, 4096, 700)], np.int64)
    rt = Retime(alpha_us=[5.0] * 3, bytes_per_us=[1e4] * 3, source_model=src, target_model=tgt)
    spec = ScenarioSpec(count=3, retime=rt)
    a, b = _both_paths(monkeypatch, g, spec)
    _assert_same(a, b)
    assert a.span[1, 2] > a.span[0, 2] > a.span[2, 2]
    status = np.zeros(3, np.int32)
    start = np.zeros((g.n, 3), np.int64)
    fin = np.zeros((g.n, 3), np.int64)
    DeviceGraph(g).replay_batch(spec, start=start, fin=fin, status=status)
    assert (status == 1).all()  # every scenario went through the fix-up
    assert np.array_equal(start, a.start) and np.array_equal(fin, a.fin)


def test_allreduce_without_bytes_is_left_alone(tmp_path):
    # change_hidden retimes an allreduce only when it carries a byte count
    # (transform.cpp:313): drop "bytes" from one gradient allreduce in the
    # recorded trace; a width sweep must leave it as recorded (no n_params /
    # group-size errors for it either), and a dp change must raise the
    # reference's "carries no byte count" (transform.cpp:238-240)
    import json
    import os
    R.write_rank_traces(R.synth_spec(pp=1, dp=2, m=4, layers=4), str(tmp_path))
    path = os.path.join(tmp_path, "rank_0.json")
    with open(path) as f:
        tr = json.load(f)
    evs = tr["traceEvents"] if isinstance(tr, dict) else tr
    hit = [e for e in evs if e.get("cat") == "kernel" and
           e.get("args", {}).get("collective") == "allreduce" and "bytes" in e.get("args", {})]
    assert hit
    del hit[0]["args"]["bytes"]
    with open(path, "w") as f:
        json.dump(tr, f)
    h = R.ingest_traces([path])
    g = _with_meta(h)
    ar = np.flatnonzero(g.rt_kind == 3)
    assert len(ar) and (g.rt_bytes[ar] < 0).any()
    src = (1024, 4096, 350_000_000)
    tgt = np.array([(1536, 6144, 780_000_000), (2048, 8192, 1_380_000_000)] * 2, np.int64)
    rt = Retime(alpha_us=[10.0] * 4, bytes_per_us=[30000.0] * 4, source_model=src,
                target_model=tgt)
    spec = ScenarioSpec(count=4, first=2, seed=3, jitter=0.05, retime=rt)
    _check(h, g, spec, lambda s: dict(src_model=src, tgt_model=tuple(int(x) for x in tgt[s]),
                                      alpha=10.0, bytes_per_us=30000.0),
           sc=R.OrcScenarios(seed=3, jitter=0.05))
    with pytest.raises(Exception, match="carries no byte count"):
        simulate_batch(g, ScenarioSpec(count=1, retime=Retime(alpha_us=[10.0],
                                                              bytes_per_us=[30000.0],
                                                              source_dp=2, target_dp=[4])),
                       breakdown=False)
