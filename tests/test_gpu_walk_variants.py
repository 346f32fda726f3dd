"""The benchmarked K1 walk variant under parity.

Every benchmark launch replays two scenarios per thread (kS = 2: one
Philox2x32-10 call per task serves the thread's scenario pair, 16-byte output
stores, the shared-memory class-scale table).  The walk picks that variant on
its own once a launch has >= 148 * 8 * 32 (component, scenario-pair) units, so
the tests here use batches large enough to take it *naturally* (no
LUMOS_WALK_KS override) and check the launch counters (ts_walk_counts) to
prove it ran.  Sampled columns — first, last, an odd count's duplicated last
column — are compared bit for bit with the compiled reference simulate()
(simulate.cpp:341-347) and breakdown_by_rank (metrics.cpp:96-103).
"""
import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import DeviceGraph, ScenarioSpec
from paper_2504_09307_b200 import _native as N

pytestmark = pytest.mark.gpu

SPEC_175B_PP4_DP8 = dict(pp=4, dp=8, m=32, layers=96, d_model=12288, d_ffn=49152, heads=96)


@pytest.fixture(scope="module")
def config4_tp1():
    # 175B pp4 dp8 m32, generator-native (tp = 1): 309,536 tasks in 32 rank
    # components, so 2,368+ scenarios fill the machine with scenario pairs
    h, truth = R.generate(R.synth_spec(**SPEC_175B_PP4_DP8))
    assert truth == 2183270773
    return h, h.export()


def _run_sampled(h, g, spec, sc, cols, monkeypatch, expect_pairs=True):
    import torch
    monkeypatch.delenv("LUMOS_WALK_KS", raising=False)
    dg = DeviceGraph(g, device=0)
    dev = torch.device("cuda", 0)
    S = spec.count
    ld = S + (S & 1)  # even leading dimension; an odd count still disables 16-byte stores
    start = torch.empty((dg.n_tasks, ld), dtype=torch.int64, device=dev)
    fin = torch.empty((dg.n_tasks, ld), dtype=torch.int64, device=dev)
    span = torch.empty((S, 3), dtype=torch.int64, device=dev)
    bd = torch.empty((S, dg.n_ranks, 5), dtype=torch.int64, device=dev)
    before = N.walk_counts()
    dg.replay_batch(spec, start=start, fin=fin, ld=ld, span=span, rank_breakdown=bd,
                    stream=torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize()
    after = N.walk_counts()
    d = [a - b for a, b in zip(after, before)]
    if expect_pairs:
        assert d[2] + d[3] >= 1 and d[0] + d[1] == 0, d  # the two-scenario walk ran
    span_h = span.cpu().numpy()
    bd_h = bd.cpu().numpy()
    for c in cols:
        s_col = start[:, c].cpu().numpy()
        f_col = fin[:, c].cpu().numpy()
        dur = R.orc_durations(g, sc, spec.first + c)
        rs, rf, rspan = h.simulate(dur)
        assert np.array_equal(s_col, rs), f"column {c} start"
        assert np.array_equal(f_col, rf), f"column {c} fin"
        assert np.array_equal(span_h[c], rspan), f"column {c} span"
        wend = max(g.window_end, g.window_start + int(rspan[2]))
        ref = h.breakdown_by_rank(rs, rf, g.window_start, wend)
        for i, r in enumerate(sorted(ref)):
            assert tuple(bd_h[c, i]) == ref[r], f"column {c} rank {r}"
    return d


def test_natural_pairs_jitter(config4_tp1, monkeypatch):
    # config-5 scenario law (jitter 0.1) on the natural two-scenario walk,
    # 16-byte stores, columns at both ends of the batch
    h, g = config4_tp1
    spec = ScenarioSpec(count=2560, first=0, seed=250409307, jitter=0.1)
    _run_sampled(h, g, spec, R.OrcScenarios(seed=250409307, jitter=0.1), [0, 1, 1277, 2558, 2559],
                 monkeypatch)


def test_natural_pairs_class_scale(config4_tp1, monkeypatch):
    # config-4 scenario law (per-class factors 768..1536 / 1024): the
    # shared-memory numerator table exists only in the two-scenario walk
    h, g = config4_tp1
    kw = dict(scale_lo=768, scale_hi=1536, scale_den=1024)
    spec = ScenarioSpec(count=2560, first=63488, seed=250409307, **kw)
    _run_sampled(h, g, spec, R.OrcScenarios(seed=250409307, **kw), [0, 513, 2559], monkeypatch)


def test_natural_pairs_odd_count_scale_and_jitter(config4_tp1, monkeypatch):
    # odd count: the last thread duplicates its column (no 16-byte stores),
    # jitter on top of a non-power-of-two class denominator
    h, g = config4_tp1
    kw = dict(jitter=0.05, scale_lo=900, scale_hi=1100, scale_den=1000)
    spec = ScenarioSpec(count=2561, first=4096, seed=99, **kw)
    _run_sampled(h, g, spec, R.OrcScenarios(seed=99, **kw), [0, 2559, 2560], monkeypatch)


def test_forced_variant_counters(monkeypatch):
    # LUMOS_WALK_KS pins the variant; an odd first id always takes one
    # scenario per thread (Philox pairs never straddle threads)
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    dg = DeviceGraph(g, device=0)
    span = np.zeros((64, 3), np.int64)
    for ks, first, want in [("2", 10, 2), ("1", 10, 0), ("2", 11, 0)]:
        monkeypatch.setenv("LUMOS_WALK_KS", ks)
        before = N.walk_counts()
        dg.replay_batch(ScenarioSpec(count=64, first=first, jitter=0.1), span=span)
        d = [a - b for a, b in zip(N.walk_counts(), before)]
        assert d[want] + d[want + 1] == 1 and sum(d) == 1, (ks, first, d)
