"""GPU parity of the estimate (generator-semantics) mode: the batched replay of
generate_graph(estimate=True) with scenario durations must reproduce the
reference's build_pipeline(spec, DurationHook) (pipeline.cpp:361-477) event
times bit-for-bit — p2p rendezvous and collective barriers included."""
import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import ScenarioSpec, simulate_batch
from paper_2504_09307_b200.synth import generate_graph
from test_synth_graph import FIELDS, _my_lane_sequences, _ref_pipeline, _spec

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("walk_ks")]


def _orc_graph(g):
    return R.Graph(**{k: getattr(g, k) for k in FIELDS}, window_start=g.window_start,
                   window_end=g.window_end)


def _check(shape, S, seed, jitter, every=1, tp=1):
    pp, dp, m, layers, d, f = shape
    sg = generate_graph(_spec(pp, dp, m, layers, d, f, tp=tp, estimate=True))
    g = sg.graph
    spec = ScenarioSpec(count=S, seed=seed, jitter=jitter)
    res = simulate_batch(g, spec, breakdown=False)
    og = _orc_graph(g)
    sc = R.OrcScenarios(seed=seed, jitter=jitter)
    spec_json = R.synth_spec(pp=pp, dp=dp, m=m, layers=layers, d_model=d, d_ffn=f)
    for s in range(0, S, every):
        dur = R.orc_durations(og, sc, s)
        for t in range(tp):
            sel = np.where(g.rank % tp == t)[0]
            hook = np.zeros(sg.n_ops, np.int64)
            hook[sg.op_index[sel]] = dur[sel]
            ref, _ = _ref_pipeline(spec_json, hook)
            sub = R.Graph(**{k: (getattr(g, k)[sel] if k in ("duration", "original_start",
                                                              "rank", "lane_kind", "lane",
                                                              "op_class", "task_kind")
                                 else getattr(g, k)) for k in FIELDS},
                          window_start=g.window_start, window_end=g.window_end)
            sub.rank = sub.rank // tp
            got = _my_lane_sequences(sub, res.start[sel, s], res.fin[sel, s])
            assert got == ref, f"scenario {s} replica {t}"
    return res


@pytest.mark.parametrize("shape", [(2, 2, 4, 4, 1024, 4096), (1, 2, 4, 4, 1024, 4096),
                                   (4, 2, 8, 4, 1024, 4096), (2, 4, 4, 4, 1024, 4096),
                                   (8, 1, 8, 8, 1024, 4096)])
def test_estimate_batch_matches_build_pipeline(shape):
    _check(shape, S=40, seed=21, jitter=0.3)


def test_estimate_config3_44b_tp4_sampled():
    # BASELINE config 3: 44B (48 L, d 12288, f 24576) pp4 dp4 m16 x TP4 replicas
    res = _check((4, 4, 16, 48, 12288, 24576), S=6, seed=250409307, jitter=0.1, tp=4)
    assert res.span.shape == (6, 3)


def test_estimate_nominal_equals_generator_truth():
    sg = generate_graph(_spec(4, 2, 8, 4, estimate=True))
    res = simulate_batch(sg.graph, ScenarioSpec(count=2), breakdown=False)
    assert (res.makespan == sg.truth_makespan).all()


def test_estimate_cooperative_and_single_walks_agree(monkeypatch):
    # components coupling several ranks walk cooperatively (one warp per rank,
    # cross-rank values through shared-memory mailboxes); LUMOS_COOP=0 compiles
    # them as one program instead — both must equal build_pipeline
    monkeypatch.setenv("LUMOS_COOP", "0")
    _check((2, 2, 4, 4, 1024, 4096), S=16, seed=5, jitter=0.2)
    monkeypatch.setenv("LUMOS_COOP", "1")
    _check((2, 2, 4, 4, 1024, 4096), S=16, seed=5, jitter=0.2)


def test_estimate_uint32_window_wrap_fixup(monkeypatch):
    # a cooperative walk forced onto uint32 offsets for a timeline longer than
    # 2^32 us (class scale x 30000): every wrapped addition must be caught and
    # the chunk re-run in int64, still matching build_pipeline
    monkeypatch.setenv("LUMOS_COOP_FORCE_U32", "1")
    pp, dp, m, layers, d, f = (2, 2, 4, 4, 1024, 4096)
    sg = generate_graph(_spec(pp, dp, m, layers, d, f, estimate=True))
    g = sg.graph
    S = 8
    spec = ScenarioSpec(count=S, seed=3, jitter=0.1, scale_lo=30000, scale_hi=30000, scale_den=1)
    res = simulate_batch(g, spec, breakdown=False)
    assert int(res.makespan.max()) > 2 ** 32
    og = _orc_graph(g)
    sc = R.OrcScenarios(seed=3, jitter=0.1, scale_lo=30000, scale_hi=30000, scale_den=1)
    spec_json = R.synth_spec(pp=pp, dp=dp, m=m, layers=layers, d_model=d, d_ffn=f)
    for s in range(S):
        dur = R.orc_durations(og, sc, s)
        hook = np.zeros(sg.n_ops, np.int64)
        hook[sg.op_index] = dur
        ref, _ = _ref_pipeline(spec_json, hook)
        assert _my_lane_sequences(og, res.start[:, s], res.fin[:, s]) == ref, f"scenario {s}"


@pytest.mark.parametrize("pp,dp,m,tp", [(3, 2, 5, 1), (2, 3, 7, 2), (4, 2, 9, 1)])
def test_estimate_batch_from_pipeline_spec(pp, dp, m, tp):
    # Mode-B boundary: a hand-edited reference PipelineSpec (non-generator
    # kernels, odd microbatch counts, moved streams / costs) replayed by
    # estimate_batch must equal build_pipeline(spec, hook) per scenario, hook
    # slot op_index[t] carrying the oracle's duration of task t
    from paper_2504_09307_b200 import estimate_batch
    from test_pipeline_spec import hand_edited
    sp = hand_edited(pp, dp, m)
    spec = ScenarioSpec(count=24, first=6, seed=77, jitter=0.2)
    res, sg = estimate_batch(sp, spec, tp=tp)
    _check_spec_batch(sp, spec, res, sg, tp)


@pytest.mark.parametrize("tp", [1, 2])
def test_estimate_whatif_matches_build_pipeline(tp):
    # estimate() for a structural what-if: rebuild_pipeline measures the
    # source (pp2 dp2 m8, 4 layers) and lays out pp4 dp4 m8 with 8 layers;
    # the batched replay of the rebuilt spec's estimate graph equals
    # build_pipeline(rebuilt spec, hook) scenario by scenario
    from paper_2504_09307_b200 import (ModelConfig, ParallelismConfig, WhatIfConfig,
                                       estimate_whatif)
    src = _spec(2, 2, 8, 4, 1024, 4096)
    w = WhatIfConfig(ModelConfig(4, 1024, 4096, 16, 64), ModelConfig(8, 1024, 4096, 16, 64),
                     ParallelismConfig(1, 2, 2, 8), ParallelismConfig(1, 4, 4, 8))
    spec = ScenarioSpec(count=20, first=3, seed=41, jitter=0.25)
    res, sg, sp = estimate_whatif(src, w, spec, tp=tp)
    assert sp.pp == 4 and sp.dp == 4 and len(sp.stages[0].layers_fwd) == 2
    _check_spec_batch(sp, spec, res, sg, tp)


def _check_spec_batch(sp, spec, res, sg, tp):
    from test_synth_graph import _lane_sequences
    S = spec.count
    g = sg.graph
    og = _orc_graph(g)
    sc = R.OrcScenarios(seed=spec.seed, jitter=spec.jitter)
    js = sp.to_json()
    for s in range(0, S, 5):
        dur = R.orc_durations(og, sc, spec.first + s)
        for t in range(tp):
            sel = np.where(g.rank % tp == t)[0]
            hook = np.zeros(sg.n_ops, np.int64)
            hook[sg.op_index[sel]] = dur[sel]
            pid, tid, ts, du, _, end = R.pipeline_events_json(js, hook)
            sub = R.Graph(**{k: (getattr(g, k)[sel] if k in ("duration", "original_start",
                                                              "rank", "lane_kind", "lane",
                                                              "op_class", "task_kind")
                                 else getattr(g, k)) for k in FIELDS},
                          window_start=g.window_start, window_end=g.window_end)
            sub.rank = sub.rank // tp
            got = _my_lane_sequences(sub, res.start[sel, s], res.fin[sel, s])
            assert got == _lane_sequences(pid, tid, ts, du), f"scenario {s} replica {t}"


@pytest.mark.parametrize("force_u32", ["0", "1"])
def test_estimate_split_accounting(force_u32, monkeypatch):
    # cooperative walks sum |A| per warp (= rank); the split accounting's
    # breakdown and stream busy equal the full sweep (LUMOS_FUSED_REDUCE=0) and
    # the C restatement of breakdown_by_rank on the same timestamps — also
    # after the uint32-wrap int64 re-run (force_u32 with a > 2^32 us timeline)
    monkeypatch.setenv("LUMOS_COOP_FORCE_U32", force_u32)
    sg = generate_graph(_spec(4, 2, 8, 4, estimate=True))
    g = sg.graph
    kw = (dict(jitter=0.1, scale_lo=30000, scale_hi=30000, scale_den=1) if force_u32 == "1"
          else dict(jitter=0.25))
    spec = ScenarioSpec(count=48, first=4, seed=12, **kw)
    out = {}
    for env in ("1", "0"):
        monkeypatch.setenv("LUMOS_FUSED_REDUCE", env)
        from paper_2504_09307_b200 import DeviceGraph
        dg = DeviceGraph(g)
        assert (dg.info["n_fused_ranks"] == dg.n_ranks) == (env == "1")
        out[env] = simulate_batch(dg, spec, timestamps=True, breakdown=True)
    a, b = out["1"], out["0"]
    if force_u32 == "1":
        assert int(a.makespan.max()) > 2 ** 32
    assert np.array_equal(a.rank_breakdown, b.rank_breakdown)
    assert np.array_equal(a.stream_busy, b.stream_busy)
    og = _orc_graph(g)
    ranks = sorted(set(int(r) for r in g.rank))
    for s in (0, 23, 47):
        wend = max(g.window_end, g.window_start + int(a.span[s, 2]))
        st = np.ascontiguousarray(a.start[:, s])
        fi = np.ascontiguousarray(a.fin[:, s])
        for i, r in enumerate(ranks):
            want = R.orc_breakdown_rank(og, st, fi, r, g.window_start, wend)
            assert tuple(a.rank_breakdown[s, i]) == want, (s, r)


@pytest.mark.parametrize("shape", [(4, 2, 8, 4, 1024, 4096), (2, 4, 4, 4, 1024, 4096)])
def test_cluster_walk_equals_cooperative_walk(shape, monkeypatch):
    # K1x (one CTA per rank program in a thread-block cluster, two scenarios
    # per thread, L2 mailboxes) and the cooperative walk (LUMOS_CLUSTER=0)
    # give identical timestamps, spans and breakdowns; both equal
    # build_pipeline per scenario (_check); the launch counters prove which ran
    from paper_2504_09307_b200 import DeviceGraph
    from paper_2504_09307_b200 import _native as N
    pp, dp, m, layers, d, f = shape
    sg = generate_graph(_spec(pp, dp, m, layers, d, f, estimate=True))
    spec = ScenarioSpec(count=600, first=8, seed=17, jitter=0.2)
    # an odd first id keeps the cooperative walk (scenario pairs share Philox)
    before = N.walk_counts()
    simulate_batch(sg.graph, ScenarioSpec(count=64, first=9, seed=17, jitter=0.2))
    assert N.walk_counts()[4] == before[4]
    out = {}
    for env in ("1", "0"):
        monkeypatch.setenv("LUMOS_CLUSTER", env)
        before = N.walk_counts()
        out[env] = simulate_batch(DeviceGraph(sg.graph), spec, timestamps=True, breakdown=True)
        ran = N.walk_counts()[4] - before[4]
        assert (ran > 0) == (env == "1"), ran
    for k in ("start", "fin", "span", "rank_breakdown", "stream_busy"):
        assert np.array_equal(getattr(out["1"], k), getattr(out["0"], k)), k
    monkeypatch.setenv("LUMOS_CLUSTER", "1")
    _check(shape, S=40, seed=17, jitter=0.2, every=7)
