"""GPU parity: the CUDA replay path vs the compiled reference (oracle/_ref) and
the C restatement (oracle/lumos_oracle.c), bit-exact on every start/finish.

Reference test strategy mirrored (proj/tests/): hand fixtures of
test_simulator.cpp:58-195, generator replay exactness of test_synth.cpp:175-196
and acceptance C1 (acceptance_main.cpp:133-159), breakdown of
test_metrics.cpp / C3.
"""
import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import (DeviceGraph, ScenarioSpec, SimulationError,
                                   UnsupportedGraphError, simulate, simulate_batch)
from paper_2504_09307_b200.graph import ExecutionGraph

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("walk_ks")]


def _graph(tasks, edges=(), rules=(), window=None):
    """tasks: (lane_kind, lane, start, dur[, rank]) tuples, like make_task in
    test_simulator.cpp:20-33 (GPU tasks are Compute, CPU tasks Other)."""
    n = len(tasks)
    kind = [t[0] for t in tasks]
    g = R.Graph(duration=np.array([t[3] for t in tasks], np.int64),
                original_start=np.array([t[2] for t in tasks], np.int64),
                rank=np.array([t[4] if len(t) > 4 else 0 for t in tasks], np.int32),
                lane_kind=np.array(kind, np.int32), lane=np.array([t[1] for t in tasks], np.int32),
                op_class=np.array([0 if k == 1 else 6 for k in kind], np.uint8),
                task_kind=np.array(kind, np.uint8),
                edge_from=np.array([e[0] for e in edges], np.int32),
                edge_to=np.array([e[1] for e in edges], np.int32),
                rule_kind=np.array([r[0] for r in rules], np.int32),
                rule_task=np.array([r[1] for r in rules], np.int32),
                rule_bound=np.array([r[2] for r in rules], np.int32),
                rule_watch_off=np.cumsum([0] + [len(r[3]) for r in rules]).astype(np.int32),
                watch_rank=np.array([w[0] for r in rules for w in r[3]], np.int32),
                watch_kind=np.array([w[1] for r in rules for w in r[3]], np.int32),
                watch_lane=np.array([w[2] for r in rules for w in r[3]], np.int32),
                window_start=0, window_end=0)
    lo = min((t[2] for t in tasks), default=0)
    hi = max((t[2] + t[3] for t in tasks), default=0)
    g.window_start, g.window_end = (lo, hi) if window is None else window
    return g


def _by_task(trace):
    out = {}
    for tid, s, e in trace.entries:
        out[tid] = (s, e)
    return out


# ----------------------------------------------------------- golden vectors

def test_chain_across_lanes_golden():
    # test_simulator.cpp:58-68: start 10 (recorded 20 ignored), makespan 60
    g = _graph([(0, 1, 0, 10), (1, 7, 20, 50)], edges=[(0, 1)])
    sim = simulate(g)
    e = _by_task(sim)
    assert e[0][0] == 0 and e[1][0] == 10 and sim.makespan == 60


def test_independent_lanes_overlap_golden():
    # test_simulator.cpp:70-77
    assert simulate(_graph([(0, 1, 0, 40), (1, 7, 5, 40)])).makespan == 40


def test_zero_duration_chain():
    # chained variant of test_simulator.cpp:91-105 (zero-duration tasks do not hold the lane)
    g = _graph([(0, 1, 0, 0), (0, 1, 1, 0), (0, 1, 2, 5), (0, 2, 0, 3)],
               edges=[(0, 1), (1, 2), (1, 3)])
    sim = simulate(g)
    e = _by_task(sim)
    assert e[0][1] == 0 and e[1][1] == 0 and e[2][0] == 0 and e[3][0] == 0
    assert sim.makespan == 5


def test_record_wait_fixture_golden():
    # test_simulator.cpp:107-143 through the reference's own parse_trace/build_graph
    ev = []

    def E(name, cat, tid, ts, dur, args=None):
        d = {"name": name, "cat": cat, "ph": "X", "pid": 0, "tid": tid, "ts": ts, "dur": dur}
        if args:
            d["args"] = args
        ev.append(d)
    E("k1", "kernel", 7, 0, 50, {"stream": 7})
    E("cudaEventRecord", "cuda_runtime", 100, 1, 1, {"event": 2, "stream": 7})
    E("cudaStreamWaitEvent", "cuda_runtime", 100, 2, 1, {"event": 2, "stream": 9})
    E("filler", "cpu_op", 100, 3, 2)
    E("cudaLaunchKernel", "cuda_runtime", 100, 5, 1, {"correlation": 4})
    E("k2", "kernel", 9, 61, 20, {"correlation": 4, "stream": 9})
    import json
    h = R.from_trace(json.dumps({"traceEvents": ev}))
    g = h.export(names=True)
    sim = simulate(g)
    e = _by_task(sim)
    k1, k2 = g.names.index("k1"), g.names.index("k2")
    assert e[k1][0] == 0 and e[k2][0] == 50 and sim.makespan == 70


def test_event_sync_golden():
    # test_simulator.cpp:170-195 made chained: the sync passes when its bound task ends (30)
    g = _graph([(1, 7, 0, 30), (1, 7, 1, 100), (0, 1, 2, 4)], edges=[(0, 1)],
               rules=[(2, 2, 0, [])])
    assert _by_task(simulate(g))[2][0] == 30
    g2 = _graph([(1, 7, 0, 30), (1, 7, 1, 100), (0, 1, 2, 4)], edges=[(0, 1)],
                rules=[(2, 2, -1, [])])
    assert _by_task(simulate(g2))[2][0] == 0


def test_stream_sync_static_binding():
    # test_simulator.cpp:145-168 made chained (both kernels queued before the
    # sync): the sync drains the queue -> sync 110, follower 114, makespan 119
    g = _graph([(1, 7, 0, 100), (1, 7, 3, 10), (0, 1, 0, 2), (0, 1, 5, 4), (0, 1, 20, 5)],
               edges=[(0, 1), (2, 3), (3, 4)], rules=[(0, 3, -1, [(0, 1, 7)])])
    h = R.from_graph(g)
    rs, rf, rspan = h.simulate()
    sim = simulate(g)
    e = _by_task(sim)
    assert [e[i][0] for i in range(5)] == rs.tolist()
    assert e[1][0] == 100 and e[3][0] == 110 and e[4][0] == 114 and sim.makespan == 119
    assert sim.makespan == rspan[2]


def test_invalid_graphs_raise_simulation_error():
    # test_simulator.cpp:222-278
    with pytest.raises(SimulationError, match="negative duration"):
        DeviceGraph(_graph([(0, 1, 0, -5)]))
    with pytest.raises(SimulationError, match="invalid task"):
        DeviceGraph(_graph([(0, 1, 0, 5)], edges=[(0, 7)]))
    with pytest.raises(SimulationError, match="cycle"):
        DeviceGraph(_graph([(0, 1, 0, 5), (0, 2, 0, 5)], edges=[(0, 1), (1, 0)]))


def test_empty_scope_sync_is_a_noop():
    # test_simulator.cpp:262-276: empty watch list is a warning; makespan 5
    g = _graph([(0, 1, 0, 5)], rules=[(0, 0, -1, [])])
    assert simulate(g).makespan == 5


# ---- the reference's own (unchained) fixtures, on the event-driven kernel

def test_one_lane_runs_in_recorded_order_golden():
    # test_simulator.cpp:79-89: task 1 (recorded 50) dispatches first
    g = _graph([(0, 1, 100, 10), (0, 1, 50, 10)])
    dg = DeviceGraph(g)
    assert dg.info["n_programs"] == 0  # event-driven path
    e = _by_task(dg.simulate())
    assert e[1][0] == 50 and e[0][0] == 60


def test_zero_duration_golden_unchained():
    # test_simulator.cpp:91-105 exactly
    g = _graph([(0, 1, 0, 0), (0, 1, 1, 0), (0, 1, 2, 5), (0, 2, 0, 3)], edges=[(1, 3)])
    sim = simulate(g)
    e = _by_task(sim)
    assert e[0][1] == 0 and e[1][1] == 0 and e[2][0] == 0 and e[3][0] == 0
    assert sim.makespan == 5


def test_stream_sync_golden_unchained():
    # test_simulator.cpp:145-168 exactly: sync 110, follower 114, makespan 119
    g = _graph([(1, 7, 0, 100), (1, 7, 10, 10), (0, 1, 5, 4), (0, 1, 20, 5)], edges=[(0, 1)],
               rules=[(0, 2, -1, [(0, 1, 7)])])
    sim = simulate(g)
    e = _by_task(sim)
    assert e[1][0] == 100 and e[2][0] == 110 and e[3][0] == 114 and sim.makespan == 119


def test_event_sync_golden_unchained():
    # test_simulator.cpp:170-195 exactly
    g = _graph([(1, 7, 0, 30), (1, 7, 1, 100), (0, 1, 2, 4)], edges=[(0, 1)],
               rules=[(2, 2, 0, [])])
    assert _by_task(simulate(g))[2][0] == 30
    g2 = _graph([(1, 7, 0, 30), (1, 7, 1, 100), (0, 1, 2, 4)], edges=[(0, 1)],
                rules=[(2, 2, -1, [])])
    assert _by_task(simulate(g2))[2][0] == 0


def test_deadlock_raises_simulation_error():
    # test_simulator.cpp:197-220: two syncs watching each other's lanes
    g = _graph([(0, 1, 0, 5), (0, 2, 0, 5)],
               rules=[(0, 0, -1, [(0, 0, 2)]), (0, 1, -1, [(0, 0, 1)])])
    with pytest.raises(SimulationError, match="deadlock") as e:
        simulate(g)
    # the reference's full message, witness chain included (simulate.cpp:258-303)
    with pytest.raises(R.RefError) as r:
        R.from_graph(g).simulate()
    assert str(e.value) == str(r.value).split("] ", 1)[1]


def test_certificate_failure_is_resolved_exactly():
    # chained graph, but the second kernel is enqueued after the sync: the
    # static binding misses it, the certificate fails and the scenario is
    # re-run on the event-driven kernel (same answer as the reference)
    g = _graph([(1, 7, 0, 100), (1, 7, 10, 10), (0, 1, 0, 2), (0, 1, 5, 4), (0, 1, 20, 5)],
               edges=[(0, 1), (2, 3), (3, 4)], rules=[(0, 3, -1, [(0, 1, 7)])])
    h = R.from_graph(g)
    rs, rf, rspan = h.simulate()
    dg = DeviceGraph(g)
    assert dg.info["n_syncs"] == 1 and dg.info["n_programs"] == 1
    status = np.zeros(1, np.int32)
    start = np.zeros((g.n, 1), np.int64)
    fin = np.zeros((g.n, 1), np.int64)
    span = np.zeros((1, 3), np.int64)
    bd = np.zeros((1, dg.n_ranks, 5), np.int64)
    busy = np.zeros((1, dg.n_streams), np.int64)
    dg.replay_batch(ScenarioSpec(count=1), start=start, fin=fin, span=span, status=status,
                    rank_breakdown=bd, stream_busy=busy)
    assert status[0] == 1  # resolved by the exact path
    assert np.array_equal(start[:, 0], rs) and np.array_equal(fin[:, 0], rf)
    assert np.array_equal(span[0], rspan)
    # the rank is on the split accounting; the fix-up reduces the scenario itself
    assert dg.info["n_fused_ranks"] == 1
    wend = max(g.window_end, g.window_start + int(rspan[2]))
    ref_bd = h.breakdown_by_rank(rs, rf, g.window_start, wend)
    assert tuple(bd[0, 0]) == ref_bd[0]
    assert np.array_equal(busy[0], _expected_stream_busy(g, dg, rs, rf, wend))


# ----------------------------------------------------- generator graphs (C1)

C1_SHAPES = [(1, 1, 1, 4), (1, 1, 4, 4), (1, 2, 4, 4), (1, 4, 2, 4), (2, 1, 2, 4), (2, 1, 4, 4),
             (2, 2, 4, 4), (2, 4, 4, 4), (4, 1, 4, 4), (4, 1, 8, 4), (4, 2, 8, 4), (8, 1, 8, 8)]


@pytest.mark.parametrize("jitter", [0.0, 0.05])
@pytest.mark.parametrize("shape", C1_SHAPES)
def test_generated_traces_replay_exactly(shape, jitter):
    pp, dp, m, layers = shape
    h, truth = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers, jitter=jitter, seed=7))
    g = h.export()
    sim = simulate(g)
    rs, rf, rspan = h.simulate()
    e = _by_task(sim)
    assert np.array_equal(np.array([e[i][0] for i in range(g.n)]), rs)
    assert np.array_equal(np.array([e[i][1] for i in range(g.n)]), rf)
    assert sim.makespan == truth == rspan[2]
    # acceptance C1: replay reproduces the recorded starts exactly
    assert np.array_equal(rs, g.original_start)


def _expected_stream_busy(g, dg, rs, rf, wend):
    """Per-stream busy time: sum of the stream's kernel intervals clipped to
    [window_start, wend) (the union is the sum: one stream is one chain)."""
    a = np.clip(rs, g.window_start, wend)
    b = np.clip(rf, g.window_start, wend)
    out = np.zeros(dg.n_streams, np.int64)
    for k in range(dg.n_streams):
        m = (g.rank == dg.stream_rank[k]) & (g.lane_kind == 1) & (g.lane == dg.stream_lane[k])
        out[k] = int(np.maximum(b[m] - a[m], 0).sum())
    return out


def _check_batch(h, g, spec, sc, check_breakdown=True, every=1):
    res = simulate_batch(g, spec, timestamps=True, breakdown=check_breakdown)
    dg = DeviceGraph(g) if check_breakdown else None
    for s in range(0, spec.count, every):
        dur = R.orc_durations(g, sc, spec.first + s)
        rs, rf, rspan = h.simulate(dur)
        assert np.array_equal(res.start[:, s], rs), f"scenario {s} start"
        assert np.array_equal(res.fin[:, s], rf), f"scenario {s} fin"
        assert np.array_equal(res.span[s], rspan), f"scenario {s} span"
        if check_breakdown:
            wend = max(g.window_end, g.window_start + int(rspan[2]))
            ref_bd = h.breakdown_by_rank(rs, rf, g.window_start, wend)
            ranks = sorted(ref_bd)
            for i, r in enumerate(ranks):
                assert tuple(res.rank_breakdown[s, i]) == ref_bd[r], f"scenario {s} rank {r}"
            assert np.array_equal(res.stream_busy[s, :dg.n_streams],
                                  _expected_stream_busy(g, dg, rs, rf, wend)), f"scenario {s} busy"
    return res


@pytest.mark.parametrize("shape", [(1, 2, 4, 4), (2, 2, 4, 4), (4, 2, 8, 4), (1, 1, 6, 4)])
def test_batched_jitter_matches_reference(shape):
    pp, dp, m, layers = shape
    h, _ = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers))
    g = h.export()
    spec = ScenarioSpec(count=200, first=1000, seed=11, jitter=0.3)
    _check_batch(h, g, spec, R.OrcScenarios(seed=11, jitter=0.3))


def test_batched_class_scale_matches_reference():
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4))
    g = h.export()
    spec = ScenarioSpec(count=130, first=5, seed=3, scale_lo=512, scale_hi=2048, scale_den=1024)
    _check_batch(h, g, spec, R.OrcScenarios(seed=3, scale_lo=512, scale_hi=2048, scale_den=1024))


def test_batched_scale_and_jitter_odd_denominator():
    h, _ = R.generate(R.synth_spec(pp=1, dp=2, m=4))
    g = h.export()
    spec = ScenarioSpec(count=64, first=77, seed=5, jitter=0.1, scale_lo=900, scale_hi=1100,
                        scale_den=1000)
    _check_batch(h, g, spec, R.OrcScenarios(seed=5, jitter=0.1, scale_lo=900, scale_hi=1100,
                                            scale_den=1000))


def test_config2_tp2_pp2_dp2_batch():
    # BASELINE config 2: 15B TP2 PP2 DP2 (9,672 tasks), perturbation scenarios
    h, truth = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=48, d_model=6144, d_ffn=12288),
                          tp=2)
    g = h.export()
    assert g.n == 9672
    spec = ScenarioSpec(count=256, seed=250409307, jitter=0.1)
    res = _check_batch(h, g, spec, R.OrcScenarios(seed=250409307, jitter=0.1), every=3)
    assert res.span.shape == (256, 3)


def test_config1_known_answer():
    # 15B pp1 dp2 m4 rank 0: makespan 76,131,231; breakdown
    # {compute 75,535,200, comm 595,937, overlap 0, other 94}
    h, truth = R.generate(R.synth_spec(pp=1, dp=2, m=4, layers=48, d_model=6144, d_ffn=12288),
                          slice_rank=0)
    g = h.export()
    res = simulate_batch(g, ScenarioSpec(count=1))
    assert res.makespan[0] == 76131231 == truth
    assert tuple(res.rank_breakdown[0, 0]) == (76131231, 75535200, 595937, 0, 94)


def test_durations_kernel_matches_restatement():
    h, _ = R.generate(R.synth_spec(pp=2, dp=1, m=2))
    g = h.export()
    dg = DeviceGraph(g)
    for spec, sc in [(ScenarioSpec(count=40, first=9, seed=1, jitter=0.45),
                      R.OrcScenarios(seed=1, jitter=0.45)),
                     (ScenarioSpec(count=40, first=0, seed=2, scale_lo=1, scale_hi=5000,
                                   scale_den=1024),
                      R.OrcScenarios(seed=2, scale_lo=1, scale_hi=5000, scale_den=1024))]:
        dur = dg.scenario_durations(spec)
        for s in range(spec.count):
            assert np.array_equal(dur[:, s], R.orc_durations(g, sc, spec.first + s))


def test_explicit_durations_mode():
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4))
    g = h.export()
    rng = np.random.default_rng(0)
    S = 20
    durs = (g.duration[:, None] * rng.uniform(0.5, 1.5, (g.n, S))).astype(np.int64)
    res = simulate_batch(g, ScenarioSpec(count=S, durations=durs))
    for s in range(S):
        rs, rf, rspan = h.simulate(np.ascontiguousarray(durs[:, s]))
        assert np.array_equal(res.start[:, s], rs) and np.array_equal(res.fin[:, s], rf)


def test_random_graphs_match_reference_and_tick_oracle():
    # acceptance C2 (acceptance_main.cpp:161-202): 1000 draws of the reference
    # fuzz generator (oracles.cpp:222-295); same outcome (incl. deadlock) and
    # identical schedules as simulate() and the microsecond-tick oracle
    rng = R.RefRng(20260818)
    deadlocks = 0
    for trial in range(1000):
        h = rng.random_graph()
        g = h.export()
        # deadlocks are classified by the tick oracle: the reference Engine's
        # deadlock *report* (simulate.cpp:257-302) walks its ready sets with
        # undefined behaviour and can crash; its completed schedules are fine
        try:
            ts_, tf, tspan = h.simulate(tick=True)
            ref_dead = False
        except R.RefError:
            ref_dead = True
        if not ref_dead:
            rs, rf, rspan = h.simulate()
            assert np.array_equal(ts_, rs) and np.array_equal(tf, rf)
        try:
            sim = simulate(g)
        except SimulationError:
            assert ref_dead, f"trial {trial}: device deadlock, reference did not"
            deadlocks += 1
            continue
        assert not ref_dead, f"trial {trial}: reference deadlocked, device did not"
        e = _by_task(sim)
        assert [e[i][0] for i in range(g.n)] == rs.tolist(), f"trial {trial}"
        assert [e[i][1] for i in range(g.n)] == rf.tolist(), f"trial {trial}"
        assert sim.makespan == rspan[2]
    assert deadlocks < 1000


def test_random_graphs_batched_scenarios():
    # event-driven path under scenario durations, checked per scenario
    rng = R.RefRng(7)
    sc = R.OrcScenarios(seed=3, jitter=0.45)
    for trial in range(40):
        h = rng.random_graph()
        g = h.export()
        if R.orc_simulate(g)[0] != 0:  # deadlocking draw (restatement == tick oracle)
            continue
        try:
            res = simulate_batch(g, ScenarioSpec(count=16, seed=3, jitter=0.45))
        except SimulationError:
            continue
        dg = DeviceGraph(g)
        for s_ in range(16):
            dur = R.orc_durations(g, sc, s_)
            rs, rf, rspan = h.simulate(dur)
            assert np.array_equal(res.start[:, s_], rs) and np.array_equal(res.fin[:, s_], rf)
            wend = max(g.window_end, g.window_start + int(rspan[2]))
            ref_bd = h.breakdown_by_rank(rs, rf, g.window_start, wend)
            for i, r in enumerate(sorted(ref_bd)):
                assert tuple(res.rank_breakdown[s_, i]) == ref_bd[r]
            assert np.array_equal(res.stream_busy[s_, :dg.n_streams],
                                  _expected_stream_busy(g, dg, rs, rf, wend))


def test_large_config4_sampled():
    # 175B pp4 dp8 (generator-native, 309,536 tasks): 4 jittered scenarios vs reference
    h, truth = R.generate(R.synth_spec(pp=4, dp=8, m=32, layers=96, d_model=12288, d_ffn=49152,
                                       heads=96))
    g = h.export()
    assert truth == 2183270773
    spec = ScenarioSpec(count=4, first=123, seed=9, jitter=0.1)
    _check_batch(h, g, spec, R.OrcScenarios(seed=9, jitter=0.1), check_breakdown=True)


def test_reduce_fast_and_generic_ranks():
    # K5 has two paths: ranks with one compute-only stream and <= 3 comm-only
    # streams (interval sweep) and everything else (event merge).  Mixing a
    # comm kernel into rank 0's compute stream and a compute kernel into rank
    # 1's p2p stream sends those ranks to the merge while ranks 2/3 stay on the
    # sweep; breakdown and per-stream busy must match the reference on both.
    h0, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h0.export()
    kern = g.task_kind == 1
    r0 = np.flatnonzero(kern & (g.rank == 0) & (g.op_class == 0))
    r1 = np.flatnonzero(kern & (g.rank == 1) & (g.op_class == 1))
    assert len(r0) and len(r1)
    g.op_class = g.op_class.copy()
    g.op_class[r0[len(r0) // 2]] = 1
    g.op_class[r1[len(r1) // 2]] = 0
    h = R.from_graph(g)
    spec = ScenarioSpec(count=64, first=5, seed=21, jitter=0.3)
    _check_batch(h, g, spec, R.OrcScenarios(seed=21, jitter=0.3))
    # and the unmodified graph (every rank on the sweep)
    _check_batch(h0, h0.export(), spec, R.OrcScenarios(seed=21, jitter=0.3))


def test_walk_value_width_paths():
    # the walk keeps uint32 offsets from W when the per-component duration sum
    # bounds every time below W + 2^32 - 1, else int64: one long task pushes
    # the same graph onto the int64 path; both must match the reference
    h0, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h0.export()
    spec = ScenarioSpec(count=32, first=3, seed=17, jitter=0.2)
    sc = R.OrcScenarios(seed=17, jitter=0.2)
    _check_batch(h0, g, spec, sc, every=4)          # uint32 path
    g2 = h0.export()
    g2.duration = g2.duration.copy()
    t = int(np.flatnonzero(g2.task_kind == 1)[-1])  # a late kernel
    g2.duration[t] = 5_000_000_000                  # > 2^32 us on its own
    h2 = R.from_graph(g2)
    _check_batch(h2, g2, spec, sc, every=4)         # int64 path


@pytest.mark.parametrize("first,count", [(0, 37), (1000, 129), (7, 40), (3, 37)])
def test_scenario_pairs_share_philox(first, count):
    # two scenarios per thread draw their jitter from one Philox call (words 0
    # and 1 of counter (task, s >> 1)); odd counts leave a duplicated last
    # column, odd first ids take the one-scenario walk — all equal the oracle
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    spec = ScenarioSpec(count=count, first=first, seed=21, jitter=0.25, scale_lo=800,
                        scale_hi=1200, scale_den=1000)
    _check_batch(h, g, spec, R.OrcScenarios(seed=21, jitter=0.25, scale_lo=800, scale_hi=1200,
                                            scale_den=1000), every=3)


@pytest.mark.parametrize("shape", [(4, 2, 8, 4), (1, 2, 4, 4), (2, 1, 4, 4)])
def test_split_accounting_equals_full_sweep(shape, monkeypatch):
    # split accounting (program.hpp FusedDesc): |A| summed by the walk, only
    # the compute kernels DAG-incomparable with a comm kernel re-read.  Same
    # breakdown / stream busy as the full K5 sweep (LUMOS_FUSED_REDUCE=0) and
    # as the reference breakdown_by_rank.
    pp, dp, m, layers = shape
    h, _ = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers))
    g = h.export()
    spec = ScenarioSpec(count=96, first=40, seed=5, jitter=0.3)
    out = {}
    for env in ("1", "0"):
        monkeypatch.setenv("LUMOS_FUSED_REDUCE", env)
        dg = DeviceGraph(g)
        assert (dg.info["n_fused_ranks"] == dg.n_ranks) == (env == "1")
        if env == "1":
            assert 0 < dg.info["n_candidates"] < dg.info["n_gpu_tasks"] // 4 or pp == 1
        res = simulate_batch(dg, spec, timestamps=True, breakdown=True)
        out[env] = res
    assert np.array_equal(out["1"].rank_breakdown, out["0"].rank_breakdown)
    assert np.array_equal(out["1"].stream_busy, out["0"].stream_busy)
    sc = R.OrcScenarios(seed=5, jitter=0.3)
    for s_ in (0, 47, 95):
        rs, rf, rspan = h.simulate(R.orc_durations(g, sc, spec.first + s_))
        wend = max(g.window_end, g.window_start + int(rspan[2]))
        ref = h.breakdown_by_rank(rs, rf, g.window_start, wend)
        for i, r in enumerate(sorted(ref)):
            assert tuple(out["1"].rank_breakdown[s_, i]) == ref[r]


@pytest.mark.parametrize("des_smem", ["1", "0"])
def test_event_driven_path_equals_walk(monkeypatch, des_smem):
    # two independent device restatements of simulate(): the straight-line
    # walk and the event-driven kernel (LUMOS_FORCE_DES=1 sends every scenario
    # to it; lane state in shared or global memory) agree on every timestamp,
    # span, breakdown and stream busy value
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    spec = ScenarioSpec(count=40, first=6, seed=31, jitter=0.2)
    walk = simulate_batch(g, spec)
    monkeypatch.setenv("LUMOS_FORCE_DES", "1")
    monkeypatch.setenv("LUMOS_DES_SMEM", des_smem)
    dg = DeviceGraph(g)
    assert dg.info["des_only"] == 1
    des = simulate_batch(dg, spec)
    for k in ("start", "fin", "span", "rank_breakdown", "stream_busy"):
        assert np.array_equal(getattr(walk, k), getattr(des, k)), k


def test_edge_cases_match_reference():
    # reference edge cases (test_simulator.cpp, oracles.cpp fuzz): an empty
    # graph, a single task, all-zero durations, and durations near 2^40 us
    # (int64 walk), each on both walk variants via the module fixture
    empty = _graph([])
    res = simulate_batch(empty, ScenarioSpec(count=3, jitter=0.1))
    assert res.span.tolist() == [[0, 0, 0]] * 3
    one = _graph([(1, 7, 5, 40)])
    res = simulate_batch(one, ScenarioSpec(count=5, first=2, seed=4, jitter=0.3))
    h = R.from_graph(one)
    sc = R.OrcScenarios(seed=4, jitter=0.3)
    for s in range(5):
        rs, rf, rspan = h.simulate(R.orc_durations(one, sc, 2 + s))
        assert res.start[0, s] == rs[0] and res.fin[0, s] == rf[0]
        assert np.array_equal(res.span[s], rspan)
    h0, _ = R.generate(R.synth_spec(pp=2, dp=1, m=2, layers=2))
    for scale in (0, 1 << 28):
        g = h0.export()
        g.duration = np.where(g.duration > 0, g.duration * scale + (scale > 0), 0).astype(np.int64)
        hg = R.from_graph(g)
        spec = ScenarioSpec(count=9, first=10, seed=8, jitter=0.2)
        res = simulate_batch(g, spec)
        sc = R.OrcScenarios(seed=8, jitter=0.2)
        for s in (0, 4, 8):
            rs, rf, rspan = hg.simulate(R.orc_durations(g, sc, 10 + s))
            assert np.array_equal(res.start[:, s], rs) and np.array_equal(res.fin[:, s], rf)
            assert np.array_equal(res.span[s], rspan)
