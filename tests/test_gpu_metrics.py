"""GPU parity of the per-scenario metric reductions beyond the 4-way breakdown
(SURVEY §8(f) row 1): utilization_by_rank bins (metrics.cpp:105-155) and the
compare_replay start deltas (metrics.cpp:189-221), checked against the
compiled reference (oracle/_ref) on the same replays.

Reference test strategy mirrored: test_metrics.cpp:98-165 (bins cover the
window and normalise the short tail; overlapping streams are not
double-counted; bins vs a per-microsecond oracle) and :167-193 (compare_replay
ranks tasks by absolute start delta).
"""
import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import ScenarioSpec, SimulationError, simulate_batch
from test_gpu_parity import _graph

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("walk_ks")]


def _check_util(h, g, res, s, rs, rf, width):
    wend = max(g.window_end, g.window_start + int(res.span[s, 2]))
    ref = h.utilization_by_rank(rs, rf, g.window_start, wend, width)
    mine = res.utilization(s, g.window_start, g.window_end)
    if wend <= g.window_start:
        assert ref == {} and res.util_n_bins[s] == 0
        return
    assert sorted(ref) == sorted(set(int(r) for r in g.rank))
    for i, r in enumerate(sorted(ref)):
        assert res.util_n_bins[s] == len(ref[r]), f"scenario {s} rank {r} bins"
        # same double division as metrics.cpp:148-149 -> exact equality
        kept = min(len(ref[r]), res.util_covered.shape[-1])
        assert np.array_equal(mine[i, :kept], ref[r][:kept]), f"scenario {s} rank {r}"


def _check_deltas(h, res, s, rs, rf, n):
    rep = h.compare_replay(rs, rf, worst_n=res.delta_worst.shape[1])
    mine = res.replay_report(s, n, rep["reference_makespan"])
    assert mine["max_abs_delta"] == rep["max_abs_delta"]
    assert mine["simulated_makespan"] == rep["simulated_makespan"]
    assert mine["mean_abs_delta"] == rep["mean_abs_delta"]  # exact sums below 2^53
    assert mine["relative_error"] == rep["relative_error"]
    assert mine["worst"] == rep["worst"]


def test_util_bins_golden():
    # test_metrics.cpp:98-109: window [0,1500), width 1000 -> {0.5, 0.5}.
    # Replay reproduces the intervals: GPU [0,500) on stream 7, a CPU task
    # [0,1000) gating a comm kernel [1000,1250) on stream 9.
    g = _graph([(1, 7, 0, 500), (0, 1, 0, 1000), (1, 9, 1000, 250)], edges=[(1, 2)],
               window=(0, 1500))
    g.op_class[2] = 1
    res = simulate_batch(g, ScenarioSpec(count=2), util_bin_width=1000, util_max_bins=4,
                         deltas=True)
    assert res.util_n_bins.tolist() == [2, 2]
    assert res.util_covered[0, 0, :2].tolist() == [500, 250]
    assert res.utilization(0, 0, 1500).tolist() == [[0.5, 0.5]]
    h = R.from_graph(g)
    rs, rf, _ = h.simulate()
    _check_util(h, g, res, 0, rs, rf, 1000)
    _check_deltas(h, res, 0, rs, rf, g.n)


def test_util_overlap_not_double_counted():
    # test_metrics.cpp:111-116: [0,800) on stream 7 and [400,1000) on stream 9
    g = _graph([(1, 7, 0, 800), (0, 1, 0, 400), (1, 9, 400, 600)], edges=[(1, 2)],
               window=(0, 1000))
    g.op_class[2] = 1
    res = simulate_batch(g, ScenarioSpec(count=1), util_bin_width=1000, util_max_bins=1)
    assert res.utilization(0, 0, 1000).tolist() == [[1.0]]


def test_compare_replay_golden():
    # test_metrics.cpp:167-193: recorded t0 [0,10), t1 [30,40) lane A, t2 [5,25) lane B
    g = _graph([(0, 1, 0, 10), (0, 1, 30, 10), (0, 2, 5, 20)], edges=[(0, 1)], window=(0, 40))
    res = simulate_batch(g, ScenarioSpec(count=1), deltas=True, worst_n=2)
    rep = res.replay_report(0, g.n, 40)
    assert rep["simulated_makespan"] == 20
    assert rep["max_abs_delta"] == 20
    assert rep["mean_abs_delta"] == pytest.approx(25.0 / 3)
    assert rep["worst"] == [{"task": 1, "delta": -20}, {"task": 2, "delta": -5}]  # worst_n = 2
    assert rep["relative_error"] == pytest.approx(0.5)
    full = simulate_batch(g, ScenarioSpec(count=1), deltas=True).replay_report(0, g.n, 40)
    assert [w["task"] for w in full["worst"]] == [1, 2, 0]  # default 10: every task


@pytest.mark.parametrize("width", [1_000, 7_777, 250_000])
def test_util_and_deltas_generator_jitter(width):
    # fast-path ranks (one compute stream + comm streams), 48 jittered scenarios
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    S = 48
    spec = ScenarioSpec(count=S, first=77, seed=5, jitter=0.2)
    res = simulate_batch(g, spec, util_bin_width=width, util_max_bins=4096, deltas=True)
    sc = R.OrcScenarios(seed=5, jitter=0.2)
    for s in range(0, S, 3):
        rs, rf, _ = h.simulate(R.orc_durations(g, sc, spec.first + s))
        assert np.array_equal(res.start[:, s], rs)
        _check_util(h, g, res, s, rs, rf, width)
        _check_deltas(h, res, s, rs, rf, g.n)


def test_util_generic_ranks_all_bins_or_loud_failure():
    # mixed streams send ranks 0/1 to the event merge; a util_max_bins below a
    # window's bin count fails loudly with the count it needs, and the default
    # (util_max_bins=0) returns every bin of every window
    h0, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h0.export()
    kern = g.task_kind == 1
    g.op_class = g.op_class.copy()
    g.op_class[np.flatnonzero(kern & (g.rank == 0) & (g.op_class == 0))[5]] = 1
    g.op_class[np.flatnonzero(kern & (g.rank == 1) & (g.op_class == 1))[3]] = 0
    h = R.from_graph(g)
    S, width = 32, 3_000
    spec = ScenarioSpec(count=S, seed=8, jitter=0.25)
    with pytest.raises(ValueError, match=r"utilization needs \d+ bins per rank; util_max_bins is 7"):
        simulate_batch(g, spec, util_bin_width=width, util_max_bins=7, deltas=True)
    res = simulate_batch(g, spec, util_bin_width=width, deltas=True, worst_n=25)
    assert res.util_covered.shape[-1] == res.util_n_bins.max() > 7
    sc = R.OrcScenarios(seed=8, jitter=0.25)
    for s in range(0, S, 5):
        rs, rf, _ = h.simulate(R.orc_durations(g, sc, s))
        _check_util(h, g, res, s, rs, rf, width)
        _check_deltas(h, res, s, rs, rf, g.n)


@pytest.mark.parametrize("worst_n", [1, 10, 64])
def test_compare_replay_worst_list(worst_n):
    # the device's worst list equals compare_replay's (metrics.cpp:213-217)
    # for the reference default 10 and the bounds, ties broken by task id
    # (a nominal replay of a generator graph has many equal |delta| = 0)
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    spec = ScenarioSpec(count=12, first=3, seed=13, jitter=0.15)
    res = simulate_batch(g, spec, deltas=True, worst_n=worst_n)
    assert res.delta_worst.shape == (12, worst_n, 3)
    sc = R.OrcScenarios(seed=13, jitter=0.15)
    for s in range(0, 12, 4):
        rs, rf, _ = h.simulate(R.orc_durations(g, sc, spec.first + s))
        _check_deltas(h, res, s, rs, rf, g.n)
    nominal = simulate_batch(g, ScenarioSpec(count=2), deltas=True, worst_n=worst_n)
    rs, rf, _ = h.simulate()
    _check_deltas(h, nominal, 0, rs, rf, g.n)


def test_util_random_graphs_event_path():
    # graphs outside the chained class take the event-driven replay, whose
    # reductions (des.cu) also produce the bins
    rng = R.RefRng(11)
    sc = R.OrcScenarios(seed=4, jitter=0.4)
    checked = 0
    for trial in range(40):
        h = rng.random_graph()
        g = h.export()
        if R.orc_simulate(g)[0] != 0:
            continue
        try:
            res = simulate_batch(g, ScenarioSpec(count=8, seed=4, jitter=0.4),
                                 util_bin_width=37, util_max_bins=512, deltas=True)
        except SimulationError:
            continue
        for s in range(8):
            rs, rf, _ = h.simulate(R.orc_durations(g, sc, s))
            assert np.array_equal(res.start[:, s], rs)
            _check_util(h, g, res, s, rs, rf, 37)
            _check_deltas(h, res, s, rs, rf, g.n)
        checked += 1
    assert checked > 10


def test_util_without_timestamps_tiles():
    # no timestamps requested: the reductions run per internal scratch tile
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export()
    spec = ScenarioSpec(count=40, seed=2, jitter=0.1)
    full = simulate_batch(g, spec, util_bin_width=5_000, util_max_bins=1024, deltas=True)
    lean = simulate_batch(g, spec, timestamps=False, breakdown=False, util_bin_width=5_000,
                          util_max_bins=1024, deltas=True)
    assert np.array_equal(full.util_covered, lean.util_covered)
    assert np.array_equal(full.util_n_bins, lean.util_n_bins)
    assert np.array_equal(full.delta_abs_sum, lean.delta_abs_sum)
    assert np.array_equal(full.delta_worst, lean.delta_worst)


def test_scenario_trace_and_chrome_export():
    # a selected scenario of a batch as a SimulatedTrace
    # (entries in (sim_start, task_id) order like simulate()) and as Chrome
    # trace-event JSON for visual audit
    import json
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=4))
    g = h.export(names=True)
    spec = ScenarioSpec(count=8, first=100, seed=3, jitter=0.2)
    res = simulate_batch(g, spec)
    rs, rf, rspan = h.simulate(R.orc_durations(g, R.OrcScenarios(seed=3, jitter=0.2), 105))
    tr = res.trace(5)
    order = np.lexsort((np.arange(g.n), rs))
    assert tr.task_id.tolist() == order.tolist()
    assert tr.sim_start.tolist() == rs[order].tolist() and tr.sim_end.tolist() == rf[order].tolist()
    assert (tr.start, tr.end, tr.makespan) == tuple(int(x) for x in rspan)
    doc = json.loads(res.chrome_trace(g, 5))
    evs = doc["traceEvents"]
    assert len(evs) == g.n and doc["schema_version"] == 1
    assert [e["ts"] for e in evs] == rs[order].tolist()
    assert all(e["cat"] == "kernel" for e in evs if "args" in e)
