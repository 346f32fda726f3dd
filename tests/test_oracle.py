"""Pins the CPU restatement (oracle/lumos_oracle.c) before it is trusted as a
checker (CPU only):

* the reference's golden vectors: test_simulator.cpp:58-195 hand fixtures,
  test_metrics.cpp:38-58 breakdown fixtures, SURVEY §8c config-1 known answer;
* the compiled reference (oracle/_ref) and its tick oracle on the reference's
  own fuzz generator (acceptance C2 seeds) and on generator graphs;
* the scenario-duration formulas: Philox2x32-10 Random123 known-answer
  vectors, exact big-integer mul_div (transform.cpp:38-43), exact rational
  jitter rounding (synth.cpp:150-155 semantics).
"""
import ctypes as C
from fractions import Fraction

import numpy as np
import pytest

import refshim as R


def G(tasks, edges=(), rules=(), window=None):
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


def sim(g):
    rc, s, f, span = R.orc_simulate(g)
    return rc, s, f, span


# ----------------------------------------------------------- golden vectors

def test_golden_chain_across_lanes():
    rc, s, f, span = sim(G([(0, 1, 0, 10), (1, 7, 20, 50)], edges=[(0, 1)]))
    assert rc == 0 and s.tolist() == [0, 10] and span[2] == 60


def test_golden_overlap_and_lane_order():
    assert sim(G([(0, 1, 0, 40), (1, 7, 5, 40)]))[3][2] == 40
    rc, s, f, span = sim(G([(0, 1, 100, 10), (0, 1, 50, 10)]))
    assert s.tolist() == [60, 50] and span[2] == 20


def test_golden_zero_duration():
    rc, s, f, span = sim(G([(0, 1, 0, 0), (0, 1, 1, 0), (0, 1, 2, 5), (0, 2, 0, 3)],
                           edges=[(1, 3)]))
    assert f[0] == 0 and f[1] == 0 and s[2] == 0 and s[3] == 0 and span[2] == 5


def test_golden_stream_sync():
    g = G([(1, 7, 0, 100), (1, 7, 10, 10), (0, 1, 5, 4), (0, 1, 20, 5)], edges=[(0, 1)],
          rules=[(0, 2, -1, [(0, 1, 7)])])
    rc, s, f, span = sim(g)
    assert (s[1], s[2], s[3], span[2]) == (100, 110, 114, 119)


def test_golden_event_sync_and_deadlock_and_validation():
    base = [(1, 7, 0, 30), (1, 7, 1, 100), (0, 1, 2, 4)]
    assert sim(G(base, edges=[(0, 1)], rules=[(2, 2, 0, [])]))[1][2] == 30
    assert sim(G(base, edges=[(0, 1)], rules=[(2, 2, -1, [])]))[1][2] == 0
    dead = G([(0, 1, 0, 5), (0, 2, 0, 5)],
             rules=[(0, 0, -1, [(0, 0, 2)]), (0, 1, -1, [(0, 0, 1)])])
    assert sim(dead)[0] == 2
    assert sim(G([(0, 1, 0, -5)]))[0] == 1
    assert sim(G([(0, 1, 0, 5)], edges=[(0, 7)]))[0] == 1
    assert sim(G([(0, 1, 0, 5), (0, 2, 0, 5)], edges=[(0, 1), (1, 0)]))[0] == 1
    assert sim(G([(0, 1, 0, 5)], rules=[(0, 0, -1, [])]))[3][2] == 5


def test_golden_breakdown_fixtures():
    # test_metrics.cpp:38-48: 5/5/5/5 ; :50-58 clipping
    g = G([(1, 7, 0, 10), (1, 9, 5, 10)])
    g.op_class = np.array([0, 1], np.uint8)
    s = np.array([0, 5], np.int64)
    f = np.array([10, 15], np.int64)
    assert R.orc_breakdown_rank(g, s, f, 0, 0, 20) == (20, 5, 5, 5, 5)
    g2 = G([(0, 1, 0, 20), (1, 7, -5, 13), (1, 7, 18, 12)])
    g2.op_class = np.array([6, 0, 1], np.uint8)
    s2 = np.array([0, -5, 18], np.int64)
    f2 = np.array([20, 8, 30], np.int64)
    assert R.orc_breakdown_rank(g2, s2, f2, 0, 0, 20) == (20, 8, 2, 0, 10)


def test_config1_known_answer():
    h, truth = R.generate(R.synth_spec(pp=1, dp=2, m=4, layers=48, d_model=6144, d_ffn=12288),
                          slice_rank=0)
    g = h.export()
    rc, s, f, span = sim(g)
    assert rc == 0 and span[2] == truth == 76131231
    wend = max(g.window_end, g.window_start + int(span[2]))
    assert R.orc_breakdown_rank(g, s, f, 0, g.window_start, wend) == \
        (76131231, 75535200, 595937, 0, 94)


# ------------------------------------------------- vs the compiled reference

def test_restatement_matches_reference_on_fuzz_graphs():
    rng = R.RefRng(20260818)  # acceptance C2 seed
    dead = 0
    for trial in range(1000):
        h = rng.random_graph()
        g = h.export()
        rc, s, f, span = sim(g)
        try:
            ts, tf, tspan = h.simulate(tick=True)
            tdead = False
        except R.RefError:
            tdead = True
        assert tdead == (rc == 2), trial
        if rc == 0:
            rs, rf, rspan = h.simulate()
            assert np.array_equal(rs, s) and np.array_equal(rf, f), trial
            assert np.array_equal(ts, s) and np.array_equal(rspan, span), trial
        else:
            dead += 1
    assert 0 < dead < 1000


@pytest.mark.parametrize("shape", [(1, 2, 4, 4), (2, 2, 4, 4), (4, 2, 8, 4)])
def test_restatement_matches_reference_under_durations(shape):
    pp, dp, m, layers = shape
    h, _ = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers))
    g = h.export()
    sc = R.OrcScenarios(seed=9, jitter=0.3, scale_lo=800, scale_hi=1300, scale_den=1024)
    for scen in range(5):
        dur = R.orc_durations(g, sc, scen)
        rc, s, f, span = sim(g.__class__(**{**g.__dict__, "duration": dur}))
        rs, rf, rspan = h.simulate(dur)
        assert rc == 0 and np.array_equal(rs, s) and np.array_equal(rf, f)
        wend = max(g.window_end, g.window_start + int(span[2]))
        ref_bd = h.breakdown_by_rank(rs, rf, g.window_start, wend)
        for r, b in ref_bd.items():
            assert R.orc_breakdown_rank(g, s, f, r, g.window_start, wend) == b


# ------------------------------------------------------ duration formulas

def test_philox_known_answers():
    # Random123 kat_vectors, philox2x32 10 rounds
    out = (C.c_uint32 * 2)()
    for ctr0, ctr1, key, want in [(0, 0, 0, (0xff1dae59, 0x6cd10df2)),
                                  (0xffffffff, 0xffffffff, 0xffffffff, (0x2c3f628b, 0xab4fd7ad)),
                                  (0x243f6a88, 0x85a308d3, 0x13198a2e, (0xdd7ce038, 0xf62a4c12))]:
        R.orc().orc_philox2x32_10(ctr0, ctr1, key, out)
        assert (out[0], out[1]) == want


def test_mul_div_exact():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        a = int(rng.integers(0, 2**40))
        num = int(rng.integers(0, 2**22))
        den = int(rng.integers(1, 2**20))
        assert R.orc().orc_mul_div(a, num, den) == (a * num + den // 2) // den
    # transform.cpp:38-43 golden: rescale 1200 by 4096^3 / 1024^3 ... within int64
    assert R.orc().orc_mul_div(1200, 64, 1) == 76800


def _jitter_exact(d, w, j):
    """max(1, llround(d * (1 + u))) with u = 2j*U01 - j, U01 = w * 2^-32,
    evaluated in IEEE double exactly as the restatement does (round-to-nearest
    at each op)."""
    import struct

    def rn(x):  # round a Fraction to the nearest double
        return float(x)
    u01 = float(w) * 2.0 ** -32
    t = rn(Fraction(2.0 * j) * Fraction(u01))
    u = rn(Fraction(t) + Fraction(-j))
    fct = rn(Fraction(1.0) + Fraction(u))
    p = Fraction(float(d)) * Fraction(fct)
    p = Fraction(rn(p))
    q = int(p + Fraction(1, 2)) if p >= 0 else -int(-p + Fraction(1, 2))
    _ = struct
    return max(1, q)


def test_jitter_formula_exact():
    sc = R.OrcScenarios(seed=12345, jitter=0.37)
    out = (C.c_uint32 * 2)()
    key = (12345 ^ (12345 >> 32)) & 0xffffffff
    rng = np.random.default_rng(2)
    for _ in range(3000):
        d = int(rng.integers(0, 10**9))
        task = int(rng.integers(0, 2**31))
        scen = int(rng.integers(0, 2**31))
        got = R.orc().orc_scenario_duration(C.byref(sc), scen, task, d, 0)
        if d == 0:
            assert got == 0
            continue
        # one Philox call per scenario pair: word (scen & 1) of (task, scen >> 1)
        R.orc().orc_philox2x32_10(task, scen >> 1, key, out)
        assert got == _jitter_exact(d, out[scen & 1], 0.37)


def test_reference_metric_shims_golden():
    # the checker for the device metric reductions (tests/test_gpu_metrics.py)
    # is the reference's own metrics.cpp; pin the shim on its unit-test values:
    # utilization bins test_metrics.cpp:98-109, compare_replay :167-193
    from test_gpu_parity import _graph
    g = _graph([(1, 7, 0, 500), (0, 1, 0, 1000), (1, 9, 1000, 250)], edges=[(1, 2)],
               window=(0, 1500))
    g.op_class[2] = 1
    h = R.from_graph(g)
    rs, rf, _ = h.simulate()
    util = h.utilization_by_rank(rs, rf, 0, 1500, 1000)
    assert list(util) == [0] and util[0].tolist() == [0.5, 0.5]
    g = _graph([(0, 1, 0, 10), (0, 1, 30, 10), (0, 2, 5, 20)], edges=[(0, 1)], window=(0, 40))
    h = R.from_graph(g)
    rs, rf, _ = h.simulate()
    rep = h.compare_replay(rs, rf, worst_n=2)
    assert rep["reference_makespan"] == 40 and rep["simulated_makespan"] == 20
    assert rep["max_abs_delta"] == 20 and rep["mean_abs_delta"] == pytest.approx(25.0 / 3)
    assert rep["worst"] == [{"task": 1, "delta": -20}, {"task": 2, "delta": -5}]
    assert rep["relative_error"] == pytest.approx(0.5)
