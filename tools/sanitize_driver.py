"""Small workload for compute-sanitizer (development tool, not a test).

Runs every kernel family once at test size through the C ABI: the K1 walk
(both scenario-per-thread variants, uint32 and int64 slots, jitter / class
scale / explicit durations, the retime walk), K1c cooperative walk (estimate
graph), K4 / K4r / K4v duration kernels, K5 (split accounting, fast and
generic sweeps, utilization bins), K6 deltas, and the event-driven DES path
(an unchained graph and a certificate fix-up).  Results are checked against
the compiled reference where that is cheap; the point is the sanitizer log.

  compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import refshim as R  # noqa: E402
from paper_2504_09307_b200 import DeviceGraph, Retime, ScenarioSpec, simulate_batch  # noqa: E402
from paper_2504_09307_b200.synth import SynthSpec, generate_graph  # noqa: E402


def check(h, g, res, spec, sc, cols):
    for s in cols:
        rs, rf, _ = h.simulate(R.orc_durations(g, sc, spec.first + s))
        assert np.array_equal(res.start[:, s], rs) and np.array_equal(res.fin[:, s], rf), s


def main():
    h, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=2))
    g = h.export()
    sc = R.OrcScenarios(seed=3, jitter=0.2)
    for ks in ("1", "2"):
        os.environ["LUMOS_WALK_KS"] = ks
        spec = ScenarioSpec(count=64, first=8, seed=3, jitter=0.2)
        res = simulate_batch(g, spec, deltas=True, util_bin_width=5000)
        check(h, g, res, spec, sc, [0, 63])
        spec2 = ScenarioSpec(count=33, first=2, seed=3, scale_lo=700, scale_hi=1300,
                             scale_den=1024)
        simulate_batch(g, spec2)
    os.environ.pop("LUMOS_WALK_KS")
    # int64 slots: one very long task
    g2 = h.export()
    g2.duration = g2.duration.copy()
    g2.duration[int(np.flatnonzero(g2.task_kind == 1)[-1])] = 5_000_000_000
    simulate_batch(g2, ScenarioSpec(count=16, seed=1, jitter=0.1))
    # explicit durations and the durations kernel
    dg = DeviceGraph(g)
    dur = dg.scenario_durations(ScenarioSpec(count=8, seed=2, jitter=0.3))
    simulate_batch(g, ScenarioSpec(count=8, durations=dur))
    # generic K5 (mixed streams) without split accounting
    g3 = h.export()
    g3.op_class = g3.op_class.copy()
    g3.op_class[np.flatnonzero((g3.task_kind == 1) & (g3.op_class == 0))[3]] = 1
    simulate_batch(g3, ScenarioSpec(count=16, seed=4, jitter=0.2), util_bin_width=3000)
    # retime walk (K4v + walk) and the materialised retime (K4r)
    hm, _ = R.generate(R.synth_spec(pp=2, dp=2, m=4, layers=2))
    gm = hm.export()
    gm.rt_kind, gm.rt_bytes, gm.rt_group, gm.rt_mnk = hm.retime_meta()
    rt = Retime(alpha_us=[10.0] * 8, bytes_per_us=[40000.0] * 8, source_dp=2,
                target_dp=[2, 4] * 4, source_model=(1024, 4096, 350_000_000),
                target_model=[(1536, 6144, 780_000_000)] * 8)
    simulate_batch(gm, ScenarioSpec(count=8, seed=1, jitter=0.1, retime=rt))
    os.environ["LUMOS_RT_FUSED"] = "0"
    simulate_batch(gm, ScenarioSpec(count=8, seed=1, jitter=0.1, retime=rt))
    os.environ.pop("LUMOS_RT_FUSED")
    # estimate graph: cooperative walk (K1c), incl. the uint32 wrap fix-up path
    sg = generate_graph(SynthSpec(n_layers=4, d_model=1024, d_ffn=4096, n_heads=16, d_head=64,
                                  pp=2, dp=2, num_microbatches=4, estimate=True))
    simulate_batch(sg.graph, ScenarioSpec(count=40, seed=5, jitter=0.2), breakdown=False)
    # event-driven path: an unchained graph, and a certificate failure fix-up
    rng = R.RefRng(7)
    done = 0
    while done < 3:
        gr = rng.random_graph().export()
        if R.orc_simulate(gr)[0] != 0:
            continue
        simulate_batch(gr, ScenarioSpec(count=4, seed=3, jitter=0.3), util_bin_width=37)
        done += 1
    from test_gpu_parity import _graph
    gc = _graph([(1, 7, 0, 100), (1, 7, 10, 10), (0, 1, 0, 2), (0, 1, 5, 4), (0, 1, 20, 5)],
                edges=[(0, 1), (2, 3), (3, 4)], rules=[(0, 3, -1, [(0, 1, 7)])])
    res = simulate_batch(gc, ScenarioSpec(count=2))
    assert res.n_fixups == 2
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
