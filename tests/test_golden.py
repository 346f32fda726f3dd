"""Committed golden fixtures (tests/golden/*.npz, made by tools/make_golden.py
from the unmodified reference: generator graphs, tracesim::simulate()
simulate.cpp:341-347 and breakdown_by_rank() metrics.cpp:43-103 on explicit
scenario durations).  They travel to the GPU box, where /root/reference does
not exist, and pin:

* the C restatement (oracle/liblumos_oracle.so) — CPU;
* the CUDA batched path through the C ABI — GPU, bit-exact on every start,
  finish, span and per-rank breakdown value.
"""
import glob
import os

import numpy as np
import pytest

import refshim as R

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _load(path):
    d = np.load(path)
    g = R.Graph(**{k[2:]: d[k] for k in d.files if k.startswith("g_") and k != "g_window"},
                window_start=int(d["g_window"][0]), window_end=int(d["g_window"][1]))
    seed, lo, hi, den = (int(x) for x in d["sc"])
    return d, g, dict(seed=seed, jitter=float(d["jitter"]), scale_lo=lo, scale_hi=hi,
                      scale_den=den)


def test_golden_fixtures_present():
    names = {os.path.basename(p) for p in GOLDEN}
    assert {"config1_jitter.npz", "pp2dp2tp2_scale.npz"} <= names


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_restatement_matches_golden(path):
    d, g, sc = _load(path)
    osc = R.OrcScenarios(**sc)
    first = int(d["first"])
    for i in range(d["durations"].shape[0]):
        dur = R.orc_durations(g, osc, first + i)
        assert np.array_equal(dur, d["durations"][i])
        gi = R.Graph(**{**g.__dict__, "duration": dur})
        rc, s, f, span = R.orc_simulate(gi)
        assert rc == 0
        assert np.array_equal(s, d["start"][i]) and np.array_equal(f, d["fin"][i])
        assert np.array_equal(span, d["span"][i])
        wend = max(g.window_end, g.window_start + int(span[2]))
        ranks = sorted(set(int(r) for r in g.rank))
        got = [R.orc_breakdown_rank(g, s, f, r, g.window_start, wend) for r in ranks]
        assert np.array_equal(np.array(got, np.int64), d["breakdown"][i])


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_cuda_path_matches_golden(path, walk_ks):
    from paper_2504_09307_b200 import ScenarioSpec, simulate_batch
    d, g, sc = _load(path)
    count = d["durations"].shape[0]
    spec = ScenarioSpec(count=count, first=int(d["first"]), **sc)
    res = simulate_batch(g, spec, timestamps=True, breakdown=True)
    for i in range(count):
        assert np.array_equal(res.start[:, i], d["start"][i]), f"scenario {i} start"
        assert np.array_equal(res.fin[:, i], d["fin"][i]), f"scenario {i} fin"
        assert np.array_equal(res.span[i], d["span"][i]), f"scenario {i} span"
        assert np.array_equal(res.rank_breakdown[i], d["breakdown"][i]), f"scenario {i} ranks"
