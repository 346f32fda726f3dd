"""The C-ABI library (CPU only, no compute calls): it loads, exports every
function include/lumos_b200.h declares, compiles graphs host-side, reports the
reference's error taxonomy, and refuses to replay without a device (there is
no CPU path)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import (DeviceError, DeviceGraph, ScenarioSpec, SimulationError,
                                   _native as N)
from paper_2504_09307_b200.synth import SynthSpec, generate_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "lumos_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = C.CDLL(N.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(N.EXPORTED) <= set(names)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {N.LIB_PATH} 2>/dev/null").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_compile_only_programs():
    sg = generate_graph(SynthSpec(pp=2, dp=2, num_microbatches=4))
    dg = DeviceGraph(sg.graph, compile_only=True)
    assert dg.info["n_components"] == 4 and dg.info["n_programs"] == 2
    assert 2 < dg.info["max_slots"] < 32
    assert dg.n_ranks == 4 and dg.n_streams == 12


def test_estimate_graph_compiles_to_one_component_per_replica():
    sg = generate_graph(SynthSpec(pp=2, dp=2, num_microbatches=4, tp=2, estimate=True))
    dg = DeviceGraph(sg.graph, compile_only=True)
    assert dg.info["n_components"] == 2 and sg.graph.gate_from.shape[0] > 0


def test_invalid_graph_messages_follow_the_reference():
    g = generate_graph(SynthSpec(pp=1, dp=1, num_microbatches=1)).graph
    bad = g.with_durations(np.where(np.arange(g.n) == 3, -1, g.duration))
    with pytest.raises(SimulationError, match="invalid graph: task 3 has negative duration"):
        DeviceGraph(bad, compile_only=True)


def test_replay_without_device_fails_loudly():
    sg = generate_graph(SynthSpec(pp=1, dp=1, num_microbatches=1))
    dg = DeviceGraph(sg.graph, compile_only=True)
    with pytest.raises(DeviceError):
        dg.simulate()
    with pytest.raises(DeviceError):
        dg.replay_batch(ScenarioSpec(count=4), span=np.zeros((4, 3), np.int64))
