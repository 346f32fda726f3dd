"""Host-side graph sources vs the reference (CPU only).

* generate_graph(estimate=False) == the reference's generate -> build_graph
  -> merge_ranks graph, field by field (build.cpp:338-542, synth.cpp:140-170);
* build_graph_from_events on hand-written traces == the reference's
  parse_trace -> build_graph (test_graph_builder.cpp fixtures' shapes);
* generate_graph(estimate=True): the generator-semantics graph evaluated as a
  max-plus longest path with gates (a small pure-Python restatement here)
  reproduces build_pipeline's event times, nominal and with a DurationHook.
"""
import json
from collections import defaultdict

import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200.synth import (SynthSpec, build_graph_from_events, events_from_chrome,
                                         generate_graph)

FIELDS = ["duration", "original_start", "rank", "lane_kind", "lane", "op_class", "task_kind",
          "edge_from", "edge_to", "rule_kind", "rule_task", "rule_bound", "rule_watch_off",
          "watch_rank", "watch_kind", "watch_lane"]


def _spec(pp, dp, m, layers=4, d=1024, f=4096, tp=1, sl=-1, estimate=False):
    heads = d // 128 if d >= 2048 else 16
    return SynthSpec(n_layers=layers, d_model=d, d_ffn=f, n_heads=heads, d_head=d // heads, tp=tp,
                     pp=pp, dp=dp, num_microbatches=m, slice_rank=sl, estimate=estimate)


def _assert_same(mine, ref):
    for k in FIELDS:
        assert np.array_equal(getattr(mine, k), getattr(ref, k)), k
    assert (mine.window_start, mine.window_end) == (ref.window_start, ref.window_end)


SHAPES = [(1, 1, 1, 4), (1, 1, 4, 4), (1, 2, 4, 4), (1, 4, 2, 4), (2, 1, 2, 4), (2, 1, 4, 4),
          (2, 2, 4, 4), (2, 4, 4, 4), (4, 1, 4, 4), (4, 1, 8, 4), (4, 2, 8, 4), (8, 1, 8, 8)]


@pytest.mark.parametrize("shape", SHAPES)
def test_replay_graph_matches_reference(shape):
    pp, dp, m, layers = shape
    mine = generate_graph(_spec(pp, dp, m, layers))
    h, truth = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers))
    _assert_same(mine.graph, h.export())
    assert mine.truth_makespan == truth


def test_config_graphs_match_reference():
    # BASELINE config 1 (15B pp1 dp2 m4, rank 0) and config 2 (15B TP2 PP2 DP2)
    for kw, tp, sl in [(dict(pp=1, dp=2, m=4), 1, 0), (dict(pp=2, dp=2, m=4), 2, -1)]:
        mine = generate_graph(_spec(kw["pp"], kw["dp"], kw["m"], 48, 6144, 12288, tp=tp, sl=sl))
        h, truth = R.generate(R.synth_spec(layers=48, d_model=6144, d_ffn=12288, **kw), tp=tp,
                              slice_rank=sl)
        _assert_same(mine.graph, h.export())
    assert mine.graph.n == 9672


def test_config4_graph_matches_reference():
    # 175B pp4 dp8 m32 (generator-native, 309,536 tasks)
    mine = generate_graph(_spec(4, 8, 32, 96, 12288, 49152))
    h, truth = R.generate(R.synth_spec(pp=4, dp=8, m=32, layers=96, d_model=12288, d_ffn=49152,
                                       heads=96))
    _assert_same(mine.graph, h.export())
    assert mine.truth_makespan == truth == 2183270773


def _ev(name, cat, tid, ts, dur, args=None, pid=0):
    d = {"name": name, "cat": cat, "ph": "X", "pid": pid, "tid": tid, "ts": ts, "dur": dur}
    if args:
        d["args"] = args
    return d


TRACES = {
    # test_simulator.cpp:107-143 record/wait fixture
    "record_wait": [
        _ev("k1", "kernel", 7, 0, 50, {"stream": 7}),
        _ev("cudaEventRecord", "cuda_runtime", 100, 1, 1, {"event": 2, "stream": 7}),
        _ev("cudaStreamWaitEvent", "cuda_runtime", 100, 2, 1, {"event": 2, "stream": 9}),
        _ev("filler", "cpu_op", 100, 3, 2),
        _ev("cudaLaunchKernel", "cuda_runtime", 100, 5, 1, {"correlation": 4}),
        _ev("k2", "kernel", 9, 61, 20, {"correlation": 4, "stream": 9})],
    # nested span dropping, orphan kernel, gap edge across threads, syncs
    "mixed": [
        _ev("outer", "cpu_op", 1, 0, 100), _ev("inner", "cpu_op", 1, 10, 20),
        _ev("cudaLaunchKernel", "cuda_runtime", 1, 40, 5, {"correlation": 9}),
        _ev("gemm", "kernel", 7, 50, 500, {"correlation": 9, "stream": 7}),
        _ev("orphan_nccl_AllReduce", "kernel", 9, 60, 30, {"stream": 9}),
        _ev("cudaStreamSynchronize", "cuda_runtime", 1, 110, 450, {"stream": 7}),
        _ev("worker", "cpu_op", 2, 3000, 10),
        _ev("cudaDeviceSynchronize", "cuda_runtime", 2, 3020, 5),
        _ev("cudaEventSynchronize", "cuda_runtime", 2, 3030, 5, {"event": 77})],
}


@pytest.mark.parametrize("name", sorted(TRACES))
def test_build_graph_from_trace_matches_reference(name):
    doc = {"traceEvents": TRACES[name]}
    mine = build_graph_from_events(events_from_chrome(doc))
    ref = R.from_trace(json.dumps(doc)).export()
    _assert_same(mine, ref)


def test_build_graph_cycle_raises_graph_error():
    from paper_2504_09307_b200 import GraphError
    # a wait whose record-side kernel runs after the waiting stream's kernel
    # that it precedes in the lane chain -> the reference reports a cycle
    evs = [_ev("cudaLaunchKernel", "cuda_runtime", 1, 0, 1, {"correlation": 1}),
           _ev("a", "kernel", 7, 5, 10, {"correlation": 1, "stream": 7}),
           _ev("cudaLaunchKernel", "cuda_runtime", 1, 2, 1, {"correlation": 2}),
           _ev("b", "kernel", 9, 1, 10, {"correlation": 2, "stream": 9}),
           _ev("cudaEventRecord", "cuda_runtime", 1, 4, 1, {"event": 5, "stream": 7}),
           _ev("cudaStreamWaitEvent", "cuda_runtime", 1, 6, 1, {"event": 5, "stream": 9}),
           _ev("cudaLaunchKernel", "cuda_runtime", 1, 8, 1, {"correlation": 3}),
           _ev("c", "kernel", 9, 0, 10, {"correlation": 3, "stream": 9})]
    doc = {"traceEvents": evs}
    try:
        R.from_trace(json.dumps(doc)).export()
        ref_raises = False
    except RuntimeError:
        ref_raises = True
    if ref_raises:
        with pytest.raises(GraphError, match="dependency cycle"):
            build_graph_from_events(events_from_chrome(doc))
    else:
        _assert_same(build_graph_from_events(events_from_chrome(doc)), R.from_trace(
            json.dumps(doc)).export())


# ------------------------------------------------------------ estimate mode

def longest_path_with_gates(g, dur):
    """start = max(W, preds' finish); finish = max(start, gate values) + d,
    gate value = finish(from) (kind 0) or start(from) (kind 1).  Evaluated in
    topological order of the split graph {S(v), F(v)} (Kahn)."""
    n = g.n
    W = g.window_start
    deps = defaultdict(list)  # node -> nodes it reads; S(v) = v, F(v) = n + v
    for u, v in zip(g.edge_from.tolist(), g.edge_to.tolist()):
        deps[v].append(n + u)
    for v in range(n):
        deps[n + v].append(v)
    for u, v, k in zip(g.gate_from.tolist(), g.gate_to.tolist(), g.gate_kind.tolist()):
        deps[n + v].append(n + u if k == 0 else u)
    users = defaultdict(list)
    indeg = [0] * (2 * n)
    for x, ds in deps.items():
        indeg[x] = len(ds)
        for y in ds:
            users[y].append(x)
    val = [0] * (2 * n)
    queue = [x for x in range(2 * n) if indeg[x] == 0]
    done = 0
    while queue:
        x = queue.pop()
        done += 1
        if x < n:
            val[x] = max([W] + [val[y] for y in deps[x]])
        else:
            val[x] = max(val[y] for y in deps[x]) + int(dur[x - n])
        for z in users[x]:
            indeg[z] -= 1
            if indeg[z] == 0:
                queue.append(z)
    assert done == 2 * n, "cycle"
    return np.array(val[:n], np.int64), np.array(val[n:], np.int64)


def _lane_sequences(pid, tid, ts, dur):
    seq = defaultdict(list)
    for p, t, a, d in zip(pid, tid, ts, dur):
        seq[(int(p), int(t))].append((int(a), int(a + d)))
    return seq


def _ref_pipeline(spec_json, hook=None):
    import ctypes as C
    lib = R.ref()
    lib.ref_pipeline_events.restype = C.c_int64
    lib.ref_pipeline_events.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.c_int64,
                                        C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int64,
                                        C.POINTER(C.c_int64)]
    cap = 4_000_000
    pid = np.zeros(cap, np.int32)
    tid = np.zeros(cap, np.int32)
    ts = np.zeros(cap, np.int64)
    dur = np.zeros(cap, np.int64)
    nops = C.c_int64(0)
    h = None if hook is None else np.ascontiguousarray(hook, np.int64)
    n = lib.ref_pipeline_events(spec_json.encode(),
                                None if h is None else h.ctypes.data_as(C.POINTER(C.c_int64)),
                                0 if h is None else h.shape[0],
                                pid.ctypes.data_as(C.POINTER(C.c_int32)),
                                tid.ctypes.data_as(C.POINTER(C.c_int32)),
                                ts.ctypes.data_as(C.POINTER(C.c_int64)),
                                dur.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(nops))
    assert n > 0, R.ref().ref_last_error()
    return _lane_sequences(pid[:n], tid[:n], ts[:n], dur[:n]), int(nops.value)


def _my_lane_sequences(g, start, fin):
    tid = np.where(g.lane_kind == 1, g.lane, g.lane)
    order = np.lexsort((np.arange(g.n), start, g.rank))
    seq = defaultdict(list)
    # per lane in processing order == by (start, task id) within the lane
    for i in order:
        seq[(int(g.rank[i]), int(tid[i]))].append((int(start[i]), int(fin[i])))
    return seq


@pytest.mark.parametrize("shape", [(2, 2, 4, 4), (1, 2, 4, 4), (4, 2, 8, 4), (2, 4, 4, 4),
                                   (1, 1, 2, 4)])
def test_estimate_graph_nominal_matches_build_pipeline(shape):
    pp, dp, m, layers = shape
    sg = generate_graph(_spec(pp, dp, m, layers, estimate=True))
    g = sg.graph
    start, fin = longest_path_with_gates(g, g.duration)
    ref, nops = _ref_pipeline(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers))
    assert nops == sg.n_ops
    assert _my_lane_sequences(g, start, fin) == ref
    assert int(fin.max()) - g.window_start == sg.truth_makespan


@pytest.mark.parametrize("shape", [(2, 2, 4, 4), (1, 2, 4, 4), (4, 2, 8, 4)])
def test_estimate_graph_with_hook_matches_build_pipeline(shape):
    # scenario durations through the DurationHook (pipeline.hpp:72-74): the
    # hook returns the oracle's scenario duration of the task behind op_index
    pp, dp, m, layers = shape
    sg = generate_graph(_spec(pp, dp, m, layers, estimate=True))
    g = sg.graph
    sc = R.OrcScenarios(seed=5, jitter=0.4)
    for scen in (0, 17):
        dur = R.orc_durations(R.Graph(**{k: getattr(g, k) for k in FIELDS},
                                      window_start=g.window_start, window_end=g.window_end),
                              sc, scen)
        hook = np.zeros(sg.n_ops, np.int64)
        hook[sg.op_index] = dur
        start, fin = longest_path_with_gates(g, dur)
        ref, _ = _ref_pipeline(R.synth_spec(pp=pp, dp=dp, m=m, layers=layers), hook)
        assert _my_lane_sequences(g, start, fin) == ref


@pytest.mark.parametrize("shape", [(1, 2, 4), (2, 2, 4), (4, 1, 8), (2, 4, 4)])
def test_generator_retime_metadata_matches_reference(shape):
    # the per-task retime metadata (ts_graph_desc.rt_*) our generator attaches
    # equals what the reference's Task.meta yields (synth.cpp:46-48, 122-133,
    # pipeline.cpp:162-166, 297), task for task
    pp, dp, m = shape
    sg = generate_graph(SynthSpec(pp=pp, dp=dp, num_microbatches=m, n_layers=4))
    h, _ = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=4))
    kind, nbytes, group, mnk = h.retime_meta()
    g = sg.graph
    assert np.array_equal(g.rt_kind, kind)
    assert np.array_equal(g.rt_bytes, nbytes)
    assert np.array_equal(g.rt_group, group)
    assert np.array_equal(g.rt_mnk, mnk)
