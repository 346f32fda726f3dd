"""Native parallel trace ingest against the reference's own
input path (CPU only): parse_trace + load_multirank / split-by-pid + build_graph
+ merge_ranks (cli.cpp:93-137, trace_parse.cpp:79-154, build.cpp:338-542) on
Chrome-trace files written by the reference generator, field by field —
including the names, the iteration window and the retime metadata of
Task.meta.  Error cases follow trace_parse.cpp's ParseError messages."""
import glob
import json
import os

import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200.synth import ingest_traces

FIELDS = ["duration", "original_start", "rank", "lane_kind", "lane", "op_class", "task_kind",
          "edge_from", "edge_to", "rule_kind", "rule_task", "rule_bound", "rule_watch_off",
          "watch_rank", "watch_kind", "watch_lane"]


def _same(g, h):
    r = h.export(names=True)
    for f in FIELDS:
        assert np.array_equal(getattr(g, f), getattr(r, f)), f
    assert (g.window_start, g.window_end) == (r.window_start, r.window_end)
    assert g.names == r.names
    kind, nbytes, group, mnk = h.retime_meta()
    assert np.array_equal(g.rt_kind, kind) and np.array_equal(g.rt_bytes, nbytes)
    assert np.array_equal(g.rt_group, group) and np.array_equal(g.rt_mnk, mnk)


@pytest.mark.parametrize("shape", [(1, 2, 4, 0.0), (2, 2, 4, 0.05), (4, 1, 8, 0.0),
                                   (2, 4, 4, 0.03)])
def test_ingest_matches_reference(tmp_path, shape):
    pp, dp, m, jitter = shape
    k = R.write_rank_traces(R.synth_spec(pp=pp, dp=dp, m=m, layers=4, jitter=jitter),
                            str(tmp_path))
    paths = sorted(glob.glob(str(tmp_path / "rank_*.json")))
    assert len(paths) == k == pp * dp
    h = R.ingest_traces(paths)
    for threads in (1, 3, 0):
        _same(ingest_traces(paths, threads=threads, names=True), h)


def test_unmarked_file_splits_by_pid(tmp_path):
    # one file without a rank_<N> marker: ranks are the process ids (load_inputs)
    R.write_rank_traces(R.synth_spec(pp=2, dp=2, m=4, layers=4), str(tmp_path))
    paths = sorted(glob.glob(str(tmp_path / "rank_*.json")))
    events = []
    for p in paths:
        events += json.load(open(p))["traceEvents"]
    allp = tmp_path / "combined.json"
    allp.write_text(json.dumps({"traceEvents": events}))
    _same(ingest_traces([str(allp)], threads=2, names=True), R.ingest_traces(paths))


def test_fractional_and_edge_fields(tmp_path):
    # float timestamps round half away from zero; string args parse like the
    # reference; zero-duration EventRecord records are kept
    evs = [
        {"ph": "X", "cat": "cuda_runtime", "name": "cudaLaunchKernel", "pid": 3, "tid": 9,
         "ts": 100.5, "dur": 4.49, "args": {"correlation": "7"}},
        {"ph": "X", "cat": "Kernel", "name": "k0", "pid": 3, "tid": 7, "ts": 110, "dur": 20,
         "args": {"correlation": 7, "stream": "7", "bytes": "12x"}},
        {"ph": "i", "cat": "cuda_runtime", "name": "cudaEventRecord", "pid": 3, "tid": 9,
         "ts": 111, "args": {"event": 5, "stream": 7}},
        {"ph": "M", "name": "process_name", "pid": 3, "args": {"name": "x"}},
        {"ph": "X", "cat": "cpu_op", "name": "aten::mm", "pid": 3, "tid": 9, "ts": 130.5,
         "dur": 1.5},
    ]
    p = tmp_path / "rank_3.json"
    p.write_text(json.dumps(evs))
    _same(ingest_traces([str(p)], names=True), R.ingest_traces([str(p)]))


@pytest.mark.parametrize("body,msg", [
    ('{"traceEvents": [{"ph": "X", "name": "a", "cat": "cpu_op", "ts": 1}]}',
     'missing dur \\(truncated trace\\?\\)'),
    ('{"traceEvents": [{"ph": "X", "name": "a", "cat": "cpu_op", "ts": 1, "dur": -2}]}',
     "negative dur"),
    ('{"traceEvents": [{"ph": "X", "name": "cudaLaunchKernel", "cat": "cuda_runtime", '
     '"ts": 1, "dur": 2}]}', "without a correlation id"),
    ('{"traceEvents": [1]}', "event is not an object"),
    ('{"events": []}', "must be an event array or an object with traceEvents"),
    ('{"traceEvents": [', "malformed trace JSON"),
])
def test_ingest_errors(tmp_path, body, msg):
    p = tmp_path / "rank_0.json"
    p.write_text(body)
    with pytest.raises(Exception, match=msg):
        ingest_traces([str(p)])


def test_duplicate_rank_rejected(tmp_path):
    R.write_rank_traces(R.synth_spec(pp=1, dp=1, m=2, layers=2), str(tmp_path))
    a = str(tmp_path / "rank_0.json")
    b = str(tmp_path / "copy_rank_0.json")
    os.link(a, b)
    with pytest.raises(Exception, match="rank 0 appears in more than one input"):
        ingest_traces([a, b])
