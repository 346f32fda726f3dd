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
from paper_2504_09307_b200.synth import ingest_traces, ingest_traces_ex

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
    # both files carry a rank_<N> marker: load_multirank's duplicate check
    # (trace_parse.cpp:286-296) fires before load_inputs' take()
    with pytest.raises(Exception, match="duplicate rank 0 from '.*copy_rank_0.json'"):
        ingest_traces([a, b])
    with pytest.raises(Exception, match="duplicate rank 0 from"):
        R.ingest_traces_ex([a, b])


def _two_iterations(src, dst, shift):
    """A rank trace holding two copies of its iteration `shift` us apart (new
    correlation / event ids for the copy)."""
    doc = json.load(open(src))
    evs = doc["traceEvents"]
    more = []
    for e in evs:
        c = dict(e)
        c["ts"] = e["ts"] + shift
        if "args" in e:
            a = dict(e["args"])
            for k in ("correlation", "event"):
                if k in a:
                    a[k] = int(a[k]) + 1_000_000
            c["args"] = a
        more.append(c)
    # the second iteration gets a few extra host ops so it wins detect_iteration_window
    main = [e for e in evs if e.get("cat") == "cpu_op" or e.get("cat") == "cuda_runtime"]
    t_end = max(e["ts"] + e.get("dur", 0) for e in more)
    for k in range(3):
        more.append({"name": "extra_op", "cat": "cpu_op", "ph": "X", "ts": t_end + 10 * k + 1,
                     "dur": 2, "pid": main[0]["pid"], "tid": main[0]["tid"]})
    json.dump({"traceEvents": evs + more}, open(dst, "w"))


@pytest.mark.parametrize("window", ["auto", "first", "second"])
def test_ingest_window_options(tmp_path, window):
    # --window auto picks the iteration with the most main-thread events
    # (detect_iteration_window), START:END keeps events starting inside plus
    # kernels of kept launches (filter_window)
    src = tmp_path / "src"
    src.mkdir()
    R.write_rank_traces(R.synth_spec(pp=2, dp=1, m=4, layers=4), str(src))
    paths = []
    for p in sorted(glob.glob(str(src / "rank_*.json"))):
        d = str(tmp_path / os.path.basename(p))
        _two_iterations(p, d, 50_000_000)
        paths.append(d)
    w = {"auto": "auto", "first": "0:40000000", "second": "50000000:99000000"}[window]
    h = R.ingest_traces_ex(paths, window=w)
    g = ingest_traces_ex(paths, window=w, names=True)
    _same(g, h)
    full = ingest_traces_ex(paths, names=True)
    assert g.n * 2 < full.n + 10


def test_ingest_manifest_categories_policy(tmp_path):
    # a manifest maps ranks to files without rank markers (relative paths), a
    # custom category table renames the kernel category, a build policy moves
    # the gap threshold and the communication patterns
    src = tmp_path / "src"
    src.mkdir()
    R.write_rank_traces(R.synth_spec(pp=2, dp=2, m=4, layers=4), str(src))
    man = {}
    for p in sorted(glob.glob(str(src / "rank_*.json"))):
        r = int(os.path.basename(p)[5:-5])
        doc = json.load(open(p))
        for e in doc["traceEvents"]:
            if e.get("cat") == "kernel":
                e["cat"] = "device_kernel"
        name = f"trace_{r}.json"
        json.dump(doc, open(tmp_path / name, "w"))
        man[str(r)] = name
    (tmp_path / "manifest.json").write_text(json.dumps(man))
    cats = json.dumps({"device_kernel": "GpuKernel"})
    policy = json.dumps({"gap_threshold_us": 20, "comm_patterns": ["nccl", "sendrecv"],
                         "sync_names": {"cudaDeviceSynchronize": "device",
                                        "cudaStreamSynchronize": "stream"}})
    (tmp_path / "cats.json").write_text(cats)
    (tmp_path / "policy.json").write_text(policy)
    h = R.ingest_traces_ex([], manifest=str(tmp_path / "manifest.json"), categories=cats,
                           policy=policy)
    g = ingest_traces_ex([], manifest=str(tmp_path / "manifest.json"),
                         categories_path=str(tmp_path / "cats.json"),
                         policy_path=str(tmp_path / "policy.json"), threads=3, names=True)
    _same(g, h)
    assert (g.task_kind == 1).sum() > 0
    # errors of the options follow the reference's ParseError texts
    (tmp_path / "bad.json").write_text(json.dumps({"x": "Kernelish"}))
    with pytest.raises(Exception, match="unknown category 'Kernelish'"):
        ingest_traces_ex([], manifest=str(tmp_path / "manifest.json"),
                         categories_path=str(tmp_path / "bad.json"))
    (tmp_path / "badp.json").write_text(json.dumps({"sync_names": {"a": "b"}}))
    with pytest.raises(Exception, match="must be device.stream.event"):
        ingest_traces_ex([], manifest=str(tmp_path / "manifest.json"),
                         policy_path=str(tmp_path / "badp.json"))
    with pytest.raises(Exception, match="window must be 'full', 'auto' or START:END"):
        ingest_traces_ex([], manifest=str(tmp_path / "manifest.json"), window="last")


def _tricky_events():
    """Records that exercise the fast scanner's JSON handling: escapes and
    UTF-8 in names, every number form, duplicate keys, args of every type,
    skipped phases and non-object args."""
    return [
        {"ph": "X", "cat": "cuda_runtime", "name": "cudaLaunchKernel", "pid": 0, "tid": 9,
         "ts": 100, "dur": 4, "args": {"correlation": 1, "Input Dims": [[1, 2], []],
                                         "flag": True, "none": None, "ratio": 0.25,
                                         "nested": {"a": [1, {"b": "c"}]}}},
        {"ph": "X", "cat": "KERNEL", "name": "gemm \"q\\k\"\tv/é\U0001F600 layers.3",
         "pid": 0, "tid": 7, "ts": 1.04e2, "dur": 20, "args": {"correlation": 1, "stream": 7,
                                                                "m": "2048", "n": 4096,
                                                                "k": "1024", "region": "p2p",
                                                                "bytes": 18446744073709551615}},
        {"ph": "X", "cat": "cuda_runtime", "name": "cudaLaunchKernel", "pid": 0, "tid": 9,
         "ts": 104, "dur": 3, "args": {"correlation_id": "2"}},
        {"ph": "X", "cat": "kernel", "name": "ncclDevKernel_AllReduce", "pid": 0, "tid": 9,
         "ts": 130, "dur": 5, "args": {"correlation": 2, "stream": "11", "collective": "allreduce",
                                      "group_size": "4", "bytes": "1048576"}},
        {"ph": "i", "cat": "cuda_runtime", "name": "cudaEventRecord", "pid": 0, "tid": 9,
         "ts": 140, "args": {"event": "5x", "stream": 11}},
        {"ph": "B", "cat": "cpu_op", "name": "begin-only", "pid": 0, "tid": 9, "ts": 141},
        {"ph": "M", "name": "thread_name", "pid": 0, "tid": 9, "args": {"name": "main"}},
        {"ph": "X", "cat": "cpu_op", "name": "aten::mm", "pid": 0, "tid": 9, "ts": 150.5,
         "dur": 2.5, "args": [1, 2]},
        {"ph": "X", "cat": "cpu_op", "name": "late", "pid": 0, "tid": 9, "ts": 149, "dur": 1},
        {"ph": "X", "cat": "unknown_cat", "pid": 0, "tid": 9, "ts": 160, "dur": 0},
    ]


def _write_tricky(path, dup_keys):
    text = json.dumps({"meta": {"x": [1, 2.5, "y"]}, "traceEvents": _tricky_events(),
                       "tail": None}, ensure_ascii=False, indent=1)
    if dup_keys:  # a repeated key: the last value wins (nlohmann)
        text = text.replace('"ts": 149', '"ts": 1, "ts": 149', 1)
        text = text.replace('"args": {"event": "5x"', '"args": {"stream": 3, "event": "5x"', 1)
    path.write_text(text, encoding="utf-8")


@pytest.mark.parametrize("dup_keys", [False, True])
def test_fast_scanner_equals_dom_and_reference(tmp_path, monkeypatch, dup_keys):
    # the single-pass scanner (default) and the DOM path (LUMOS_INGEST_DOM=1)
    # must both equal the reference's parse_trace + build_graph
    p = tmp_path / "rank_0.json"
    _write_tricky(p, dup_keys)
    ref = R.ingest_traces([str(p)])
    for dom in ("0", "1"):
        monkeypatch.setenv("LUMOS_INGEST_DOM", dom)
        _same(ingest_traces([str(p)], names=True), ref)


def test_fast_scanner_on_generated_traces(tmp_path, monkeypatch):
    R.write_rank_traces(R.synth_spec(pp=2, dp=2, m=4, layers=4, jitter=0.05), str(tmp_path))
    paths = sorted(glob.glob(str(tmp_path / "rank_*.json")))
    h = R.ingest_traces(paths)
    for dom in ("0", "1"):
        monkeypatch.setenv("LUMOS_INGEST_DOM", dom)
        _same(ingest_traces(paths, threads=2, names=True), h)


@pytest.mark.parametrize("body", [
    '{"traceEvents": [{"ph": "X", "name": "a", "cat": "cpu_op", "ts": 1, "dur": 2,}]}',
    '{"traceEvents": [{"ph": "X", "name": "a\\x", "cat": "cpu_op", "ts": 1, "dur": 2}]}',
    '{"traceEvents": [{"ph": "X", "name": "\\ud800", "cat": "cpu_op", "ts": 1, "dur": 2}]}',
    '{"traceEvents": [{"ph": "X", "name": "a", "cat": "cpu_op", "ts": 01, "dur": 2}]}',
    '{"traceEvents": []} trailing',
    '{"traceEvents": [{"ph": 3, "name": "a", "cat": "cpu_op", "ts": 1, "dur": 2}]}',
    '{"traceEvents": [{"ph": "X", "name": "a", "cat": "cpu_op", "ts": "1", "dur": 2}]}',
])
def test_fast_scanner_defers_errors_to_the_dom_path(tmp_path, monkeypatch, body):
    # malformed JSON and unexpected field types raise exactly what the DOM
    # path raises (the scanner hands such files to it)
    p = tmp_path / "rank_0.json"
    p.write_text(body)
    errs = []
    for dom in ("0", "1"):
        monkeypatch.setenv("LUMOS_INGEST_DOM", dom)
        with pytest.raises(Exception) as e:
            ingest_traces([str(p)])
        errs.append(str(e.value))
    assert errs[0] == errs[1]
