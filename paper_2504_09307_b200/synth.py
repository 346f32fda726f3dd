"""Synthetic GPT-like training-iteration graphs (host side, C++ via the C ABI).

Restates the reference generator (``synth.cpp:71-170``, ``pipeline.cpp``):
``generate_graph`` returns the replay graph that ``build_graph`` +
``merge_ranks`` produce from the generated one-iteration trace, or, with
``estimate=True``, the generator's own dependency graph with gates (the
``build_pipeline(spec, DurationHook)`` / ``estimate()`` semantics).
``tp > 1`` adds TP replicas of every rank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields
from typing import Optional

import numpy as np

from . import _native as N
from .graph import ExecutionGraph


class TsSynthSpec(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("d_ffn", C.c_int32),
                ("n_heads", C.c_int32), ("d_head", C.c_int32), ("tp", C.c_int32),
                ("pp", C.c_int32), ("dp", C.c_int32), ("num_microbatches", C.c_int32),
                ("tokens_per_microbatch", C.c_int64), ("vocab", C.c_int64),
                ("launch_us", C.c_int64), ("record_us", C.c_int64), ("wait_us", C.c_int64),
                ("sync_us", C.c_int64), ("gemm_ref_us", C.c_int64), ("gemm_ref_mnk", C.c_int64),
                ("bwd_gemm_factor", C.c_double), ("attn_misc_us", C.c_int64),
                ("embed_us", C.c_int64), ("head_us", C.c_int64), ("loss_grad_us", C.c_int64),
                ("optimizer_ref_us", C.c_int64), ("optimizer_ref_bytes", C.c_int64),
                ("alpha_us", C.c_double), ("bytes_per_us", C.c_double),
                ("p2p_recv_base_us", C.c_int64), ("origin", C.c_int64), ("estimate", C.c_int32),
                ("slice_rank", C.c_int32), ("keep_meta", C.c_int32), ("pad", C.c_int32)]


def _lib():
    L = N.lib()
    if not getattr(L, "_synth_bound", False):
        L.ts_synth_defaults.argtypes = [C.POINTER(TsSynthSpec)]
        L.ts_synth_graph.restype = C.c_int
        L.ts_synth_graph.argtypes = [C.POINTER(TsSynthSpec), C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_int64)]
        L.ts_host_graph_desc.restype = C.c_int
        L.ts_host_graph_desc.argtypes = [C.c_void_p, C.POINTER(N.TsGraphDesc)]
        L.ts_host_graph_op_index.restype = C.c_int
        L.ts_host_graph_op_index.argtypes = [C.c_void_p, N.i64p]
        L.ts_host_graph_n_ops.restype = C.c_int64
        L.ts_host_graph_n_ops.argtypes = [C.c_void_p]
        L.ts_host_graph_name_ids.restype = C.c_int
        L.ts_host_graph_name_ids.argtypes = [C.c_void_p, N.i32p]
        L.ts_host_graph_name.restype = C.c_char_p
        L.ts_host_graph_name.argtypes = [C.c_void_p, C.c_int32]
        L.ts_host_graph_free.argtypes = [C.c_void_p]
        L.ts_ingest_traces.restype = C.c_int
        L.ts_ingest_traces.argtypes = [C.POINTER(C.c_char_p), C.c_int32, C.c_int32, C.c_int64,
                                       C.POINTER(C.c_void_p)]
        L.ts_build_rank_graph.restype = C.c_int
        L.ts_build_rank_graph.argtypes = [C.c_int32, C.c_int64, N.i32p, N.u8p, N.i64p, N.i64p,
                                          N.i32p, N.i64p, N.i32p, N.i64p, N.i64p, C.c_char_p,
                                          C.c_int64, C.POINTER(C.c_void_p)]
        L._synth_bound = True
    return L


@dataclass
class SynthSpec:
    """SynthSpec (reference synth.hpp:36-50) plus tp replicas and the mode."""
    n_layers: int = 4
    d_model: int = 1024
    d_ffn: int = 4096
    n_heads: int = 16
    d_head: int = 64
    tp: int = 1
    pp: int = 1
    dp: int = 1
    num_microbatches: int = 4
    tokens_per_microbatch: int = 2048
    vocab: int = 32768
    estimate: bool = False
    slice_rank: int = -1
    origin: int = 1000000
    keep_meta: bool = False  # replay graph keeps Task.meta (the source of a what-if rebuild)

    def to_c(self) -> TsSynthSpec:
        s = TsSynthSpec()
        _lib().ts_synth_defaults(C.byref(s))
        for f in fields(self):
            setattr(s, f.name, int(getattr(self, f.name)))
        return s


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


@dataclass
class SynthGraph:
    graph: ExecutionGraph
    truth_makespan: int
    op_index: np.ndarray   # per task: generator cost index (DurationHook op_index)
    n_ops: int
    names: list


def _from_host(h, names: bool) -> tuple:
    L = _lib()
    d = N.TsGraphDesc()
    L.ts_host_graph_desc(h, C.byref(d))
    n, e, r = d.n_tasks, d.n_edges, d.n_rules
    w = _arr(d.rule_watch_off, r + 1, np.int32)[-1] if r else 0
    g = ExecutionGraph(
        duration=_arr(d.duration, n, np.int64), original_start=_arr(d.original_start, n, np.int64),
        rank=_arr(d.rank, n, np.int32), lane_kind=_arr(d.lane_kind, n, np.int32),
        lane=_arr(d.lane, n, np.int32), op_class=_arr(d.op_class, n, np.uint8),
        task_kind=_arr(d.task_kind, n, np.uint8), edge_from=_arr(d.edge_from, e, np.int32),
        edge_to=_arr(d.edge_to, e, np.int32), rule_kind=_arr(d.rule_kind, r, np.int32),
        rule_task=_arr(d.rule_task, r, np.int32), rule_bound=_arr(d.rule_bound, r, np.int32),
        rule_watch_off=_arr(d.rule_watch_off, r + 1, np.int32),
        watch_rank=_arr(d.watch_rank, w, np.int32), watch_kind=_arr(d.watch_kind, w, np.int32),
        watch_lane=_arr(d.watch_lane, w, np.int32), window_start=d.window_start,
        window_end=d.window_end, gate_from=_arr(d.gate_from, d.n_gates, np.int32),
        gate_to=_arr(d.gate_to, d.n_gates, np.int32),
        gate_kind=_arr(d.gate_kind, d.n_gates, np.uint8))
    if d.rt_kind:
        g.rt_kind = _arr(d.rt_kind, n, np.uint8)
        g.rt_bytes = _arr(d.rt_bytes, n, np.int64)
        g.rt_group = _arr(d.rt_group, n, np.int32)
        g.rt_mnk = _arr(d.rt_mnk, 3 * n, np.int64).reshape(n, 3)
    op_index = np.zeros(max(1, n), np.int64)
    L.ts_host_graph_op_index(h, op_index.ctypes.data_as(N.i64p))
    nm = []
    if names and n:
        ids = np.zeros(n, np.int32)
        L.ts_host_graph_name_ids(h, ids.ctypes.data_as(N.i32p))
        table = {}
        for i in np.unique(ids):
            table[int(i)] = L.ts_host_graph_name(h, int(i)).decode()
        nm = [table[int(i)] for i in ids]
    g.names = nm
    return g, op_index[:n], int(L.ts_host_graph_n_ops(h))


def generate_graph(spec: SynthSpec, names: bool = False) -> SynthGraph:
    L = _lib()
    cs = spec.to_c()
    h = C.c_void_p()
    truth = C.c_int64(0)
    rc = L.ts_synth_graph(C.byref(cs), C.byref(h), C.byref(truth))
    if rc != N.TS_OK:
        from .replay import _raise
        _raise(rc)
    try:
        g, op_index, n_ops = _from_host(h, names)
    finally:
        L.ts_host_graph_free(h)
    return SynthGraph(graph=g, truth_makespan=int(truth.value), op_index=op_index, n_ops=n_ops,
                      names=g.names)


# ------------------------------------------------------------- trace ingest
CATEGORIES = {"cpu_op": 0, "user_annotation": 0, "python_function": 0, "cuda_runtime": 1,
              "cuda_driver": 1, "kernel": 2, "gpu_memcpy": 3, "gpu_memset": 4}


def build_graph_from_events(per_rank: dict, gap_threshold_us: int = 1000) -> ExecutionGraph:
    """build_graph (build.cpp:338-510) per rank + merge_ranks, on parsed events.

    per_rank maps rank -> list of dicts with keys name, cat (EventCategory int),
    ts, dur, tid and optional corr, stream, event (args.event), arg_stream
    (args.stream).  Raises GraphError on a dependency cycle."""
    L = _lib()
    h = C.c_void_p()
    try:
        for rank in sorted(per_rank):
            evs = per_rank[rank]
            names = sorted({e["name"] for e in evs})
            idx = {s: i for i, s in enumerate(names)}
            n = len(evs)
            NOARG = np.iinfo(np.int64).min
            col = lambda k, dt, dflt: np.array([e.get(k, dflt) if e.get(k) is not None else dflt
                                                for e in evs], dt)
            name = np.array([idx[e["name"]] for e in evs], np.int32)
            cat = col("cat", np.uint8, 5)
            ts, dur = col("ts", np.int64, 0), col("dur", np.int64, 0)
            tid = col("tid", np.int32, 0)
            corr = col("corr", np.int64, -1)
            stream = col("stream", np.int32, -1)
            aev = col("event", np.int64, NOARG)
            ast = col("arg_stream", np.int64, NOARG)
            blob = "\n".join(names).encode() + b"\0"
            rc = L.ts_build_rank_graph(rank, n, name.ctypes.data_as(N.i32p),
                                       cat.ctypes.data_as(N.u8p), ts.ctypes.data_as(N.i64p),
                                       dur.ctypes.data_as(N.i64p), tid.ctypes.data_as(N.i32p),
                                       corr.ctypes.data_as(N.i64p), stream.ctypes.data_as(N.i32p),
                                       aev.ctypes.data_as(N.i64p), ast.ctypes.data_as(N.i64p),
                                       blob, gap_threshold_us, C.byref(h))
            if rc != N.TS_OK:
                from .replay import _raise
                _raise(rc)
        g, _, _ = _from_host(h, names=True)
    finally:
        if h:
            L.ts_host_graph_free(h)
    return g


def events_from_chrome(trace: dict, categories: Optional[dict] = None) -> dict:
    """Minimal Chrome trace-event reader (trace_parse.cpp:79-154 semantics for
    the fields the builder uses): ph:"X" events, integer µs (floats rounded
    half away from zero), kineto category names, stream from args or tid for
    GPU events.  Returns rank -> event list for build_graph_from_events."""
    cats = dict(CATEGORIES, **(categories or {}))
    events = trace["traceEvents"] if isinstance(trace, dict) else trace
    out = {}

    def us(v):
        return int(v) if isinstance(v, int) else int(np.sign(v) * np.floor(abs(v) + 0.5))

    def as_int(v):
        try:
            return int(v)
        except (TypeError, ValueError):
            return None
    for i, ev in enumerate(events):
        ph = ev.get("ph", "X")
        if ph == "M":
            continue
        args = ev.get("args") or {}
        keep_zero = any(s in ev.get("name", "") for s in ("EventRecord", "WaitEvent")) or \
            "correlation" in args or "correlation_id" in args
        if ph != "X" and not keep_zero:
            continue
        cat = cats.get(ev.get("cat", ""), 5)
        e = {"name": ev.get("name", ""), "cat": cat, "ts": us(ev["ts"]),
             "dur": us(ev["dur"]) if ph == "X" else 0, "tid": int(ev.get("tid", 0))}
        corr = as_int(args.get("correlation", args.get("correlation_id")))
        if corr is not None:
            e["corr"] = corr
        st = as_int(args.get("stream"))
        if st is not None:
            e["stream"] = st
            e["arg_stream"] = st
        if cat in (2, 3, 4) and "stream" not in e:
            e["stream"] = e["tid"]
        evn = as_int(args.get("event"))
        if evn is not None:
            e["event"] = evn
        out.setdefault(int(ev.get("pid", 0)), []).append(e)
    for r in out:  # parse_trace output order: (pid, ts, tid), stable
        out[r].sort(key=lambda e: (e["ts"], e["tid"]))
    return out


class TsIngestOptions(C.Structure):
    _fields_ = [("paths", C.POINTER(C.c_char_p)), ("n_paths", C.c_int32),
                ("n_threads", C.c_int32), ("manifest", C.c_char_p), ("window", C.c_char_p),
                ("categories_path", C.c_char_p), ("policy_path", C.c_char_p),
                ("keep_meta", C.c_int32), ("pad", C.c_int32)]


def ingest_traces_ex(paths=(), manifest=None, window=None, categories_path=None,
                     policy_path=None, threads: int = 0, names: bool = False) -> ExecutionGraph:
    """ts_ingest_traces_ex: the reference's build_from_inputs with every input
    option (cli.cpp:52-58, 118-137) — a rank manifest, the iteration window
    ("full", "auto" or "START:END"), a custom category table and a build
    policy (JSON file paths, like the CLI's --categories / --policy)."""
    L = _lib()
    if not getattr(L, "_ingest_ex_bound", False):
        L.ts_ingest_traces_ex.restype = C.c_int
        L.ts_ingest_traces_ex.argtypes = [C.POINTER(TsIngestOptions), C.POINTER(C.c_void_p)]
        L._ingest_ex_bound = True
    arr = (C.c_char_p * max(1, len(paths)))(*[str(p).encode() for p in paths])
    enc = lambda x: None if x is None else str(x).encode()
    o = TsIngestOptions(arr, len(paths), int(threads), enc(manifest), enc(window),
                        enc(categories_path), enc(policy_path), 0, 0)
    h = C.c_void_p()
    rc = L.ts_ingest_traces_ex(C.byref(o), C.byref(h))
    if rc != N.TS_OK:
        from .replay import _raise
        _raise(rc)
    try:
        g, _, _ = _from_host(h, names=names)
    finally:
        L.ts_host_graph_free(h)
    return g


def ingest_traces(paths, threads: int = 0, gap_threshold_us: int = 1000,
                  names: bool = False) -> ExecutionGraph:
    """Native parallel ingest of recorded Chrome traces (ts_ingest_traces): the
    reference's parse_trace + build_graph + merge_ranks path for default options
    (cli.cpp:93-137, window "full"), one rank per rank_<N> file or per process id,
    files parsed and ranks built on ``threads`` host threads (0: all cores).
    Raises ValueError (ParseError text) or GraphError (cycles)."""
    L = _lib()
    arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
    h = C.c_void_p()
    rc = L.ts_ingest_traces(arr, len(paths), int(threads), int(gap_threshold_us), C.byref(h))
    if rc != N.TS_OK:
        from .replay import _raise
        _raise(rc)
    try:
        g, _, _ = _from_host(h, names=names)
    finally:
        L.ts_host_graph_free(h)
    return g

