"""ctypes driver for the oracle libraries (TEST INFRASTRUCTURE ONLY).

* ``oracle/_ref/libtracesim_ref.so`` — the unmodified reference compiled by
  ``oracle/Makefile`` (namespace ``tracesim_ref``) plus ``oracle/ref_shim.cpp``.
* ``oracle/liblumos_oracle.so`` — the plain-C restatement ``oracle/lumos_oracle.c``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline/reference
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtracesim_ref.so")
ORC_SO = os.path.join(ROOT, "oracle", "liblumos_oracle.so")

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


def _p(a, t):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:  # a strided view would be read (or written) wrongly
        raise ValueError("refshim: arrays passed to the C side must be C-contiguous")
    return a.ctypes.data_as(t)


class OrcScenarios(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("jitter", C.c_double), ("scale_lo", C.c_int32),
                ("scale_hi", C.c_int32), ("scale_den", C.c_int32), ("reserved", C.c_int32)]


class OrcGraph(C.Structure):
    _fields_ = [("n", C.c_int32), ("duration", _i64p), ("original_start", _i64p),
                ("rank", _i32p), ("lane_kind", _i32p), ("lane", _i32p),
                ("n_edges", C.c_int64), ("edge_from", _i32p), ("edge_to", _i32p),
                ("n_rules", C.c_int32), ("rule_kind", _i32p), ("rule_task", _i32p),
                ("rule_bound", _i32p), ("rule_watch_off", _i32p), ("watch_rank", _i32p),
                ("watch_kind", _i32p), ("watch_lane", _i32p), ("window_start", C.c_int64)]


@dataclass
class Graph:
    """SoA copy of a tracesim ExecutionGraph (build.hpp:73-85)."""
    duration: np.ndarray
    original_start: np.ndarray
    rank: np.ndarray
    lane_kind: np.ndarray
    lane: np.ndarray
    op_class: np.ndarray
    task_kind: np.ndarray
    edge_from: np.ndarray
    edge_to: np.ndarray
    rule_kind: np.ndarray
    rule_task: np.ndarray
    rule_bound: np.ndarray
    rule_watch_off: np.ndarray
    watch_rank: np.ndarray
    watch_kind: np.ndarray
    watch_lane: np.ndarray
    window_start: int
    window_end: int
    names: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return int(self.duration.shape[0])

    def default_scale_class(self) -> np.ndarray:
        """Default scenario class: 0 host task, 1 GPU compute, 2 GPU communication."""
        cls = np.zeros(self.n, np.uint8)
        cls[self.task_kind == 1] = 1
        cls[(self.task_kind == 1) & (self.op_class == 1)] = 2
        return cls

    def is_comm(self) -> np.ndarray:
        return (self.op_class == 1).astype(np.uint8)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    # the reference library (-std=c++20) must resolve libstdc++'s locale facet
    # ids globally: with numpy's runtime libraries loaded first, its std::regex
    # (tag_tasks) otherwise picks up a mismatched collate facet and crashes
    C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
    return C.CDLL(path)


_ref = None
_orc = None


def ref():
    global _ref
    if _ref is None:
        lib = _load(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_graph_generate.restype = C.c_void_p
        lib.ref_graph_generate.argtypes = [C.c_char_p, C.c_int, C.c_int, _i64p]
        lib.ref_graph_from_trace.restype = C.c_void_p
        lib.ref_graph_from_trace.argtypes = [C.c_char_p, C.c_int]
        lib.ref_graph_from_arrays.restype = C.c_void_p
        lib.ref_graph_from_arrays.argtypes = [C.c_int32, _i64p, _i64p, _i32p, _i32p, _i32p, _u8p,
                                              C.c_int64, _i32p, _i32p, C.c_int32, _i32p, _i32p,
                                              _i32p, _i32p, _i32p, _i32p, _i32p, C.c_int64,
                                              C.c_int64]
        lib.ref_rng_new.restype = C.c_void_p
        lib.ref_rng_new.argtypes = [C.c_uint64]
        lib.ref_rng_free.argtypes = [C.c_void_p]
        lib.ref_graph_random.restype = C.c_void_p
        lib.ref_graph_random.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.ref_graph_free.argtypes = [C.c_void_p]
        lib.ref_graph_sizes.argtypes = [C.c_void_p, _i64p]
        lib.ref_graph_export.argtypes = [C.c_void_p, _i64p, _i64p, _i32p, _i32p, _i32p, _u8p, _u8p,
                                         _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p,
                                         _i32p]
        lib.ref_graph_names.restype = C.c_int64
        lib.ref_graph_names.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        for fn in (lib.ref_simulate, lib.ref_tick_simulate):
            fn.restype = C.c_int
            fn.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p]
        lib.ref_breakdown_by_rank.restype = C.c_int
        lib.ref_breakdown_by_rank.argtypes = [C.c_void_p, _i64p, _i64p, C.c_int64, C.c_int64,
                                              _i64p, C.c_int]
        lib.ref_utilization_by_rank.restype = C.c_int
        lib.ref_utilization_by_rank.argtypes = [C.c_void_p, _i64p, _i64p, C.c_int64, C.c_int64,
                                                C.c_int64, C.POINTER(C.c_double), _i32p, _i32p,
                                                C.c_int, C.c_int]
        lib.ref_compare_replay.restype = C.c_int
        lib.ref_compare_replay.argtypes = [C.c_void_p, _i64p, _i64p, C.c_int32, _i64p,
                                           C.POINTER(C.c_double)]
        lib.ref_graph_retime_meta.restype = C.c_int
        lib.ref_graph_retime_meta.argtypes = [C.c_void_p, _u8p, _i64p, _i32p, _i64p]
        lib.ref_apply_retime.restype = C.c_void_p
        lib.ref_apply_retime.argtypes = [C.c_void_p, _i64p, _i64p, C.c_int, C.c_int, C.c_double,
                                         C.c_double]
        lib.ref_apply_whatif.restype = C.c_void_p
        lib.ref_apply_whatif.argtypes = [C.c_void_p, _i64p, _i64p, _i32p, _i32p, C.c_double,
                                         C.c_double, C.c_int64, C.c_char_p, C.c_int64]
        lib.ref_write_rank_traces.restype = C.c_int
        lib.ref_write_rank_traces.argtypes = [C.c_char_p, C.c_char_p]
        lib.ref_ingest_traces.restype = C.c_void_p
        lib.ref_ingest_traces.argtypes = [C.POINTER(C.c_char_p), C.c_int]
        lib.ref_bench_simulate.restype = C.c_double
        lib.ref_bench_simulate.argtypes = [C.c_void_p, C.POINTER(OrcScenarios), C.c_int64,
                                           C.c_int32, _u8p, C.c_int, _i64p,
                                           C.POINTER(C.c_double)]
        _ref = lib
    return _ref


def orc():
    global _orc
    if _orc is None:
        lib = _load(ORC_SO)
        lib.orc_simulate.restype = C.c_int
        lib.orc_simulate.argtypes = [C.POINTER(OrcGraph), _i64p, _i64p, _i64p]
        lib.orc_breakdown_rank.argtypes = [C.c_int32, _i32p, _i32p, _u8p, _i64p, _i64p, C.c_int32,
                                           C.c_int64, C.c_int64, _i64p]
        lib.orc_philox2x32_10.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.POINTER(C.c_uint32)]
        lib.orc_mul_div.restype = C.c_int64
        lib.orc_mul_div.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        lib.orc_class_num.restype = C.c_int32
        lib.orc_class_num.argtypes = [C.POINTER(OrcScenarios), C.c_int64, C.c_int32]
        lib.orc_scenario_duration.restype = C.c_int64
        lib.orc_scenario_duration.argtypes = [C.POINTER(OrcScenarios), C.c_int64, C.c_int32,
                                              C.c_int64, C.c_int32]
        lib.orc_fill_durations.argtypes = [C.POINTER(OrcScenarios), C.c_int64, C.c_int32, _i64p,
                                           _u8p, _i64p]
        _orc = lib
    return _orc


class RefGraphHandle:
    """Owns a tracesim_ref::ExecutionGraph inside the reference library."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(ref().ref_last_error().decode())
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_graph_free(self.h)
            self.h = None

    def export(self, names: bool = False) -> Graph:
        lib = ref()
        sz = np.zeros(6, np.int64)
        lib.ref_graph_sizes(self.h, _p(sz, _i64p))
        n, e, r, w = (int(x) for x in sz[:4])
        g = Graph(duration=np.zeros(n, np.int64), original_start=np.zeros(n, np.int64),
                  rank=np.zeros(n, np.int32), lane_kind=np.zeros(n, np.int32),
                  lane=np.zeros(n, np.int32), op_class=np.zeros(n, np.uint8),
                  task_kind=np.zeros(n, np.uint8), edge_from=np.zeros(e, np.int32),
                  edge_to=np.zeros(e, np.int32), rule_kind=np.zeros(r, np.int32),
                  rule_task=np.zeros(r, np.int32), rule_bound=np.zeros(r, np.int32),
                  rule_watch_off=np.zeros(r + 1, np.int32), watch_rank=np.zeros(w, np.int32),
                  watch_kind=np.zeros(w, np.int32), watch_lane=np.zeros(w, np.int32),
                  window_start=int(sz[4]), window_end=int(sz[5]))
        lib.ref_graph_export(self.h, _p(g.duration, _i64p), _p(g.original_start, _i64p),
                             _p(g.rank, _i32p), _p(g.lane_kind, _i32p), _p(g.lane, _i32p),
                             _p(g.op_class, _u8p), _p(g.task_kind, _u8p), _p(g.edge_from, _i32p),
                             _p(g.edge_to, _i32p), _p(g.rule_kind, _i32p), _p(g.rule_task, _i32p),
                             _p(g.rule_bound, _i32p), _p(g.rule_watch_off, _i32p),
                             _p(g.watch_rank, _i32p), _p(g.watch_kind, _i32p),
                             _p(g.watch_lane, _i32p))
        if names:
            nb = lib.ref_graph_names(self.h, None, 0)
            buf = C.create_string_buffer(int(nb) + 1)
            lib.ref_graph_names(self.h, buf, nb)
            g.names = buf.raw[:nb].decode().split("\n")[:-1]
        return g

    def simulate(self, durations=None, tick=False):
        """Reference simulate() (or the tick oracle); returns (start, fin, span) or raises."""
        lib = ref()
        sz = np.zeros(6, np.int64)
        lib.ref_graph_sizes(self.h, _p(sz, _i64p))
        n = int(sz[0])
        start = np.zeros(n, np.int64)
        fin = np.zeros(n, np.int64)
        span = np.zeros(3, np.int64)
        d = None if durations is None else np.ascontiguousarray(durations, np.int64)
        fn = lib.ref_tick_simulate if tick else lib.ref_simulate
        rc = fn(self.h, _p(d, _i64p), _p(start, _i64p), _p(fin, _i64p), _p(span, _i64p))
        if rc != 0:
            raise RefError(rc, lib.ref_last_error().decode())
        return start, fin, span

    def breakdown_by_rank(self, start, fin, wstart, wend, max_ranks=4096):
        out = np.zeros((max_ranks, 6), np.int64)
        k = ref().ref_breakdown_by_rank(self.h, _p(start, _i64p), _p(fin, _i64p), wstart, wend,
                                        _p(out, _i64p), max_ranks)
        return {int(row[0]): tuple(int(x) for x in row[1:]) for row in out[:k]}

    def utilization_by_rank(self, start, fin, wstart, wend, bin_width, max_ranks=1024,
                            max_bins=4096):
        """{rank: np.array of bin values} from the reference metrics.cpp:105-155."""
        vals = np.zeros((max_ranks, max_bins), np.float64)
        ranks = np.zeros(max_ranks, np.int32)
        nb = np.zeros(max_ranks, np.int32)
        k = ref().ref_utilization_by_rank(self.h, _p(start, _i64p), _p(fin, _i64p), wstart, wend,
                                          bin_width, vals.ctypes.data_as(C.POINTER(C.c_double)),
                                          _p(ranks, _i32p), _p(nb, _i32p), max_ranks, max_bins)
        return {int(ranks[i]): vals[i, :nb[i]].copy() for i in range(k)}

    def compare_replay(self, start, fin, worst_n=5):
        """ReplayReport of the reference compare_replay (metrics.cpp:189-221)."""
        oi = np.zeros(5 + 2 * worst_n, np.int64)
        od = np.zeros(2, np.float64)
        ref().ref_compare_replay(self.h, _p(start, _i64p), _p(fin, _i64p), worst_n,
                                 _p(oi, _i64p), od.ctypes.data_as(C.POINTER(C.c_double)))
        nw = int(oi[4])
        return {"reference_makespan": int(oi[0]), "simulated_makespan": int(oi[1]),
                "max_abs_delta": int(oi[2]), "zero_reference": bool(oi[3]),
                "mean_abs_delta": float(od[0]), "relative_error": float(od[1]),
                "worst": [{"task": int(oi[5 + k]), "delta": int(oi[5 + worst_n + k])}
                          for k in range(nw)]}

    def retime_meta(self):
        """(rt_kind, rt_bytes, rt_group, rt_mnk) arrays of ts_graph_desc from Task.meta."""
        n = self.export().n
        kind = np.zeros(n, np.uint8)
        nb = np.zeros(n, np.int64)
        grp = np.zeros(n, np.int32)
        mnk = np.zeros((n, 3), np.int64)
        ref().ref_graph_retime_meta(self.h, _p(kind, _u8p), _p(nb, _i64p), _p(grp, _i32p),
                                    _p(mnk, _i64p))
        return kind, nb, grp, mnk

    def apply_retime(self, src_model=None, tgt_model=None, src_dp=1, tgt_dp=1, alpha=10.0,
                     bytes_per_us=50000.0):
        """The reference change_hidden then scale_dp (apply_whatif's retime path)."""
        sm = np.asarray(src_model if src_model is not None else (0, 0, 0), np.int64)
        tm = np.asarray(tgt_model, np.int64) if tgt_model is not None else None
        p = ref().ref_apply_retime(self.h, _p(sm, _i64p), _p(tm, _i64p) if tm is not None else None,
                                   src_dp, tgt_dp, alpha, bytes_per_us)
        if not p:
            raise RefError(3, ref().ref_last_error().decode())
        return RefGraphHandle(p)

    def apply_whatif(self, src_model, tgt_model, src_par, tgt_par, alpha=10.0,
                     bytes_per_us=50000.0, activation_bytes=0):
        """The reference apply_whatif (transform.cpp:713-760): (handle, notes).
        model = (n_params, n_layers, d_model, d_ffn, n_heads, d_head),
        par = (tp, pp, dp, num_microbatches)."""
        sm = np.ascontiguousarray(src_model, np.int64)
        tm = np.ascontiguousarray(tgt_model, np.int64)
        sp = np.ascontiguousarray(src_par, np.int32)
        tp = np.ascontiguousarray(tgt_par, np.int32)
        buf = C.create_string_buffer(4096)
        p = ref().ref_apply_whatif(self.h, _p(sm, _i64p), _p(tm, _i64p), _p(sp, _i32p),
                                   _p(tp, _i32p), alpha, bytes_per_us, int(activation_bytes),
                                   buf, 4096)
        if not p:
            raise RefError(3, ref().ref_last_error().decode())
        return RefGraphHandle(p), buf.value.decode()

    def bench_simulate(self, sc: OrcScenarios, first: int, count: int, cls, threads: int,
                       with_fill: bool = False):
        """Wall seconds of `count` reference simulate() calls on `threads` host
        threads (durations pre-filled outside the clock) and the makespans;
        with_fill adds the fill seconds."""
        mk = np.zeros(count, np.int64)
        fill = C.c_double(0.0)
        secs = ref().ref_bench_simulate(self.h, C.byref(sc), first, count, _p(cls, _u8p), threads,
                                        _p(mk, _i64p), C.byref(fill))
        return (secs, mk, fill.value) if with_fill else (secs, mk)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def synth_spec(pp=1, dp=1, m=4, layers=4, d_model=1024, d_ffn=4096, heads=None, jitter=0.0,
               seed=1, tokens=2048, vocab=32768) -> str:
    heads = heads or max(1, d_model // 128 if d_model >= 2048 else 16)
    return json.dumps({"parallelism": {"pp": pp, "dp": dp, "num_microbatches": m},
                       "model": {"n_layers": layers, "d_model": d_model, "d_ffn": d_ffn,
                                 "n_heads": heads, "d_head": d_model // heads},
                       "tokens_per_microbatch": tokens, "vocab": vocab,
                       "jitter_pct": jitter, "seed": seed})


def generate(spec_json: str, tp: int = 1, slice_rank: int = -1):
    truth = C.c_int64(0)
    h = RefGraphHandle(ref().ref_graph_generate(spec_json.encode(), tp, slice_rank,
                                                C.byref(truth)))
    return h, int(truth.value)


def from_trace(trace_json: str, rank: int = -1):
    return RefGraphHandle(ref().ref_graph_from_trace(trace_json.encode(), rank))


def write_rank_traces(spec_json: str, directory: str) -> int:
    """The reference generator's trace as rank_<r>.json Chrome files."""
    k = ref().ref_write_rank_traces(spec_json.encode(), directory.encode())
    if k < 0:
        raise RefError(3, ref().ref_last_error().decode())
    return k


def ingest_traces(paths) -> "RefGraphHandle":
    """The reference's load_multirank + build_graph + merge_ranks on files."""
    arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
    h = ref().ref_ingest_traces(arr, len(paths))
    if not h:
        raise RefError(3, ref().ref_last_error().decode())
    return RefGraphHandle(h)


def ingest_traces_ex(paths, manifest=None, window=None, categories=None, policy=None):
    """The reference's build_from_inputs (cli.cpp:118-137) with options; the
    category table / policy are JSON texts."""
    lib = ref()
    lib.ref_ingest_traces_ex.restype = C.c_void_p
    lib.ref_ingest_traces_ex.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_char_p,
                                         C.c_char_p, C.c_char_p]
    arr = (C.c_char_p * max(1, len(paths)))(*[p.encode() for p in paths])
    enc = lambda x: None if x is None else x.encode()
    h = lib.ref_ingest_traces_ex(arr, len(paths), enc(manifest), enc(window), enc(categories),
                                 enc(policy))
    if not h:
        raise RefError(3, lib.ref_last_error().decode())
    return RefGraphHandle(h)


def from_graph(g: Graph):
    return RefGraphHandle(ref().ref_graph_from_arrays(
        g.n, _p(g.duration, _i64p), _p(g.original_start, _i64p), _p(g.rank, _i32p),
        _p(g.lane_kind, _i32p), _p(g.lane, _i32p), _p(g.op_class, _u8p), g.edge_from.shape[0],
        _p(g.edge_from, _i32p), _p(g.edge_to, _i32p), g.rule_kind.shape[0], _p(g.rule_kind, _i32p),
        _p(g.rule_task, _i32p), _p(g.rule_bound, _i32p), _p(g.rule_watch_off, _i32p),
        _p(g.watch_rank, _i32p), _p(g.watch_kind, _i32p), _p(g.watch_lane, _i32p),
        g.window_start, g.window_end))


class RefRng:
    def __init__(self, seed):
        self.h = ref().ref_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_rng_free(self.h)
            self.h = None

    def random_graph(self, max_tasks=50, max_lanes=4):
        return RefGraphHandle(ref().ref_graph_random(self.h, max_tasks, max_lanes))


# ---------------------------------------------------------------- restatement

def orc_graph_struct(g: Graph, keep):
    """Build an OrcGraph view; `keep` collects arrays to keep them alive."""
    arrs = [np.ascontiguousarray(a) for a in (
        g.duration, g.original_start, g.rank, g.lane_kind, g.lane, g.edge_from, g.edge_to,
        g.rule_kind, g.rule_task, g.rule_bound, g.rule_watch_off, g.watch_rank, g.watch_kind,
        g.watch_lane)]
    keep.extend(arrs)
    (dur, ost, rk, lk, ln, ef, et, rki, rt, rb, rwo, wr, wk, wl) = arrs
    return OrcGraph(g.n, _p(dur, _i64p), _p(ost, _i64p), _p(rk, _i32p), _p(lk, _i32p),
                    _p(ln, _i32p), ef.shape[0], _p(ef, _i32p), _p(et, _i32p), rki.shape[0],
                    _p(rki, _i32p), _p(rt, _i32p), _p(rb, _i32p), _p(rwo, _i32p), _p(wr, _i32p),
                    _p(wk, _i32p), _p(wl, _i32p), g.window_start)


def orc_simulate(g: Graph, durations=None):
    """Plain-C restatement of simulate(); returns (status, start, fin, span)."""
    if durations is not None:
        g = Graph(**{**g.__dict__, "duration": np.ascontiguousarray(durations, np.int64)})
    keep = []
    og = orc_graph_struct(g, keep)
    start = np.zeros(g.n, np.int64)
    fin = np.zeros(g.n, np.int64)
    span = np.zeros(3, np.int64)
    rc = orc().orc_simulate(C.byref(og), _p(start, _i64p), _p(fin, _i64p), _p(span, _i64p))
    return rc, start, fin, span


def orc_breakdown_rank(g: Graph, start, fin, rank, wstart, wend):
    start = np.ascontiguousarray(start, np.int64)  # the C side reads dense arrays
    fin = np.ascontiguousarray(fin, np.int64)
    out = np.zeros(5, np.int64)
    orc().orc_breakdown_rank(g.n, _p(g.rank, _i32p), _p(g.lane_kind, _i32p),
                             _p(np.ascontiguousarray(g.is_comm()), _u8p), _p(start, _i64p),
                             _p(fin, _i64p), rank, wstart, wend, _p(out, _i64p))
    return tuple(int(x) for x in out)


def orc_durations(g: Graph, sc: OrcScenarios, scenario: int, cls=None):
    cls = g.default_scale_class() if cls is None else cls
    out = np.zeros(g.n, np.int64)
    orc().orc_fill_durations(C.byref(sc), scenario, g.n, _p(g.duration, _i64p), _p(cls, _u8p),
                             _p(out, _i64p))
    return out


def pipeline_spec_json(spec_json: str) -> dict:
    """The reference's pipeline_spec_for(SynthSpec::from_json(spec)) as JSON."""
    import json as _json
    lib = ref()
    lib.ref_pipeline_spec_json.restype = C.c_char_p
    lib.ref_pipeline_spec_json.argtypes = [C.c_char_p]
    out = lib.ref_pipeline_spec_json(spec_json.encode())
    if not out:
        raise RefError(1, lib.ref_last_error().decode())
    return _json.loads(out.decode())


def pipeline_events_json(pipeline: dict, hook=None):
    """build_pipeline(spec, hook) of a JSON PipelineSpec: (pid, tid, ts, dur, n_ops, end)."""
    import json as _json
    lib = ref()
    lib.ref_pipeline_events_json.restype = C.c_int64
    lib.ref_pipeline_events_json.argtypes = [C.c_char_p, _i64p, C.c_int64, _i32p, _i32p, _i64p,
                                             _i64p, C.c_int64, _i64p, _i64p]
    cap = 4_000_000
    pid = np.zeros(cap, np.int32)
    tid = np.zeros(cap, np.int32)
    ts = np.zeros(cap, np.int64)
    dur = np.zeros(cap, np.int64)
    nops = C.c_int64(0)
    end = C.c_int64(0)
    h = None if hook is None else np.ascontiguousarray(hook, np.int64)
    n = lib.ref_pipeline_events_json(_json.dumps(pipeline).encode(),
                                     None if h is None else _p(h, _i64p),
                                     0 if h is None else h.shape[0], _p(pid, _i32p),
                                     _p(tid, _i32p), _p(ts, _i64p), _p(dur, _i64p), cap,
                                     C.byref(nops), C.byref(end))
    if n < 0:
        raise RefError(1, lib.ref_last_error().decode())
    return pid[:n], tid[:n], ts[:n], dur[:n], int(nops.value), int(end.value)
