"""Host mirror of the reference replay interface, on the B200 engine.

Reference interface (``/root/reference/proj/include/tracesim/simulate.hpp``):

* ``simulate(const ExecutionGraph&) -> SimulatedTrace`` (``:51``): one replay at
  the graph's own durations; raises ``SimulationError`` on invalid graphs.
* ``validate_graph`` (``:37``) — the error checks run inside ``DeviceGraph``.

Batched extension (the data-parallel hot path): ``simulate_batch`` replays
``count`` duration scenarios of one graph at once — the reference equivalent
is ``count`` calls of ``simulate`` on perturbed copies (jitter hook
``synth.cpp:146-156``; class retime ``transform.cpp:38-43``).

Every call goes through the C ABI of ``lib/liblumos_b200.so``; there is no
CPU execution path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .graph import (DeviceError, ExecutionGraph, GraphError, SimulatedTrace, SimulationError,
                    UnsupportedGraphError)


def _raise(rc: int):
    msg = N.last_error()
    if rc == N.TS_E_SIMULATION:
        raise SimulationError(msg)
    if rc == N.TS_E_GRAPH:
        raise GraphError(msg)
    if rc == N.TS_E_UNSUPPORTED:
        raise UnsupportedGraphError(msg)
    if rc == N.TS_E_CUDA or rc == N.TS_E_NOMEM:
        raise DeviceError(msg)
    raise ValueError(msg)


_ITEM = {N.i64p: ("int64", 8), N.i32p: ("int32", 4), N.u8p: ("uint8", 1)}


def _ptr(a, t):
    """Raw pointer of a buffer the C ABI reads or writes as a dense row-major
    array of t's element type: strided views or other dtypes are rejected
    (the library would silently use the wrong layout)."""
    if a is None:
        return None
    name, size = _ITEM[t]
    if hasattr(a, "data_ptr"):  # torch tensor (device or host)
        if str(a.dtype) != f"torch.{name}" or not a.is_contiguous():
            raise ValueError(f"expected a contiguous torch.{name} tensor, got {a.dtype} "
                             f"(contiguous={a.is_contiguous()})")
        return C.cast(C.c_void_p(a.data_ptr()), t)
    if a.dtype != np.dtype(name) or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"expected a C-contiguous {name} array, got {a.dtype} "
                         f"(C_CONTIGUOUS={a.flags['C_CONTIGUOUS']})")
    return a.ctypes.data_as(t)


@dataclass
class ScenarioSpec:
    """A batch of duration scenarios (include/lumos_b200.h, ts_scenarios).

    jitter      u ~ U[-jitter, jitter): d -> max(1, llround(d * (1 + u))), 0 stays 0
    scale       per-class rational factor num / scale_den, num drawn in
                [scale_lo, scale_hi] (or given per scenario in ``scale_num``)
    durations   explicit [n_tasks][count] durations (overrides both)
    """
    count: int
    first: int = 0
    seed: int = 250409307
    jitter: float = 0.0
    scale_lo: int = 0
    scale_hi: int = 0
    scale_den: int = 0
    scale_num: Optional[object] = None  # [count][n_classes] int32 (numpy or torch)
    durations: Optional[object] = None  # [n_tasks][ld] int64
    durations_ld: int = 0
    retime: Optional["Retime"] = None   # per-scenario what-if retime (ts_retime)

    def to_c(self) -> N.TsScenarios:
        sc = N.TsScenarios()
        sc.first = self.first
        sc.count = self.count
        sc.seed = self.seed
        sc.jitter = self.jitter
        sc.scale_lo, sc.scale_hi, sc.scale_den = self.scale_lo, self.scale_hi, self.scale_den
        if self.scale_num is not None:
            sc.n_classes = int(self.scale_num.shape[1])
            sc.scale_num = _ptr(self.scale_num, N.i32p)
        if self.durations is not None:
            sc.durations = _ptr(self.durations, N.i64p)
            sc.durations_ld = self.durations_ld or int(self.durations.shape[1])
        if self.retime is not None:
            self._rt = self.retime.to_c(self.count)  # kept alive with the spec
            sc.retime = C.cast(C.pointer(self._rt), C.c_void_p)
        return sc


@dataclass
class Retime:
    """Device-side what-if retime per scenario (ts_retime): apply_whatif's
    non-structural width / data-parallel change (transform.cpp:713-760) —
    change_hidden then scale_dp with the analytical cost model alpha + bytes *
    scale / beta (cost.cpp:40-62).  Arrays are per scenario (host memory)."""
    alpha_us: object                      # [count] float64
    bytes_per_us: object                  # [count] float64
    source_dp: int = 1
    target_dp: Optional[object] = None    # [count] int32
    source_model: tuple = (0, 0, 0)       # (d_model, d_ffn, n_params)
    target_model: Optional[object] = None  # [count][3] int64

    def to_c(self, count: int) -> N.TsRetime:
        self._a = np.ascontiguousarray(np.broadcast_to(np.asarray(self.alpha_us, np.float64), (count,)))
        self._b = np.ascontiguousarray(np.broadcast_to(np.asarray(self.bytes_per_us, np.float64), (count,)))
        r = N.TsRetime()
        r.alpha_us = self._a.ctypes.data_as(C.POINTER(C.c_double))
        r.bytes_per_us = self._b.ctypes.data_as(C.POINTER(C.c_double))
        r.source_dp = int(self.source_dp)
        if self.target_dp is not None:
            self._t = np.ascontiguousarray(np.broadcast_to(np.asarray(self.target_dp, np.int32), (count,)))
            r.target_dp = self._t.ctypes.data_as(N.i32p)
        for k in range(3):
            r.source_model[k] = int(self.source_model[k])
        if self.target_model is not None:
            self._m = np.ascontiguousarray(
                np.broadcast_to(np.asarray(self.target_model, np.int64), (count, 3)))
            r.target_model = self._m.ctypes.data_as(N.i64p)
        return r


class DeviceGraph:
    """A compiled, device-resident ExecutionGraph (``ts_graph``).

    Construction runs validate_graph's error checks (raising SimulationError
    with the reference's message) and compiles the graph to replay programs.
    ``device=None`` uses the current CUDA device; ``compile_only=True`` builds
    host-side programs for inspection without touching a GPU.
    """

    def __init__(self, graph, device: Optional[int] = None, compile_only: bool = False):
        g = ExecutionGraph.from_any(graph)
        self.graph = g
        d = N.TsGraphDesc()
        d.n_tasks = g.n
        d.duration = _ptr(g.duration, N.i64p)
        d.original_start = _ptr(g.original_start, N.i64p)
        d.rank = _ptr(g.rank, N.i32p)
        d.lane_kind = _ptr(g.lane_kind, N.i32p)
        d.lane = _ptr(g.lane, N.i32p)
        d.op_class = _ptr(g.op_class, N.u8p)
        d.task_kind = _ptr(g.task_kind, N.u8p)
        d.scale_class = _ptr(g.scale_class, N.u8p) if g.scale_class is not None else None
        d.n_edges = g.edge_from.shape[0]
        d.edge_from = _ptr(g.edge_from, N.i32p)
        d.edge_to = _ptr(g.edge_to, N.i32p)
        d.n_rules = g.rule_kind.shape[0]
        d.rule_kind = _ptr(g.rule_kind, N.i32p)
        d.rule_task = _ptr(g.rule_task, N.i32p)
        d.rule_bound = _ptr(g.rule_bound, N.i32p)
        d.rule_watch_off = _ptr(g.rule_watch_off, N.i32p)
        d.watch_rank = _ptr(g.watch_rank, N.i32p)
        d.watch_kind = _ptr(g.watch_kind, N.i32p)
        d.watch_lane = _ptr(g.watch_lane, N.i32p)
        d.window_start = g.window_start
        d.window_end = g.window_end
        d.n_gates = g.gate_from.shape[0]
        d.gate_from = _ptr(g.gate_from, N.i32p)
        d.gate_to = _ptr(g.gate_to, N.i32p)
        d.gate_kind = _ptr(g.gate_kind, N.u8p)
        if g.rt_kind is not None:
            d.rt_kind = _ptr(g.rt_kind, N.u8p)
            d.rt_bytes = _ptr(g.rt_bytes, N.i64p) if g.rt_bytes is not None else None
            d.rt_group = _ptr(g.rt_group, N.i32p) if g.rt_group is not None else None
            d.rt_mnk = _ptr(g.rt_mnk, N.i64p) if g.rt_mnk is not None else None
        h = C.c_void_p()
        dev = N.DEVICE_NONE if compile_only else (-1 if device is None else int(device))
        rc = N.lib().ts_graph_create(C.byref(d), dev, C.byref(h))
        if rc != N.TS_OK:
            _raise(rc)
        self.h = h
        info = N.TsGraphInfo()
        N.lib().ts_graph_get_info(self.h, C.byref(info))
        self.info = {k: getattr(info, k) for k, _ in N.TsGraphInfo._fields_}
        self.n_tasks = info.n_tasks
        self.n_ranks = info.n_ranks
        self.n_streams = info.n_streams
        ranks = np.zeros(max(1, info.n_ranks), np.int32)
        N.lib().ts_graph_ranks(self.h, _ptr(ranks, N.i32p))
        self.ranks = ranks[:info.n_ranks]
        srank = np.zeros(max(1, info.n_streams), np.int32)
        slane = np.zeros(max(1, info.n_streams), np.int32)
        N.lib().ts_graph_streams(self.h, _ptr(srank, N.i32p), _ptr(slane, N.i32p))
        self.stream_rank = srank[:info.n_streams]
        self.stream_lane = slane[:info.n_streams]

    def close(self):
        if getattr(self, "h", None):
            N.lib().ts_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ API
    def simulate(self) -> SimulatedTrace:
        """simulate(const ExecutionGraph&) on the GPU (simulate.hpp:51)."""
        n = self.n_tasks
        start = np.zeros(max(1, n), np.int64)
        fin = np.zeros(max(1, n), np.int64)
        span = np.zeros(3, np.int64)
        rc = N.lib().ts_simulate(self.h, _ptr(start, N.i64p), _ptr(fin, N.i64p),
                                 _ptr(span, N.i64p))
        if rc != N.TS_OK:
            _raise(rc)
        return SimulatedTrace.from_task_arrays(start[:n], fin[:n], span)

    def replay_batch(self, spec: ScenarioSpec, start=None, fin=None, ld: int = 0, span=None,
                     rank_breakdown=None, stream_busy=None, status=None, stream=None,
                     util_bin_width: int = 0, util_covered=None, util_n_bins=None,
                     delta_abs_sum=None, delta_worst=None, n_fixups=None,
                     host_async: bool = False) -> None:
        """Raw ts_replay_batch: outputs are caller-owned numpy (host) or torch
        (device or host) buffers; see include/lumos_b200.h for shapes.  With
        host_async the host buffers are filled by copies that overlap the next
        call's kernels; wait() before reading them (pinned buffers, kept alive)."""
        sc = spec.to_c()
        r = N.TsResult()
        r.start = _ptr(start, N.i64p)
        r.fin = _ptr(fin, N.i64p)
        r.ld = ld or (int(start.shape[1]) if start is not None else
                      int(fin.shape[1]) if fin is not None else spec.count)
        r.span = _ptr(span, N.i64p)
        r.rank_breakdown = _ptr(rank_breakdown, N.i64p)
        r.stream_busy = _ptr(stream_busy, N.i64p)
        r.status = _ptr(status, N.i32p)
        r.util_bin_width = int(util_bin_width)
        r.util_max_bins = int(util_covered.shape[-1]) if util_covered is not None else 0
        r.util_covered = _ptr(util_covered, N.i64p)
        r.util_n_bins = _ptr(util_n_bins, N.i32p)
        r.delta_abs_sum = _ptr(delta_abs_sum, N.i64p)
        r.delta_worst = _ptr(delta_worst, N.i64p)
        # delta_worst: [count][worst_n][3] (a [count][3] buffer means worst_n = 1)
        r.delta_worst_n = int(delta_worst.shape[1]) if (delta_worst is not None and
                                                          len(delta_worst.shape) == 3) else 1
        r.n_fixups = _ptr(n_fixups, N.i32p)
        r.host_async = 1 if host_async else 0
        s = C.c_void_p(stream) if isinstance(stream, int) else stream
        rc = N.lib().ts_replay_batch(self.h, C.byref(sc), C.byref(r), s)
        if rc != N.TS_OK:
            _raise(rc)

    def wait(self) -> None:
        """Block until the host copies of host_async replay_batch calls have landed."""
        rc = N.lib().ts_graph_wait(self.h)
        if rc != N.TS_OK:
            _raise(rc)

    def profile(self, enable: bool = True) -> None:
        """Record CUDA events around every kernel this graph launches."""
        N.lib().ts_profile_enable(self.h, 1 if enable else 0)

    def profile_read(self) -> dict:
        """Accumulated device milliseconds per kernel class since the last read."""
        st = N.TsProfileStats()
        rc = N.lib().ts_profile_read(self.h, C.byref(st))
        if rc != N.TS_OK:
            _raise(rc)
        return {k: getattr(st, k) for k, _ in N.TsProfileStats._fields_}

    def scenario_durations(self, spec: ScenarioSpec, out=None, stream=None):
        """Materialise scenario durations [n_tasks][count] (the K4 kernel alone)."""
        if out is None:
            out = np.zeros((self.n_tasks, spec.count), np.int64)
        sc = spec.to_c()
        s = C.c_void_p(stream) if isinstance(stream, int) else stream
        rc = N.lib().ts_scenario_durations(self.h, C.byref(sc), _ptr(out, N.i64p),
                                           int(out.shape[1]), s)
        if rc != N.TS_OK:
            _raise(rc)
        return out


@dataclass
class BatchResult:
    span: np.ndarray                  # [count][3] {start, end, makespan}
    start: Optional[np.ndarray]       # [n_tasks][count]
    fin: Optional[np.ndarray]
    rank_breakdown: Optional[np.ndarray]  # [count][n_ranks][5]
    stream_busy: Optional[np.ndarray]     # [count][n_streams]
    util_bin_width: int = 0
    util_covered: Optional[np.ndarray] = None  # [count][n_ranks][max_bins] covered us
    util_n_bins: Optional[np.ndarray] = None   # [count] bins of each scenario's window
    delta_abs_sum: Optional[np.ndarray] = None  # [count] sum |sim_start - original_start|
    delta_worst: Optional[np.ndarray] = None    # [count][worst_n][3] {|delta|, task, delta}
    n_fixups: int = 0                           # scenarios re-run by the event-driven path

    @property
    def makespan(self) -> np.ndarray:
        return self.span[:, 2]

    def utilization(self, s: int, window_start: int, window_end: int) -> np.ndarray:
        """utilization_by_rank values of scenario s (metrics.cpp:145-150):
        covered / bin span, the last bin normalised by its actual span.
        window = [window_start, max(window_end, window_start + makespan))."""
        w = self.util_bin_width
        end = max(window_end, window_start + int(self.span[s, 2]))
        nb_kept = int(self.util_n_bins[s])
        spans = np.minimum(w, end - (window_start + w * np.arange(nb_kept, dtype=np.int64)))
        return self.util_covered[s, :, :nb_kept] / spans

    def trace(self, s: int) -> SimulatedTrace:
        """Scenario s as a SimulatedTrace (needs a batch run with timestamps)."""
        if self.start is None or self.fin is None:
            raise ValueError("trace() needs a batch run with timestamps=True")
        return SimulatedTrace.from_task_arrays(self.start[:, s], self.fin[:, s], self.span[s])

    def chrome_trace(self, graph, s: int) -> str:
        """Scenario s as Chrome trace-event JSON for visual audit, in the layout
        of chrome_json / simulated_to_chrome_json (trace_parse.cpp:230-256,
        simulate.cpp:349-382): one "X" event per task, kernels on their stream.
        Names come from graph.names when present; args carry the stream only
        (the C++ drop-in's simulated_to_chrome_json also emits Task.meta)."""
        import json
        g = graph if isinstance(graph, ExecutionGraph) else ExecutionGraph.from_any(graph)
        tr = self.trace(s)
        out = ['{"schema_version":1,"traceEvents":[']
        first = True
        for tid, a, b in zip(tr.task_id.tolist(), tr.sim_start.tolist(), tr.sim_end.tolist()):
            gpu = int(g.task_kind[tid]) == 1
            cat = "kernel" if gpu else ("cuda_runtime" if int(g.op_class[tid]) in (2, 3, 4, 5)
                                        else "cpu_op")
            ev = {"name": g.names[tid] if g.names else f"task{tid}", "cat": cat, "ph": "X",
                  "ts": a, "dur": b - a, "pid": int(g.rank[tid]), "tid": int(g.lane[tid])}
            if gpu:
                ev["args"] = {"stream": int(g.lane[tid])}
            out.append(("" if first else ",") + json.dumps(ev, separators=(",", ":")) + "\n")
            first = False
        out.append("]}\n")
        return "".join(out)

    def replay_report(self, s: int, n_tasks: int, reference_makespan: int) -> dict:
        """compare_replay fields of scenario s (metrics.cpp:189-221); the worst
        list has the batch's worst_n entries (largest |delta| first, ties by
        task id)."""
        if self.delta_abs_sum is None or self.delta_worst is None:
            raise ValueError("replay_report needs a batch run with deltas=True")
        sim = int(self.span[s, 2])
        zero = reference_makespan == 0
        w = self.delta_worst[s].reshape(-1, 3)
        return {"reference_makespan": reference_makespan, "simulated_makespan": sim,
                "relative_error": 0.0 if zero else abs(sim - reference_makespan) / reference_makespan,
                "zero_reference": zero,
                "mean_abs_delta": 0.0 if n_tasks == 0 else float(self.delta_abs_sum[s]) / n_tasks,
                "max_abs_delta": int(w[0, 0]),
                "worst": [{"task": int(t), "delta": int(d)} for _, t, d in w.tolist() if t >= 0]}


def simulate(graph, device: Optional[int] = None) -> SimulatedTrace:
    """Drop-in for ``tracesim::simulate`` (simulate.hpp:51), executed on the GPU."""
    dg = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device)
    return dg.simulate()


def simulate_batch(graph, spec: ScenarioSpec, timestamps: bool = True, breakdown: bool = True,
                   device: Optional[int] = None, util_bin_width: int = 0,
                   util_max_bins: int = 0, deltas: bool = False,
                   worst_n: int = 10) -> BatchResult:
    """Replay ``spec.count`` scenarios; results in host numpy arrays.
    util_bin_width > 0 adds utilization_by_rank bins (every bin of every
    window; util_max_bins > 0 caps them and fails if a window needs more);
    deltas adds the compare_replay statistics with a worst_n-entry worst list
    (compare_replay's default 10, metrics.hpp:82-83)."""
    dg = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device)
    if util_bin_width > 0 and util_max_bins <= 0:
        # every bin: the graph's window, or the device tells how many it needs
        w0 = max(1, -(-(dg.info["window_end"] - dg.info["window_start"]) // util_bin_width))
        try:
            return simulate_batch(dg, spec, timestamps, breakdown, device, util_bin_width, w0,
                                  deltas, worst_n)
        except ValueError as e:
            import re
            m = re.search(r"utilization needs (\d+) bins", str(e))
            if not m:
                raise
            return simulate_batch(dg, spec, timestamps, breakdown, device, util_bin_width,
                                  int(m.group(1)), deltas, worst_n)
    S = spec.count
    span = np.zeros((S, 3), np.int64)
    start = fin = bd = busy = util = nbins = dsum = dworst = None
    if timestamps:
        start = np.zeros((dg.n_tasks, S), np.int64)
        fin = np.zeros((dg.n_tasks, S), np.int64)
    if breakdown:
        bd = np.zeros((S, dg.n_ranks, 5), np.int64)
        busy = np.zeros((S, max(1, dg.n_streams)), np.int64)
    if util_bin_width > 0:
        util = np.zeros((S, max(1, dg.n_ranks), max(1, util_max_bins)), np.int64)
        nbins = np.zeros(S, np.int32)
    if deltas:
        dsum = np.zeros(S, np.int64)
        dworst = np.zeros((S, max(1, worst_n), 3), np.int64)
    nfix = np.zeros(1, np.int32)
    dg.replay_batch(spec, start=start, fin=fin, ld=S, span=span, rank_breakdown=bd,
                    stream_busy=busy, util_bin_width=util_bin_width, util_covered=util,
                    util_n_bins=nbins, delta_abs_sum=dsum, delta_worst=dworst, n_fixups=nfix)
    return BatchResult(span=span, start=start, fin=fin, rank_breakdown=bd, stream_busy=busy,
                       util_bin_width=util_bin_width, util_covered=util, util_n_bins=nbins,
                       delta_abs_sum=dsum, delta_worst=dworst, n_fixups=int(nfix[0]))
