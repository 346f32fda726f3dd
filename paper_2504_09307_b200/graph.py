"""ExecutionGraph as structure-of-arrays, and the reference's error taxonomy.

Mirrors ``tracesim::ExecutionGraph`` (reference ``include/tracesim/build.hpp:73-85``)
with the fields the replay path reads: per task its duration, recorded start
(the dispatch tie-break key, ``simulate.cpp:127-139``), processor
``(rank, lane_kind, lane)`` (``types.hpp:48-54``), op class and kind; the fixed
finish->start edges; the runtime sync rules (``build.hpp:46-54``); and the
iteration window.  Optional *gates* carry the generator/estimate() barrier and
rendezvous semantics (``pipeline.cpp:377-389``).
"""
from __future__ import annotations

from dataclasses import dataclass, field, fields
from typing import Optional

import numpy as np

# enums (types.hpp:29-41, build.hpp:47)
CPU_THREAD, CUDA_STREAM = 0, 1
STREAM_SYNC, DEVICE_SYNC, EVENT_SYNC = 0, 1, 2
COMPUTE, COMMUNICATION, LAUNCH, SYNC, EVENT_RECORD, EVENT_WAIT, OTHER = range(7)
GATE_FIN, GATE_START = 0, 1


class SimulationError(RuntimeError):
    """tracesim::SimulationError (types.hpp:124-127): invalid graph or deadlock."""


class GraphError(RuntimeError):
    """tracesim::GraphError (types.hpp:119-122): dependency cycle."""


class UnsupportedGraphError(RuntimeError):
    """The graph lies outside the device path's class (e.g. unchained lanes)."""


class DeviceError(RuntimeError):
    """No CUDA device or a CUDA runtime failure (there is no CPU path)."""


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


@dataclass
class ExecutionGraph:
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
    gate_from: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    gate_to: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    gate_kind: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    scale_class: Optional[np.ndarray] = None
    names: list = field(default_factory=list)
    # retime metadata (ts_graph_desc.rt_*; TS_RT_* classes of Task.meta), or None
    rt_kind: Optional[np.ndarray] = None   # [n] uint8
    rt_bytes: Optional[np.ndarray] = None  # [n] int64 (-1: no byte count)
    rt_group: Optional[np.ndarray] = None  # [n] int32
    rt_mnk: Optional[np.ndarray] = None    # [n][3] int64

    def __post_init__(self):
        self.duration = _i64(self.duration)
        self.original_start = _i64(self.original_start)
        self.rank = _i32(self.rank)
        self.lane_kind = _i32(self.lane_kind)
        self.lane = _i32(self.lane)
        self.op_class = _u8(self.op_class)
        self.task_kind = _u8(self.task_kind)
        self.edge_from = _i32(self.edge_from)
        self.edge_to = _i32(self.edge_to)
        self.rule_kind = _i32(self.rule_kind)
        self.rule_task = _i32(self.rule_task)
        self.rule_bound = _i32(self.rule_bound)
        self.rule_watch_off = _i32(self.rule_watch_off)
        if self.rule_watch_off.shape[0] == 0:
            self.rule_watch_off = np.zeros(1, np.int32)
        self.watch_rank = _i32(self.watch_rank)
        self.watch_kind = _i32(self.watch_kind)
        self.watch_lane = _i32(self.watch_lane)
        self.gate_from = _i32(self.gate_from)
        self.gate_to = _i32(self.gate_to)
        self.gate_kind = _u8(self.gate_kind)
        if self.scale_class is not None:
            self.scale_class = _u8(self.scale_class)
        if self.rt_kind is not None:
            self.rt_kind = _u8(self.rt_kind)
            n = self.rt_kind.shape[0]
            self.rt_bytes = (_i64(self.rt_bytes) if self.rt_bytes is not None
                             else np.zeros(n, np.int64))
            self.rt_group = (_i32(self.rt_group) if self.rt_group is not None
                             else np.zeros(n, np.int32))
            self.rt_mnk = (np.ascontiguousarray(self.rt_mnk, np.int64).reshape(n, 3)
                           if self.rt_mnk is not None else np.zeros((n, 3), np.int64))
        self.window_start = int(self.window_start)
        self.window_end = int(self.window_end)

    @property
    def n(self) -> int:
        return int(self.duration.shape[0])

    @classmethod
    def from_any(cls, g) -> "ExecutionGraph":
        """Accept any object with the same field names (e.g. a test fixture)."""
        if isinstance(g, ExecutionGraph):
            return g
        kw = {f.name: getattr(g, f.name) for f in fields(cls) if hasattr(g, f.name)}
        return cls(**kw)

    def with_durations(self, duration) -> "ExecutionGraph":
        kw = {f.name: getattr(self, f.name) for f in fields(self)}
        kw["duration"] = duration
        return ExecutionGraph(**kw)

    def default_scale_class(self) -> np.ndarray:
        """0 host task, 1 GPU compute, 2 GPU communication (include/lumos_b200.h)."""
        cls = np.zeros(self.n, np.uint8)
        gpu = self.task_kind == 1
        cls[gpu] = 1
        cls[gpu & (self.op_class == COMMUNICATION)] = 2
        return cls

    def ranks(self) -> list:
        """ranks_in (build.cpp:582-590)."""
        return sorted(set(int(r) for r in np.unique(self.rank)))


@dataclass
class SimulatedTrace:
    """tracesim::SimulatedTrace (simulate.hpp:19-24): entries sorted by (sim_start, task_id)."""
    task_id: np.ndarray
    sim_start: np.ndarray
    sim_end: np.ndarray
    start: int
    end: int
    makespan: int

    @property
    def entries(self):
        return list(zip(self.task_id.tolist(), self.sim_start.tolist(), self.sim_end.tolist()))

    @classmethod
    def from_task_arrays(cls, start: np.ndarray, fin: np.ndarray, span) -> "SimulatedTrace":
        ids = np.arange(start.shape[0], dtype=np.int32)
        order = np.lexsort((ids, start))
        return cls(task_id=ids[order], sim_start=start[order], sim_end=fin[order],
                   start=int(span[0]), end=int(span[1]), makespan=int(span[2]))
