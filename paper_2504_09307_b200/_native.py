"""ctypes binding of ``lib/liblumos_b200.so`` (the C ABI in include/lumos_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2504_09307_b200/csrc``).  There is no fallback: if the shared
object is missing, importing the replay API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LUMOS_B200_LIB") or os.path.join(HERE, "lib", "liblumos_b200.so")

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)

TS_OK = 0
TS_E_INVALID_ARGUMENT = 1
TS_E_SIMULATION = 3
TS_E_GRAPH = 4
TS_E_UNSUPPORTED = 6
TS_E_CUDA = 7
TS_E_NOMEM = 8
DEVICE_NONE = -2  # compile only


class TsGraphDesc(C.Structure):
    _fields_ = [("n_tasks", C.c_int32), ("duration", i64p), ("original_start", i64p),
                ("rank", i32p), ("lane_kind", i32p), ("lane", i32p), ("op_class", u8p),
                ("task_kind", u8p), ("scale_class", u8p), ("n_edges", C.c_int64),
                ("edge_from", i32p), ("edge_to", i32p), ("n_rules", C.c_int32),
                ("rule_kind", i32p), ("rule_task", i32p), ("rule_bound", i32p),
                ("rule_watch_off", i32p), ("watch_rank", i32p), ("watch_kind", i32p),
                ("watch_lane", i32p), ("window_start", C.c_int64), ("window_end", C.c_int64),
                ("n_gates", C.c_int64), ("gate_from", i32p), ("gate_to", i32p),
                ("gate_kind", u8p), ("rt_kind", u8p), ("rt_bytes", i64p), ("rt_group", i32p),
                ("rt_mnk", i64p)]


class TsGraphInfo(C.Structure):
    _fields_ = [("n_tasks", C.c_int32), ("n_components", C.c_int32), ("n_programs", C.c_int32),
                ("n_ranks", C.c_int32), ("n_streams", C.c_int32), ("max_slots", C.c_int32),
                ("program_bytes", C.c_int64), ("n_ops", C.c_int64), ("n_syncs", C.c_int32),
                ("n_gpu_tasks", C.c_int32), ("window_start", C.c_int64),
                ("window_end", C.c_int64), ("n_fused_ranks", C.c_int32), ("des_only", C.c_int32),
                ("n_candidates", C.c_int64)]


class TsScenarios(C.Structure):
    _fields_ = [("first", C.c_int64), ("count", C.c_int32), ("flags", C.c_int32),
                ("seed", C.c_uint64), ("jitter", C.c_double), ("scale_lo", C.c_int32),
                ("scale_hi", C.c_int32), ("scale_den", C.c_int32), ("n_classes", C.c_int32),
                ("scale_num", i32p), ("durations", i64p), ("durations_ld", C.c_int64),
                ("retime", C.c_void_p)]


class TsRetime(C.Structure):
    _fields_ = [("alpha_us", C.POINTER(C.c_double)), ("bytes_per_us", C.POINTER(C.c_double)),
                ("source_dp", C.c_int32), ("pad", C.c_int32), ("target_dp", i32p),
                ("source_model", C.c_int64 * 3), ("target_model", i64p)]


class TsProfileStats(C.Structure):
    _fields_ = [("walk_ms", C.c_double), ("walk_launches", C.c_int64), ("reduce_ms", C.c_double),
                ("reduce_launches", C.c_int64), ("other_ms", C.c_double),
                ("other_launches", C.c_int64)]


class TsResult(C.Structure):
    _fields_ = [("start", i64p), ("fin", i64p), ("ld", C.c_int64), ("span", i64p),
                ("rank_breakdown", i64p), ("stream_busy", i64p), ("status", i32p),
                ("util_bin_width", C.c_int64), ("util_max_bins", C.c_int32),
                ("util_pad", C.c_int32), ("util_covered", i64p), ("util_n_bins", i32p),
                ("delta_abs_sum", i64p), ("delta_worst", i64p), ("delta_worst_n", C.c_int32),
                ("host_async", C.c_int32), ("n_fixups", i32p)]


ABI_VERSION = 5  # TS_ABI_VERSION in include/lumos_b200.h
_lib = None


def lib():
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.ts_abi_version.restype = C.c_int
        L.ts_last_error.restype = C.c_char_p
        L.ts_kernel_launches.restype = C.c_int64
        L.ts_graph_create.restype = C.c_int
        L.ts_graph_create.argtypes = [C.POINTER(TsGraphDesc), C.c_int, C.POINTER(C.c_void_p)]
        L.ts_graph_destroy.argtypes = [C.c_void_p]
        L.ts_graph_get_info.restype = C.c_int
        L.ts_graph_get_info.argtypes = [C.c_void_p, C.POINTER(TsGraphInfo)]
        L.ts_graph_ranks.restype = C.c_int
        L.ts_graph_ranks.argtypes = [C.c_void_p, i32p]
        L.ts_graph_streams.restype = C.c_int
        L.ts_graph_streams.argtypes = [C.c_void_p, i32p, i32p]
        L.ts_replay_batch.restype = C.c_int
        L.ts_replay_batch.argtypes = [C.c_void_p, C.POINTER(TsScenarios), C.POINTER(TsResult),
                                      C.c_void_p]
        L.ts_graph_wait.restype = C.c_int
        L.ts_graph_wait.argtypes = [C.c_void_p]
        L.ts_simulate.restype = C.c_int
        L.ts_simulate.argtypes = [C.c_void_p, i64p, i64p, i64p]
        L.ts_scenario_durations.restype = C.c_int
        L.ts_scenario_durations.argtypes = [C.c_void_p, C.POINTER(TsScenarios), i64p, C.c_int64,
                                            C.c_void_p]
        L.ts_walk_counts.restype = C.c_int
        L.ts_walk_counts.argtypes = [i64p]
        L.ts_profile_enable.restype = C.c_int
        L.ts_profile_enable.argtypes = [C.c_void_p, C.c_int]
        L.ts_profile_read.restype = C.c_int
        L.ts_profile_read.argtypes = [C.c_void_p, C.POINTER(TsProfileStats)]
        if L.ts_abi_version() != ABI_VERSION:
            raise RuntimeError("liblumos_b200.so ABI mismatch")
        _lib = L
    return _lib


def walk_counts() -> list:
    """K1 walk launches per variant: [1/thread u32, 1/thread i64, 2/thread u32,
    2/thread i64, cluster walk (estimate mode)]."""
    out = (C.c_int64 * 5)()
    lib().ts_walk_counts(out)
    return list(out)


def last_error() -> str:
    return lib().ts_last_error().decode()


EXPORTED = ["ts_abi_version", "ts_last_error", "ts_kernel_launches", "ts_graph_create",
            "ts_graph_destroy", "ts_graph_get_info", "ts_graph_ranks", "ts_graph_streams",
            "ts_replay_batch", "ts_simulate", "ts_walk_counts", "ts_scenario_durations", "ts_profile_enable",
            "ts_profile_read", "ts_synth_defaults", "ts_synth_graph", "ts_host_graph_desc",
            "ts_host_graph_op_index", "ts_host_graph_n_ops", "ts_host_graph_name_ids",
            "ts_host_graph_name", "ts_host_graph_free", "ts_build_rank_graph",
            "ts_ingest_traces", "ts_ingest_traces_ex", "ts_pipeline_defaults", "ts_pipeline_graph",
            "ts_rebuild_pipeline", "ts_pipeline_spec_get", "ts_pipeline_free", "ts_graph_wait"]
