"""B200-native batched replay and what-if estimation engine for Lumos (arXiv 2504.09307).

Drop-in for the reference ``tracesim`` simulation path: the graph model
(:mod:`.graph`), the replay API (:mod:`.replay`), the synthetic GPT trace
generator and graph builder (:mod:`.synth`), the PipelineSpec / estimate()
boundary (:mod:`.pipeline`), all over the C ABI of
``lib/liblumos_b200.so`` (include/lumos_b200.h).
"""
from .graph import (COMMUNICATION, COMPUTE, CPU_THREAD, CUDA_STREAM, DEVICE_SYNC, EVENT_SYNC,
                    STREAM_SYNC, DeviceError, ExecutionGraph, GraphError, SimulatedTrace,
                    SimulationError, UnsupportedGraphError)
from .replay import BatchResult, DeviceGraph, Retime, ScenarioSpec, simulate, simulate_batch
from .pipeline import (KernelSpec, ModelConfig, ParallelismConfig, PipelineSpec, StageSpec,
                       WhatIfConfig, estimate_batch, estimate_whatif, pipeline_graph,
                       rebuild_pipeline)

__all__ = [
    "Retime",
    "ExecutionGraph", "SimulatedTrace", "SimulationError", "GraphError", "UnsupportedGraphError",
    "DeviceError", "DeviceGraph", "ScenarioSpec", "BatchResult", "simulate", "simulate_batch",
    "CPU_THREAD", "CUDA_STREAM", "STREAM_SYNC", "DEVICE_SYNC", "EVENT_SYNC", "COMPUTE",
    "COMMUNICATION", "KernelSpec", "StageSpec", "PipelineSpec", "pipeline_graph",
    "estimate_batch", "ModelConfig", "ParallelismConfig", "WhatIfConfig", "rebuild_pipeline",
    "estimate_whatif",
]
