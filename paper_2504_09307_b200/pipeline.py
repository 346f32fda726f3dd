"""Mode-B boundary: the reference's PipelineSpec on the B200 engine.

Mirrors ``tracesim::KernelSpec`` / ``StageSpec`` / ``PipelineSpec``
(reference ``include/tracesim/pipeline.hpp:27-70``).  ``pipeline_graph``
turns a spec into the graph of ``build_pipeline(spec, DurationHook)``
(``pipeline.cpp:474-477``) — with ``estimate=True`` the generator's own
dependency graph with its p2p rendezvous / collective-barrier gates, i.e. what
``estimate()`` (``apply_whatif`` -> ``rebuild_pipeline``, ``transform.cpp:
556-731``) replays — and ``estimate_batch`` replays it for a batch of duration
scenarios on the GPU.  A scenario's durations play the DurationHook: task t
of the graph is hook slot ``op_index[t]`` (launch = two slots, negative -> 0).
Everything goes through the C ABI (``ts_pipeline_graph``); there is no CPU path.

``rebuild_pipeline`` / ``estimate_whatif`` add the structural what-if host
step (``ts_rebuild_pipeline``: tag_tasks + measure_pipeline + rebuild_pipeline,
transform.cpp:71-701) so a measured trace can be estimated at a new PP / DP /
microbatch count / depth / width.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from . import _native as N
from .synth import SynthGraph, _from_host, _lib


class TsKernelSpec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("duration", C.c_int64), ("op_class", C.c_int32),
                ("n_args", C.c_int32), ("arg_keys", C.POINTER(C.c_char_p)),
                ("arg_values", C.POINTER(C.c_char_p))]


class TsKernelList(C.Structure):
    _fields_ = [("k", C.POINTER(TsKernelSpec)), ("n", C.c_int32), ("pad", C.c_int32)]


class TsStageSpec(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("pad", C.c_int32),
                ("layers_fwd", C.POINTER(TsKernelList)), ("layers_bwd", C.POINTER(TsKernelList)),
                ("pre_fwd", TsKernelList), ("post_fwd", TsKernelList), ("pre_bwd", TsKernelList),
                ("post_bwd", TsKernelList), ("reduce", TsKernelList), ("optimizer", TsKernelList)]


class TsPipelineSpec(C.Structure):
    _fields_ = [("pp", C.c_int32), ("dp", C.c_int32), ("num_microbatches", C.c_int32),
                ("n_stages", C.c_int32), ("stages", C.POINTER(TsStageSpec)),
                ("launch_us", C.c_int64), ("record_us", C.c_int64), ("wait_us", C.c_int64),
                ("sync_us", C.c_int64), ("p2p_send_us", C.c_int64),
                ("p2p_recv_base_us", C.c_int64), ("activation_bytes", C.c_int64),
                ("origin", C.c_int64), ("compute_stream", C.c_int32),
                ("reduce_stream", C.c_int32), ("p2p_stream", C.c_int32),
                ("main_thread", C.c_int32), ("helper_thread", C.c_int32), ("pad", C.c_int32),
                ("first_event", C.c_int64), ("first_correlation", C.c_int64)]


@dataclass
class KernelSpec:
    """KernelSpec (pipeline.hpp:27-32)."""
    name: str
    duration: int = 0
    op_class: int = 0                       # OpClass (informational: kernels classify by name)
    args: Dict[str, str] = field(default_factory=dict)


@dataclass
class StageSpec:
    """StageSpec (pipeline.hpp:34-43)."""
    layers_fwd: List[List[KernelSpec]] = field(default_factory=list)
    layers_bwd: List[List[KernelSpec]] = field(default_factory=list)
    pre_fwd: List[KernelSpec] = field(default_factory=list)
    post_fwd: List[KernelSpec] = field(default_factory=list)
    pre_bwd: List[KernelSpec] = field(default_factory=list)
    post_bwd: List[KernelSpec] = field(default_factory=list)
    reduce: List[KernelSpec] = field(default_factory=list)
    optimizer: List[KernelSpec] = field(default_factory=list)


@dataclass
class PipelineSpec:
    """PipelineSpec (pipeline.hpp:45-70) with HostCosts flattened."""
    pp: int = 1
    dp: int = 1
    num_microbatches: int = 1
    stages: List[StageSpec] = field(default_factory=list)
    launch: int = 5
    record: int = 2
    wait: int = 2
    sync: int = 5
    p2p_send: int = 0
    p2p_recv_base: int = 0
    activation_bytes: int = 0
    origin: int = 0
    compute_stream: int = 7
    reduce_stream: int = 9
    p2p_stream: int = 11
    main_thread: int = 100
    helper_thread: int = 200
    first_event: int = 1
    first_correlation: int = 1

    @staticmethod
    def from_json(d: dict) -> "PipelineSpec":
        """From the JSON layout tests/refshim's ref_pipeline_spec_json emits."""
        ks = lambda a: [KernelSpec(k["name"], int(k["duration"]), int(k.get("op_class", 0)),
                                   dict(k.get("args", {}))) for k in a]
        stages = [StageSpec(layers_fwd=[ks(l) for l in s["layers_fwd"]],
                            layers_bwd=[ks(l) for l in s["layers_bwd"]],
                            pre_fwd=ks(s["pre_fwd"]), post_fwd=ks(s["post_fwd"]),
                            pre_bwd=ks(s["pre_bwd"]), post_bwd=ks(s["post_bwd"]),
                            reduce=ks(s["reduce"]), optimizer=ks(s["optimizer"]))
                  for s in d["stages"]]
        kw = {k: int(d[k]) for k in ("pp", "dp", "num_microbatches", "launch", "record", "wait",
                                     "sync", "p2p_send", "p2p_recv_base", "activation_bytes",
                                     "origin", "compute_stream", "reduce_stream", "p2p_stream",
                                     "main_thread", "helper_thread", "first_event",
                                     "first_correlation")}
        return PipelineSpec(stages=stages, **kw)

    def to_json(self) -> dict:
        kj = lambda a: [{"name": k.name, "duration": k.duration, "op_class": k.op_class,
                         "args": dict(k.args)} for k in a]
        d = {k: getattr(self, k) for k in ("pp", "dp", "num_microbatches", "launch", "record",
                                           "wait", "sync", "p2p_send", "p2p_recv_base",
                                           "activation_bytes", "origin", "compute_stream",
                                           "reduce_stream", "p2p_stream", "main_thread",
                                           "helper_thread", "first_event", "first_correlation")}
        d["stages"] = [{"layers_fwd": [kj(l) for l in s.layers_fwd],
                        "layers_bwd": [kj(l) for l in s.layers_bwd],
                        "pre_fwd": kj(s.pre_fwd), "post_fwd": kj(s.post_fwd),
                        "pre_bwd": kj(s.pre_bwd), "post_bwd": kj(s.post_bwd),
                        "reduce": kj(s.reduce), "optimizer": kj(s.optimizer)}
                       for s in self.stages]
        return d

    def to_c(self) -> TsPipelineSpec:
        """The ts_pipeline_spec POD; its buffers live on the returned struct."""
        keep = []

        def klist(kernels):
            arr = (TsKernelSpec * max(1, len(kernels)))()
            for i, k in enumerate(kernels):
                keys = [s.encode() for s in k.args]
                vals = [str(v).encode() for v in k.args.values()]
                ka = (C.c_char_p * max(1, len(keys)))(*keys)
                va = (C.c_char_p * max(1, len(vals)))(*vals)
                nm = k.name.encode()
                keep.extend([ka, va, nm])
                arr[i] = TsKernelSpec(nm, int(k.duration), int(k.op_class), len(keys), ka, va)
            keep.append(arr)
            return TsKernelList(arr, len(kernels), 0)

        stages = (TsStageSpec * max(1, len(self.stages)))()
        for i, s in enumerate(self.stages):
            nl = len(s.layers_fwd)
            if len(s.layers_bwd) != nl:
                raise ValueError("layers_fwd and layers_bwd need one entry per layer")
            lf = (TsKernelList * max(1, nl))(*[klist(l) for l in s.layers_fwd])
            lb = (TsKernelList * max(1, nl))(*[klist(l) for l in s.layers_bwd])
            keep.extend([lf, lb])
            stages[i] = TsStageSpec(nl, 0, lf, lb, klist(s.pre_fwd), klist(s.post_fwd),
                                    klist(s.pre_bwd), klist(s.post_bwd), klist(s.reduce),
                                    klist(s.optimizer))
        keep.append(stages)
        c = TsPipelineSpec(self.pp, self.dp, self.num_microbatches, len(self.stages), stages,
                           self.launch, self.record, self.wait, self.sync, self.p2p_send,
                           self.p2p_recv_base, self.activation_bytes, self.origin,
                           self.compute_stream, self.reduce_stream, self.p2p_stream,
                           self.main_thread, self.helper_thread, 0, self.first_event,
                           self.first_correlation)
        c._keep = keep
        return c


    @staticmethod
    def from_c(c: TsPipelineSpec) -> "PipelineSpec":
        """From the ts_pipeline_spec POD (e.g. ts_rebuild_pipeline's result)."""
        def kl(lst):
            out = []
            for i in range(lst.n):
                k = lst.k[i]
                args = {k.arg_keys[a].decode(): k.arg_values[a].decode() for a in range(k.n_args)}
                out.append(KernelSpec(k.name.decode(), int(k.duration), int(k.op_class), args))
            return out
        stages = []
        for s in range(c.n_stages):
            st = c.stages[s]
            stages.append(StageSpec(layers_fwd=[kl(st.layers_fwd[l]) for l in range(st.n_layers)],
                                    layers_bwd=[kl(st.layers_bwd[l]) for l in range(st.n_layers)],
                                    pre_fwd=kl(st.pre_fwd), post_fwd=kl(st.post_fwd),
                                    pre_bwd=kl(st.pre_bwd), post_bwd=kl(st.post_bwd),
                                    reduce=kl(st.reduce), optimizer=kl(st.optimizer)))
        return PipelineSpec(pp=c.pp, dp=c.dp, num_microbatches=c.num_microbatches, stages=stages,
                            launch=c.launch_us, record=c.record_us, wait=c.wait_us,
                            sync=c.sync_us, p2p_send=c.p2p_send_us,
                            p2p_recv_base=c.p2p_recv_base_us,
                            activation_bytes=c.activation_bytes, origin=c.origin,
                            compute_stream=c.compute_stream, reduce_stream=c.reduce_stream,
                            p2p_stream=c.p2p_stream, main_thread=c.main_thread,
                            helper_thread=c.helper_thread, first_event=c.first_event,
                            first_correlation=c.first_correlation)


# ------------------------------------------------------ structural what-if
class TsModelConfig(C.Structure):
    _fields_ = [("n_params", C.c_int64), ("n_layers", C.c_int32), ("d_model", C.c_int32),
                ("d_ffn", C.c_int32), ("n_heads", C.c_int32), ("d_head", C.c_int32),
                ("pad", C.c_int32)]


class TsParConfig(C.Structure):
    _fields_ = [("tp", C.c_int32), ("pp", C.c_int32), ("dp", C.c_int32),
                ("num_microbatches", C.c_int32)]


class TsWhatIf(C.Structure):
    _fields_ = [("source_model", TsModelConfig), ("target_model", TsModelConfig),
                ("source_par", TsParConfig), ("target_par", TsParConfig),
                ("alpha_us", C.c_double), ("bytes_per_us", C.c_double),
                ("activation_bytes", C.c_int64), ("tag_policy_json", C.c_char_p)]


@dataclass
class ModelConfig:
    """ModelConfig (types.hpp:89-96)."""
    n_layers: int
    d_model: int
    d_ffn: int
    n_heads: int
    d_head: int
    n_params: int = 0

    def to_c(self) -> TsModelConfig:
        return TsModelConfig(self.n_params, self.n_layers, self.d_model, self.d_ffn,
                             self.n_heads, self.d_head, 0)


@dataclass
class ParallelismConfig:
    """ParallelismConfig (types.hpp:98-103)."""
    tp: int = 1
    pp: int = 1
    dp: int = 1
    num_microbatches: int = 1

    def to_c(self) -> TsParConfig:
        return TsParConfig(self.tp, self.pp, self.dp, self.num_microbatches)


@dataclass
class WhatIfConfig:
    """WhatIfConfig (transform.hpp:28-41) with an AnalyticalCostModel."""
    source_model: ModelConfig
    target_model: ModelConfig
    source_par: ParallelismConfig
    target_par: ParallelismConfig
    alpha_us: float = 10.0
    bytes_per_us: float = 50000.0
    activation_bytes: int = 0
    tag_policy: Optional[dict] = None       # TagPolicy::from_json document

    def to_c(self) -> TsWhatIf:
        import json
        pol = None if self.tag_policy is None else json.dumps(self.tag_policy).encode()
        c = TsWhatIf(self.source_model.to_c(), self.target_model.to_c(), self.source_par.to_c(),
                     self.target_par.to_c(), float(self.alpha_us), float(self.bytes_per_us),
                     int(self.activation_bytes), pol)
        c._keep = pol
        return c


def _bind():
    L = _lib()
    if not getattr(L, "_pipeline_bound", False):
        L.ts_pipeline_graph.restype = C.c_int
        L.ts_pipeline_graph.argtypes = [C.POINTER(TsPipelineSpec), C.c_int32, C.c_int32,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
        L.ts_rebuild_pipeline.restype = C.c_int
        L.ts_rebuild_pipeline.argtypes = [C.c_void_p, C.POINTER(TsWhatIf),
                                          C.POINTER(C.c_void_p)]
        L.ts_pipeline_spec_get.restype = C.POINTER(TsPipelineSpec)
        L.ts_pipeline_spec_get.argtypes = [C.c_void_p]
        L.ts_pipeline_free.argtypes = [C.c_void_p]
        L._pipeline_bound = True
    return L


def _source_handle(source):
    """A ts_host_graph that keeps Task.meta: from a SynthSpec (its replay
    graph, generated with keep_meta) or recorded traces (a list of paths, or a
    dict of ingest_traces_ex options)."""
    from dataclasses import replace
    from .synth import SynthSpec, TsIngestOptions
    L = _bind()
    h = C.c_void_p()
    if isinstance(source, SynthSpec):
        cs = replace(source, estimate=False, keep_meta=True, tp=1, slice_rank=-1).to_c()
        rc = L.ts_synth_graph(C.byref(cs), C.byref(h), None)
    else:
        opts = dict(source) if isinstance(source, dict) else {"paths": list(source)}
        paths = [str(p).encode() for p in opts.get("paths", ())]
        arr = (C.c_char_p * max(1, len(paths)))(*paths)
        enc = lambda x: None if x is None else str(x).encode()
        if not getattr(L, "_ingest_ex_bound", False):
            L.ts_ingest_traces_ex.restype = C.c_int
            L.ts_ingest_traces_ex.argtypes = [C.POINTER(TsIngestOptions), C.POINTER(C.c_void_p)]
            L._ingest_ex_bound = True
        o = TsIngestOptions(arr, len(paths), int(opts.get("threads", 0)),
                            enc(opts.get("manifest")), enc(opts.get("window")),
                            enc(opts.get("categories_path")), enc(opts.get("policy_path")), 1, 0)
        rc = L.ts_ingest_traces_ex(C.byref(o), C.byref(h))
    if rc != N.TS_OK:
        from .replay import _raise
        _raise(rc)
    return h


def rebuild_pipeline(source, whatif: WhatIfConfig) -> Optional[PipelineSpec]:
    """The PipelineSpec the reference's rebuild_pipeline (transform.cpp:556-701)
    builds for a structural what-if — scale_pp / change_layers / apply_whatif's
    rebuild branch — from a measured source (a SynthSpec or recorded traces,
    see _source_handle).  None when the target differs in nothing the rebuild
    cares about (the reference returns the source graph).  Raises ValueError
    with the TransformError text."""
    L = _bind()
    h = _source_handle(source)
    try:
        w = whatif.to_c()
        p = C.c_void_p()
        rc = L.ts_rebuild_pipeline(h, C.byref(w), C.byref(p))
        if rc != N.TS_OK:
            from .replay import _raise
            _raise(rc)
        if not p.value:
            return None
        try:
            return PipelineSpec.from_c(L.ts_pipeline_spec_get(p).contents)
        finally:
            L.ts_pipeline_free(p)
    finally:
        L.ts_host_graph_free(h)


def pipeline_graph(spec: PipelineSpec, estimate: bool = True, tp: int = 1,
                   names: bool = False) -> SynthGraph:
    """build_pipeline(spec) as a graph (ts_pipeline_graph): the estimate graph
    (gates, intrinsic durations) or, estimate=False, the replay graph of its
    trace; truth_makespan = BuiltPipeline end - origin."""
    L = _bind()
    cs = spec.to_c()
    h = C.c_void_p()
    truth = C.c_int64(0)
    rc = L.ts_pipeline_graph(C.byref(cs), 1 if estimate else 0, int(tp), C.byref(h),
                             C.byref(truth))
    if rc != N.TS_OK:
        from .replay import _raise
        _raise(rc)
    try:
        g, op_index, n_ops = _from_host(h, names)
    finally:
        L.ts_host_graph_free(h)
    return SynthGraph(graph=g, truth_makespan=int(truth.value), op_index=op_index, n_ops=n_ops,
                      names=g.names)


def estimate_batch(spec: PipelineSpec, scenarios, tp: int = 1, device: Optional[int] = None,
                   timestamps: bool = True):
    """Batched estimate(): replays ``scenarios`` (ScenarioSpec) on the estimate
    graph of ``spec``; returns (BatchResult, SynthGraph)."""
    from .replay import simulate_batch
    sg = pipeline_graph(spec, estimate=True, tp=tp)
    return simulate_batch(sg.graph, scenarios, timestamps=timestamps, breakdown=False,
                          device=device), sg


def estimate_whatif(source, whatif: WhatIfConfig, scenarios, tp: int = 1,
                    device: Optional[int] = None, timestamps: bool = True):
    """estimate() for a structural what-if, batched: rebuild_pipeline on the
    host, then the target pipeline's estimate graph replayed for ``scenarios``
    on the GPU.  Returns (BatchResult, SynthGraph, PipelineSpec)."""
    spec = rebuild_pipeline(source, whatif)
    if spec is None:
        raise ValueError("what-if changes nothing the pipeline rebuild models; replay the "
                         "source graph (or use a Retime sweep for pure dp / width changes)")
    res, sg = estimate_batch(spec, scenarios, tp=tp, device=device, timestamps=timestamps)
    return res, sg, spec
