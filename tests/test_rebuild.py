"""Structural what-if (estimate()'s host step): rebuild_pipeline over a
measured source — tag_tasks, measure_pipeline, the target PipelineSpec
(reference transform.cpp:71-162, 378-701) — through the C ABI
(ts_rebuild_pipeline).  The spec is checked the way the reference's own
tests check rebuilds (test_transform.cpp:230-310): the graph of the rebuilt
spec (build_pipeline + graph_from_events, i.e. ts_pipeline_graph with
estimate = 0) must equal, task for task, the graph the unmodified reference
apply_whatif returns for the same source and config; errors carry the
reference's TransformError text."""
import os

import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200 import (ModelConfig, ParallelismConfig, WhatIfConfig,
                                   rebuild_pipeline)
from paper_2504_09307_b200.pipeline import pipeline_graph
from paper_2504_09307_b200.synth import SynthSpec

FIELDS = ("duration", "original_start", "rank", "lane_kind", "lane", "op_class", "task_kind",
          "edge_from", "edge_to", "rule_kind", "rule_task", "rule_bound", "rule_watch_off",
          "watch_rank", "watch_kind", "watch_lane")


def _model(layers=4, d=1024, f=4096, heads=16, n_params=0):
    return ModelConfig(layers, d, f, heads, d // heads, n_params)


def _tuple(m: ModelConfig):
    return (m.n_params, m.n_layers, m.d_model, m.d_ffn, m.n_heads, m.d_head)


def _par(p: ParallelismConfig):
    return (p.tp, p.pp, p.dp, p.num_microbatches)


def _synth(pp, dp, m, model: ModelConfig):
    return SynthSpec(n_layers=model.n_layers, d_model=model.d_model, d_ffn=model.d_ffn,
                     n_heads=model.n_heads, d_head=model.d_head, pp=pp, dp=dp,
                     num_microbatches=m)


def _ref_source(pp, dp, m, model: ModelConfig):
    h, _ = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=model.n_layers,
                                   d_model=model.d_model, d_ffn=model.d_ffn,
                                   heads=model.n_heads))
    return h


def _assert_graph_equals_reference(spec, ref_handle):
    mine = pipeline_graph(spec, estimate=False, names=True).graph
    ref = ref_handle.export(names=True)
    for k in FIELDS:
        a, b = getattr(mine, k), getattr(ref, k)
        assert np.array_equal(a, b), k
    assert mine.window_start == ref.window_start and mine.window_end == ref.window_end
    assert list(mine.names) == list(ref.names)


CASES = {
    # name: (source pp, dp, m, model), (target pp, dp, m, model)
    "pp2dp2_to_pp4dp4": ((2, 2, 8, _model()), (4, 4, 8, _model())),
    "scale_pp_2_to_4": ((2, 1, 8, _model()), (4, 1, 8, _model())),
    "scale_pp_narrow_2_to_1": ((2, 1, 8, _model()), (1, 1, 8, _model())),
    "layers_4_to_6": ((2, 1, 4, _model()), (2, 1, 4, _model(layers=6))),
    "layers_4_to_2": ((2, 1, 4, _model()), (2, 1, 4, _model(layers=2))),
    "microbatches_4_to_6": ((2, 2, 4, _model()), (2, 2, 6, _model())),
    "dp_1_to_4": ((2, 1, 4, _model()), (2, 4, 4, _model())),
    "dp_4_to_1": ((2, 4, 4, _model()), (2, 1, 4, _model())),
    "width_at_pp2": ((2, 2, 4, _model()), (2, 2, 4, _model(d=1536, f=6144, heads=24))),
    "width_and_depth": ((2, 1, 4, _model()), (4, 2, 8, _model(layers=8, d=2048, f=8192,
                                                                   heads=32))),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_rebuilt_pipeline_equals_reference_apply_whatif(case):
    (spp, sdp, sm, smodel), (tpp, tdp, tm, tmodel) = CASES[case]
    w = WhatIfConfig(smodel, tmodel, ParallelismConfig(1, spp, sdp, sm),
                     ParallelismConfig(1, tpp, tdp, tm))
    spec = rebuild_pipeline(_synth(spp, sdp, sm, smodel), w)
    assert spec is not None and spec.pp == tpp and spec.dp == tdp
    ref, notes = _ref_source(spp, sdp, sm, smodel).apply_whatif(
        _tuple(smodel), _tuple(tmodel), _par(w.source_par), _par(w.target_par))
    assert notes.startswith("rebuilt pipeline"), notes
    _assert_graph_equals_reference(spec, ref)
    # the estimate graph of the same spec replays, at the base durations, to
    # the reference's replay of its rebuilt graph (test_transform.cpp:236-238)
    est = pipeline_graph(spec, estimate=True)
    assert est.truth_makespan == int(ref.simulate()[2][2])


def test_rebuild_from_recorded_traces(tmp_path):
    # a Chrome-trace source (one file per rank, args incl. correlation ids)
    # through ingest with keep_meta: tags come from Task.meta exactly as the
    # reference reads them from its own trace parser
    smodel, tmodel = _model(), _model(layers=8)
    n = R.write_rank_traces(R.synth_spec(pp=2, dp=2, m=4), str(tmp_path))
    paths = sorted(str(tmp_path / f) for f in os.listdir(tmp_path))
    assert len(paths) == n == 4
    w = WhatIfConfig(smodel, tmodel, ParallelismConfig(1, 2, 2, 4), ParallelismConfig(1, 4, 2, 4))
    spec = rebuild_pipeline(paths, w)
    ref, _ = R.ingest_traces(paths).apply_whatif(_tuple(smodel), _tuple(tmodel),
                                                 _par(w.source_par), _par(w.target_par))
    _assert_graph_equals_reference(spec, ref)


def test_rebuild_spec_content():
    # the rebuilt spec itself: measured host costs, p2p sizing from the
    # cost model, per-stage allreduce / optimizer sized from the measured bytes
    w = WhatIfConfig(_model(), _model(), ParallelismConfig(1, 2, 2, 8),
                     ParallelismConfig(1, 4, 4, 8), alpha_us=10.0, bytes_per_us=50000.0)
    spec = rebuild_pipeline(_synth(2, 2, 8, _model()), w)
    assert (spec.launch, spec.record, spec.wait, spec.sync) == (5, 2, 2, 5)
    assert spec.activation_bytes == 2048 * 1024 * 2
    assert spec.p2p_send == round(10.0 + spec.activation_bytes / 50000.0)
    assert [k.name for k in spec.stages[0].layers_fwd[0]] == ["gemm_qkv", "attn_core", "gemm_mlp"]
    assert spec.stages[0].pre_fwd[0].name == "embedding_fwd"
    assert spec.stages[3].post_fwd[0].name == "norm_loss_fwd"
    ar = spec.stages[1].reduce[0]
    assert ar.args["collective"] == "allreduce" and ar.args["group_size"] == "4"
    layer_bytes = (4 * 1024 * 1024 + 2 * 1024 * 4096) * 2
    assert int(ar.args["bytes"]) == layer_bytes  # one layer per stage, no vocab table
    assert spec.stages[1].optimizer[0].args["bytes"] == ar.args["bytes"]


def test_rebuild_unchanged_returns_none():
    w = WhatIfConfig(_model(), _model(), ParallelismConfig(1, 2, 2, 4),
                     ParallelismConfig(1, 2, 2, 4))
    assert rebuild_pipeline(_synth(2, 2, 4, _model()), w) is None


@pytest.mark.parametrize("mutate, msg", [
    (lambda w: setattr(w.source_par, "dp", 4),
     "graph covers 4 ranks but source parallelism implies 8"),
    (lambda w: setattr(w.target_model, "n_layers", 5),
     "target layer count must divide evenly across pipeline stages"),
    (lambda w: setattr(w.target_par, "tp", 2), "tensor-parallel rescaling is not supported"),
    (lambda w: setattr(w.target_par, "num_microbatches", 2),
     "what-if config invalid: ParallelismConfig.num_microbatches must be >= pp"),
    (lambda w: setattr(w.source_model, "n_layers", 6),
     "measured 4 forward / 4 backward layer groups, source model has 6 layers"),
])
def test_rebuild_errors_match_reference(mutate, msg):
    w = WhatIfConfig(_model(), _model(), ParallelismConfig(1, 2, 2, 4),
                     ParallelismConfig(1, 4, 2, 4))
    mutate(w)
    with pytest.raises(Exception, match=msg):
        rebuild_pipeline(_synth(2, 2, 4, _model()), w)
    with pytest.raises(Exception, match=msg.split(" (")[0]):
        _ref_source(2, 2, 4, _model()).apply_whatif(_tuple(w.source_model),
                                                     _tuple(w.target_model),
                                                     _par(w.source_par), _par(w.target_par))


def test_rebuild_needs_task_metadata():
    # a source without Task.meta cannot be measured; the error says why
    from paper_2504_09307_b200 import pipeline as P
    import ctypes as C
    L = P._bind()
    h = C.c_void_p()
    cs = _synth(2, 2, 4, _model()).to_c()  # keep_meta off
    assert L.ts_synth_graph(C.byref(cs), C.byref(h), None) == 0
    w = WhatIfConfig(_model(), _model(), ParallelismConfig(1, 2, 2, 4),
                     ParallelismConfig(1, 4, 2, 4)).to_c()
    out = C.c_void_p()
    try:
        assert L.ts_rebuild_pipeline(h, C.byref(w), C.byref(out)) != 0
        assert "task metadata" in L.ts_last_error().decode()
    finally:
        L.ts_host_graph_free(h)


def test_rebuild_from_traces_with_exotic_args(tmp_path, monkeypatch):
    # recorded traces whose kernels carry float / array / object args: those
    # files take the DOM path when Task.meta is kept (nlohmann's dump text is
    # the meta value), and the args travel into the rebuilt KernelSpecs
    import json
    smodel = _model()
    R.write_rank_traces(R.synth_spec(pp=2, dp=1, m=4), str(tmp_path))
    paths = sorted(str(tmp_path / f) for f in os.listdir(tmp_path))
    for p in paths:
        d = json.load(open(p))
        for ev in d["traceEvents"]:
            if ev.get("cat") == "kernel" and ev["name"].startswith("gemm"):
                ev.setdefault("args", {}).update({"flops": 1.5e12, "dims": [2048, [1, 2]],
                                                  "misc": {"a": None, "b": True}})
        json.dump(d, open(p, "w"))
    w = WhatIfConfig(smodel, smodel, ParallelismConfig(1, 2, 1, 4), ParallelismConfig(1, 4, 1, 4))
    spec = rebuild_pipeline(paths, w)
    k = spec.stages[0].layers_fwd[0][0]
    assert k.name == "gemm_qkv" and k.args["flops"] == "1500000000000.0", k.args
    assert k.args["dims"] == "[2048,[1,2]]" and k.args["misc"] == '{"a":null,"b":true}'
    ref, _ = R.ingest_traces(paths).apply_whatif(_tuple(smodel), _tuple(smodel),
                                                 _par(w.source_par), _par(w.target_par))
    _assert_graph_equals_reference(spec, ref)


def test_rebuild_random_whatifs_equal_reference():
    # seeded sweep over structural what-ifs (pp, dp, microbatches, layers,
    # widths): every rebuilt graph equals the reference apply_whatif graph, and
    # configs the reference rejects are rejected with the same message
    import random
    rnd = random.Random(2504)
    widths = [(1024, 4096, 16), (1536, 6144, 24), (2048, 8192, 32), (1024, 2048, 16)]
    checked = 0
    errors = 0
    for trial in range(40):
        spp, sdp = rnd.choice([1, 2, 4]), rnd.choice([1, 2])
        sm = rnd.choice([4, 6, 8])
        slayers = spp * rnd.choice([1, 2])
        sw = rnd.choice(widths)
        tpp, tdp = rnd.choice([1, 2, 4]), rnd.choice([1, 2, 4])
        tm = rnd.choice([4, 6, 8])
        tlayers = tpp * rnd.choice([1, 2, 3])
        tw = rnd.choice(widths)
        smodel = _model(layers=slayers, d=sw[0], f=sw[1], heads=sw[2])
        tmodel = _model(layers=tlayers, d=tw[0], f=tw[1], heads=tw[2])
        if sm < spp:
            continue
        w = WhatIfConfig(smodel, tmodel, ParallelismConfig(1, spp, sdp, sm),
                         ParallelismConfig(1, tpp, tdp, tm))
        ref_h = _ref_source(spp, sdp, sm, smodel)
        try:
            ref, notes = ref_h.apply_whatif(_tuple(smodel), _tuple(tmodel),
                                            _par(w.source_par), _par(w.target_par))
            ref_err = None
        except R.RefError as e:
            ref, notes, ref_err = None, "", str(e).split("] ", 1)[1]
        try:
            spec = rebuild_pipeline(_synth(spp, sdp, sm, smodel), w)
            err = None
        except Exception as e:
            spec, err = None, str(e)
        if ref_err is not None:
            assert err == ref_err, (trial, err, ref_err)
            errors += 1
            continue
        if not notes.startswith("rebuilt pipeline"):
            continue  # in-place retime / no-op: not the rebuild's branch
        assert err is None, (trial, err)
        _assert_graph_equals_reference(spec, ref)
        checked += 1
    assert checked >= 12 and errors >= 1, (checked, errors)
