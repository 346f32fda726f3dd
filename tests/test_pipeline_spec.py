"""The Mode-B boundary (ts_pipeline_graph / pipeline_graph): a reference
PipelineSpec (pipeline.hpp:27-90) — the one pipeline_spec_for builds
(synth.cpp:71-138) or a hand-edited one — becomes the graph of
build_pipeline(spec, DurationHook) (pipeline.cpp:474-477).  CPU checks: the
graphs equal the generator's field by field, and a longest path with gates at
the base durations reproduces the reference's build_pipeline event times."""
import copy

import numpy as np
import pytest

import refshim as R
from paper_2504_09307_b200.pipeline import KernelSpec, PipelineSpec, pipeline_graph
from paper_2504_09307_b200.synth import generate_graph
from test_synth_graph import FIELDS, _assert_same, _lane_sequences, _my_lane_sequences, _spec, \
    longest_path_with_gates


def _ref_spec(pp, dp, m, layers=4, d=1024, f=4096):
    return PipelineSpec.from_json(R.pipeline_spec_json(
        R.synth_spec(pp=pp, dp=dp, m=m, layers=layers, d_model=d, d_ffn=f)))


def hand_edited(pp=3, dp=2, m=5):
    """A spec no generator produces: uneven stages, extra non-GEMM kernels,
    an allreduce without bytes, a p2p-free stage mix, odd microbatch count,
    non-default streams / costs / id counters."""
    sp = _ref_spec(pp, dp, max(m, pp), layers=pp * 2)
    sp.num_microbatches = m
    sp.launch, sp.record, sp.wait, sp.sync = 7, 3, 1, 11
    sp.p2p_recv_base = 17
    sp.compute_stream, sp.reduce_stream, sp.p2p_stream = 21, 23, 25
    sp.first_event, sp.first_correlation = 1000, 5000
    sp.origin = 123456
    st0 = sp.stages[0]
    st0.layers_fwd.append([KernelSpec("fused_norm", 77, 0, {"region": "norm"}),
                           KernelSpec("gemm_x", 500, 0, {"m": "2048", "n": "1024", "k": "512"})])
    st0.layers_bwd.append([KernelSpec("gemm_x_bwd", 900, 0, {"m": "2048", "n": "1024", "k": "512"})])
    sp.stages[-1].post_fwd.append(KernelSpec("extra_head", 333))
    for st in sp.stages:
        for k in st.reduce:
            k.duration += 111
    sp.stages[1].reduce.append(KernelSpec("ncclDevKernel_AllReduce_Sum_f32", 250, 1,
                                          {"collective": "allreduce", "group_size": str(dp)}))
    sp.stages[-1].optimizer.append(KernelSpec("clip_grad", 45, 0, {"bytes": "1024"}))
    return sp


@pytest.mark.parametrize("shape", [(2, 2, 4), (1, 2, 4), (4, 2, 8), (1, 1, 2)])
@pytest.mark.parametrize("estimate", [False, True])
def test_pipeline_spec_for_equals_generator(shape, estimate):
    pp, dp, m = shape
    mine = pipeline_graph(_ref_spec(pp, dp, m), estimate=estimate)
    gen = generate_graph(_spec(pp, dp, m, estimate=estimate))
    _assert_same(mine.graph, gen.graph)
    assert mine.truth_makespan == gen.truth_makespan and mine.n_ops == gen.n_ops
    for k in ("rt_kind", "rt_bytes", "rt_group", "rt_mnk"):
        assert np.array_equal(getattr(mine.graph, k), getattr(gen.graph, k)), k
    if estimate:
        for k in ("gate_from", "gate_to", "gate_kind"):
            assert np.array_equal(getattr(mine.graph, k), getattr(gen.graph, k)), k


@pytest.mark.parametrize("pp,dp,m", [(3, 2, 5), (2, 3, 7), (1, 2, 3)])
def test_hand_edited_spec_matches_build_pipeline(pp, dp, m):
    sp = hand_edited(pp, dp, m) if pp > 1 else _ref_spec(1, dp, m)
    if pp == 1:
        sp.stages[0].layers_fwd[0].append(KernelSpec("dropout", 13))
        sp.stages[0].layers_bwd[0].append(KernelSpec("dropout_bwd", 19))
        sp.num_microbatches = m
    sg = pipeline_graph(sp, estimate=True)
    g = sg.graph
    start, fin = longest_path_with_gates(g, g.duration)
    pid, tid, ts, dur, nops, end = R.pipeline_events_json(sp.to_json())
    assert nops == sg.n_ops
    assert _my_lane_sequences(g, start, fin) == _lane_sequences(pid, tid, ts, dur)
    assert int(fin.max()) - sp.origin == sg.truth_makespan == end - sp.origin
    # the replay graph of the same spec replays to the same makespan (acceptance C1)
    rg = pipeline_graph(sp, estimate=False)
    assert rg.graph.n == g.n and rg.truth_makespan == sg.truth_makespan


def test_retime_metadata_follows_task_meta():
    # the allreduce without bytes keeps kind ALLREDUCE with bytes -1; the
    # optimizer extra kernel with bytes is OPT (region "opt" tag); the GEMM dims
    # come through; "fused_norm" carries nothing
    sp = hand_edited()
    g = pipeline_graph(sp, estimate=True).graph
    kinds = set(g.rt_kind.tolist())
    assert {1, 2, 3, 4, 5} <= kinds
    assert ((g.rt_kind == 3) & (g.rt_bytes < 0)).any()


def test_invalid_specs_raise_like_build_pipeline():
    sp = _ref_spec(2, 1, 4)
    bad = copy.deepcopy(sp)
    bad.stages = bad.stages[:1]
    with pytest.raises(ValueError, match="one stage spec per pipeline stage"):
        pipeline_graph(bad)
    bad = copy.deepcopy(sp)
    bad.num_microbatches = 0
    with pytest.raises(ValueError, match="at least one microbatch"):
        pipeline_graph(bad)
