"""Generate tests/golden/*.npz from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Runs here, where /root/reference is present and oracle/_ref/libtracesim_ref.so
has been built from it (oracle/Makefile).  Each fixture holds a reference-built
ExecutionGraph (SoA), per-scenario durations and what the reference's own
tracesim::simulate() (simulate.cpp:341-347) and breakdown_by_rank()
(metrics.cpp:43-103) return for them, so tests can pin the restatement and the
CUDA path on the GPU box, where /root/reference does not exist.

Graphs come from the reference generator (synth.cpp:71-170 via build_graph /
merge_ranks, build.cpp:338-580).  Scenario durations follow this repo's
scenario definition (Philox2x32-10 jitter, mul_div class scale),
materialised by the restatement and handed to the reference as explicit
durations, so the reference's replay is the thing recorded.

    python tools/make_golden.py        # rewrites tests/golden/
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import refshim as R  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

GRAPH_FIELDS = ("duration", "original_start", "rank", "lane_kind", "lane", "op_class",
                "task_kind", "edge_from", "edge_to", "rule_kind", "rule_task", "rule_bound",
                "rule_watch_off", "watch_rank", "watch_kind", "watch_lane")

CASES = {
    # 15B pp1 dp2 m4, rank 0 sliced (2,353 tasks)
    "config1_jitter": dict(spec=dict(pp=1, dp=2, m=4, layers=48, d_model=6144, d_ffn=12288),
                           tp=1, slice_rank=0, first=0, count=4,
                           sc=dict(seed=250409307, jitter=0.1)),
    # multi-rank: pp2 dp2 m4 x TP2 replicas, per-class duration scaling + jitter
    "pp2dp2tp2_scale": dict(spec=dict(pp=2, dp=2, m=4, layers=4), tp=2, slice_rank=-1,
                            first=1000, count=4,
                            sc=dict(seed=7, jitter=0.05, scale_lo=768, scale_hi=1536,
                                    scale_den=1024)),
}


def make(name, c):
    h, truth = R.generate(R.synth_spec(**c["spec"]), tp=c["tp"], slice_rank=c["slice_rank"])
    g = h.export()
    sc_kw = {**dict(scale_lo=0, scale_hi=0, scale_den=0), **c["sc"]}
    sc = R.OrcScenarios(**sc_kw)
    durs, starts, fins, spans, bds = [], [], [], [], []
    for s in range(c["first"], c["first"] + c["count"]):
        dur = R.orc_durations(g, sc, s)
        rs, rf, rspan = h.simulate(dur)
        wend = max(g.window_end, g.window_start + int(rspan[2]))
        bd = h.breakdown_by_rank(rs, rf, g.window_start, wend)
        durs.append(dur)
        starts.append(rs)
        fins.append(rf)
        spans.append(np.asarray(rspan, np.int64))
        bds.append(np.array([bd[r] for r in sorted(bd)], np.int64))
    rec = {f"g_{k}": getattr(g, k) for k in GRAPH_FIELDS}
    rec.update(g_window=np.array([g.window_start, g.window_end], np.int64),
               truth_makespan=np.int64(truth),
               sc=np.array([sc_kw["seed"], sc_kw["scale_lo"], sc_kw["scale_hi"],
                            sc_kw["scale_den"]], np.int64),
               jitter=np.float64(sc_kw["jitter"]), first=np.int64(c["first"]),
               durations=np.stack(durs), start=np.stack(starts), fin=np.stack(fins),
               span=np.stack(spans), breakdown=np.stack(bds))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{path}: {g.n} tasks, {c['count']} scenarios, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    for name, c in CASES.items():
        make(name, c)
