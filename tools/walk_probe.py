"""Walk / reduction timing probe (development tool, not a test).

Builds a BASELINE config graph with the package's generator, replays `calls`
tiles of `tile` scenarios exactly like bench.py (device outputs: start, fin,
span, per-rank breakdown, per-stream busy) and prints the device time per call
of each kernel class (ts_profile_read).  LUMOS_B200_LIB selects a library
build variant; LUMOS_* environment switches apply as usual.

  python tools/walk_probe.py [config5|config4] [tile] [calls] [label]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_09307_b200 import DeviceGraph, ScenarioSpec
    from paper_2504_09307_b200.synth import SynthSpec, generate_graph

    cfg = sys.argv[1] if len(sys.argv) > 1 else "config5"
    tile = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    calls = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    label = sys.argv[4] if len(sys.argv) > 4 else os.environ.get("LUMOS_B200_LIB", "default")
    metrics_only = os.environ.get("PROBE_METRICS_ONLY") == "1"
    model, par, tp, _, _ = bench.CONFIGS[cfg]

    class A:
        config = cfg
        jitter = 0.1
    sk = bench.scenario_kwargs(A)
    if cfg == "config3":
        g = bench.config3_graph(model, par, tp).graph
    else:
        g = generate_graph(SynthSpec(tp=tp, **model, **par)).graph
    dg = DeviceGraph(g, device=0)
    n = dg.n_tasks
    dev = torch.device("cuda", 0)
    start = None if metrics_only else torch.empty((n, tile), dtype=torch.int64, device=dev)
    fin = None if metrics_only else torch.empty((n, tile), dtype=torch.int64, device=dev)
    span = torch.empty((tile, 3), dtype=torch.int64, device=dev)
    bd = torch.empty((tile, dg.n_ranks, 5), dtype=torch.int64, device=dev)
    busy = torch.empty((tile, dg.n_streams), dtype=torch.int64, device=dev)
    sptr = torch.cuda.current_stream(dev).cuda_stream

    def call(k):
        dg.replay_batch(ScenarioSpec(count=tile, first=k * tile, seed=250409307, **sk),
                        start=start, fin=fin, ld=tile, span=span, rank_breakdown=bd,
                        stream_busy=busy, stream=sptr)
    call(0)
    torch.cuda.synchronize()
    dg.profile(True)
    dg.profile_read()
    t0 = time.perf_counter()
    for k in range(calls):
        call(k)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / calls
    p = dg.profile_read()
    walk = p["walk_ms"] / max(1, p["walk_launches"])
    out = {"label": label, "config": cfg, "tile": tile, "metrics_only": metrics_only,
           "des_only": dg.info["des_only"], "des_ms_per_call": p["other_ms"] / calls,
           "walk_ms": walk, "reduce_ms_per_call": p["reduce_ms"] / calls,
           "other_ms_per_call": p["other_ms"] / calls, "wall_ms_per_call": wall * 1e3,
           "walk_tb_s": n * tile * 16 / (walk / 1e3) / 1e12 if walk > 0 else None,
           "g_relax_per_s": n * tile / wall / 1e9,
           "info": {k: dg.info[k] for k in ("max_slots", "n_fused_ranks", "n_candidates")}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
