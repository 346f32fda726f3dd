"""What-if retime sweep throughput (development tool): config 5 (our
generator, with retime metadata), 1,024 scenarios per call, each scenario its
own scale_dp target, model widths (4 variants) and cost model, plus +-10 %
jitter.  Runs the retime walk (kModeRetime) and the materialised path
(LUMOS_RT_FUSED=0: K4r writes the durations, an explicit walk reads them),
checks they agree, and prints device time per call split into
retime/other, walk and reductions.  Usage: python tools/retime_probe.py [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_09307_b200 import DeviceGraph, Retime, ScenarioSpec  # noqa: E402
from paper_2504_09307_b200.synth import SynthSpec, generate_graph  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    model, par, tp, _, _ = bench.CONFIGS["config5"]
    g = generate_graph(SynthSpec(tp=tp, **model, **par)).graph
    dg = DeviceGraph(g, device=0)
    n, S = g.n, 1024
    rng = np.random.default_rng(7)
    d0, f0 = model["d_model"], model["d_ffn"]
    widths = np.array([(d0, f0, 175_000_000_000), (d0 * 5 // 4, f0 * 5 // 4, 270_000_000_000),
                       (d0 * 3 // 4, f0 * 3 // 4, 99_000_000_000), (d0, f0 * 2, 290_000_000_000)],
                      np.int64)
    rt = Retime(alpha_us=rng.uniform(5.0, 30.0, S), bytes_per_us=rng.uniform(2e4, 9e4, S),
                source_dp=par["dp"], target_dp=rng.choice([8, 16, 32, 64], S).astype(np.int32),
                source_model=tuple(int(x) for x in widths[0]),
                target_model=widths[rng.integers(0, 4, S)])
    spec = ScenarioSpec(count=S, seed=250409307, jitter=0.1, retime=rt)
    dev = torch.device("cuda", 0)
    start = torch.empty((n, S), dtype=torch.int64, device=dev)
    fin = torch.empty((n, S), dtype=torch.int64, device=dev)
    span = torch.empty((S, 3), dtype=torch.int64, device=dev)
    bd = torch.empty((S, dg.n_ranks, 5), dtype=torch.int64, device=dev)
    sp = torch.cuda.current_stream().cuda_stream
    kw = dict(start=start, fin=fin, ld=S, span=span, rank_breakdown=bd, stream=sp)
    results = {}
    for fused in ("1", "0"):
        os.environ["LUMOS_RT_FUSED"] = fused
        dg.replay_batch(spec, **kw)
        torch.cuda.synchronize()
        dg.profile(True)
        dg.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dg.replay_batch(spec, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        prof = dg.profile_read()
        dg.profile(False)
        label = "retime walk " if fused == "1" else "materialised"
        print(f"{label}: config5 {n} tasks x {S} scenarios: {ms:.2f} ms per call, "
              f"{n * S / (ms / 1e3) / 1e9:.1f} G relaxations/s; per call: retime+other "
              f"{prof['other_ms'] / reps:.2f} ms, walk {prof['walk_ms'] / reps:.2f} ms, "
              f"reduce {prof['reduce_ms'] / reps:.2f} ms", flush=True)
        results[fused] = (span.clone(), bd.clone(), fin[:: 997].clone(), start[:: 997].clone())
    same = all(torch.equal(a, b) for a, b in zip(results["1"], results["0"]))
    print(f"retime walk == materialised (span, breakdown, sampled timestamps): {same}")
    assert same
    mk = span[:, 2].cpu().numpy()
    tdp = np.asarray(rt.target_dp)
    for d in (8, 16, 32, 64):
        print(f"  target dp {d:3d}: mean makespan {mk[tdp == d].mean() / 1e6:.4f} s "
              f"({(tdp == d).sum()} scenarios)")


if __name__ == "__main__":
    main()
