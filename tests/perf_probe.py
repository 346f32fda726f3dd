"""Kernel throughput probe (development tool, not a test): replays a
generator graph built by the reference (oracle/_ref) over S scenarios and times
the device work with CUDA events.  Usage: python tests/perf_probe.py [S] [pp dp m]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import refshim as R  # noqa: E402
from paper_2504_09307_b200 import DeviceGraph, ScenarioSpec  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    pp, dp, m = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (4, 16, 32)
    reps = int(os.environ.get("REPS", "5"))
    t = time.time()
    h, truth = R.generate(R.synth_spec(pp=pp, dp=dp, m=m, layers=96, d_model=12288,
                                       d_ffn=49152, heads=96))
    g = h.export()
    print(f"graph {g.n} tasks, {g.edge_from.shape[0]} edges, gen {time.time() - t:.1f}s", flush=True)
    t = time.time()
    dg = DeviceGraph(g, device=0)
    print(f"compile+upload {time.time() - t:.2f}s info {dg.info}", flush=True)
    n = g.n
    start = torch.empty((n, S), dtype=torch.int64, device="cuda")
    fin = torch.empty((n, S), dtype=torch.int64, device="cuda")
    span = torch.empty((S, 3), dtype=torch.int64, device="cuda")
    bd = torch.empty((S, dg.n_ranks, 5), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    spec = ScenarioSpec(count=S, seed=250409307, jitter=0.1)
    for mode in ("fin+start", "fin only", "fin+start+breakdown"):
        kw = dict(start=start if mode != "fin only" else None, fin=fin, ld=S, span=span,
                  rank_breakdown=bd if "breakdown" in mode else None, stream=stream)
        for _ in range(2):
            dg.replay_batch(spec, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dg.replay_batch(spec, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        relax = n * S / (ms / 1e3)
        wbytes = n * S * (16 if mode != "fin only" else 8)
        print(f"{mode:22s} S={S} {ms:9.3f} ms  {relax / 1e9:8.2f} G relax/s  "
              f"{wbytes / (ms / 1e3) / 1e9:8.1f} GB/s written  {S / (ms / 1e3):10.1f} replays/s",
              flush=True)
    # parity spot check: scenario 0 vs reference
    dur = R.orc_durations(g, R.OrcScenarios(seed=250409307, jitter=0.1), 0)
    dg.replay_batch(spec, start=start, fin=fin, ld=S, span=span, stream=stream)
    torch.cuda.synchronize()
    rs, rf, rspan = h.simulate(dur)
    assert np.array_equal(fin[:, 0].cpu().numpy(), rf), "parity"
    print("parity scenario 0 ok, makespan", int(rspan[2]))


if __name__ == "__main__":
    main()
