#!/usr/bin/env python3
"""Benchmark of the batched Lumos replay on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[4], the one quoted at 1/2/4/8 GPUs): the
512-rank GPT-3 175B graph — 96 layers, d_model 12288, d_ffn 49152, pp4 dp16,
32 microbatches, x TP8 replicas = 4,952,576 tasks — replayed for a
65,536-scenario Monte Carlo (every task duration jittered ±10%, Philox keyed
by (task, scenario)).  A step is one pass over the whole batch: every
scenario's start/finish timestamps of every task (written to HBM, 1,024
scenarios per tile), its makespan, the per-rank 4-way breakdown and the
per-stream busy time; for N > 1 the scenarios are split across ranks and the
per-scenario results are gathered to rank 0 over NCCL (the only collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU replay (oracle/_ref, the
unmodified tracesim compiled here) on the box's host cores on a bounded sample
of the same workload ("Measurement").
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (model, parallelism, tp replicas, scenarios, label)
    "config5": (dict(n_layers=96, d_model=12288, d_ffn=49152, n_heads=96, d_head=128),
                dict(pp=4, dp=16, num_microbatches=32), 8, 65536,
                "512-rank GPT-3 175B (96L d12288 f49152, pp4 dp16 m32 x TP8 replicas)"),
    "config4": (dict(n_layers=96, d_model=12288, d_ffn=49152, n_heads=96, d_head=128),
                dict(pp=4, dp=8, num_microbatches=32), 8, 16384,
                "256-rank GPT-3 175B (pp4 dp8 m32 x TP8 replicas)"),
    # estimate() of a structural what-if: a measured pp2 dp2 trace of the 44B
    # model is rebuilt for pp4 dp4 (rebuild_pipeline, transform.cpp:556-701)
    # and the target pipeline's estimate graph (build_pipeline + DurationHook
    # semantics: p2p rendezvous / collective barrier gates) is replayed
    "config3": (dict(n_layers=48, d_model=12288, d_ffn=24576, n_heads=96, d_head=128),
                dict(pp=4, dp=4, num_microbatches=16), 4, 4096,
                "64-rank 44B estimate(): pipeline rebuilt for pp4 dp4 m16 from a measured "
                "pp2 dp2 trace (48L d12288 f24576, x TP4 replicas)"),
    "config2": (dict(n_layers=48, d_model=6144, d_ffn=12288, n_heads=48, d_head=128),
                dict(pp=2, dp=2, num_microbatches=4), 2, 1024,
                "8-rank GPT-3 15B (pp2 dp2 m4 x TP2 replicas)"),
}
METRIC = "scenario-node relaxations/sec (replays/sec) at 1/2/4/8 B200; % HBM roofline"
# per-class kernel-duration scaling sweep of config4: each
# scenario draws a rational factor num/1024, num in [768, 1536], per duration
# class (d' = mul_div(d, num, 1024), transform.cpp:38-43); no jitter
SCALE_SWEEP = dict(scale_lo=768, scale_hi=1536, scale_den=1024)


def scenario_kwargs(args):
    """ScenarioSpec / OrcScenarios fields of the workload's scenarios."""
    if args.config == "config4":
        return dict(jitter=0.0, **SCALE_SWEEP)
    return dict(jitter=args.jitter)


def workload_kind(args):
    if args.config == "config4":
        return "kernel-duration scaling sweep (per-class factors 768..1536 / 1024)"
    return f"Monte Carlo (jitter {args.jitter})"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config5", choices=sorted(CONFIGS))
    ap.add_argument("--scenarios", type=int, default=0, help="override the batch size")
    ap.add_argument("--tile", type=int, default=0,
                    help="scenarios per replay call (default: 1024; 2048 for config4/5; the whole "
                         "shard for config3, whose 4 components need wide launches)")
    ap.add_argument("--jitter", type=float, default=0.1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-audit", action="store_true", help="skip the parity audit")
    ap.add_argument("--no-cpu-full", action="store_true",
                    help="skip the same-config (whole-graph) reference sample")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def walk_traffic(config, tile):
    """dram bytes per walk launch from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "walk_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{config}/tile{tile}")
        return e
    except (OSError, ValueError):
        return None


def config3_graph(model, par, tp):
    """BASELINE config 3: the estimate graph of the pipeline rebuild_pipeline
    lays out for the target parallelism from a measured source trace (the
    generator's pp2 dp2 trace of the same model, Task.meta kept)."""
    from paper_2504_09307_b200 import (ModelConfig, ParallelismConfig, WhatIfConfig,
                                       pipeline_graph, rebuild_pipeline)
    from paper_2504_09307_b200.synth import SynthSpec
    src = dict(pp=2, dp=2, num_microbatches=par["num_microbatches"])
    mc = ModelConfig(model["n_layers"], model["d_model"], model["d_ffn"], model["n_heads"],
                     model["d_head"])
    w = WhatIfConfig(mc, mc, ParallelismConfig(1, **src), ParallelismConfig(1, **par))
    spec = rebuild_pipeline(SynthSpec(**model, **src), w)
    return pipeline_graph(spec, estimate=True, tp=tp)


# ------------------------------------------------------------ reference arm

def cpu_sample_graph(args):
    """The reference's own graph for the bounded CPU sample: one TP replica of
    the workload (the tp=1 generator graph, identical per-replica structure)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refshim as R
    model, par, tp, _, _ = CONFIGS[args.config]
    spec = R.synth_spec(pp=par["pp"], dp=par["dp"], m=par["num_microbatches"],
                        layers=model["n_layers"], d_model=model["d_model"], d_ffn=model["d_ffn"],
                        heads=model["n_heads"])
    h, _ = R.generate(spec, tp=1)
    g = h.export()
    return R, h, g


def host_info():
    """Host cores and CPU model of the box the reference arm runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        mem_gb = psutil.virtual_memory().available / 2 ** 30
    except Exception:
        mem_gb = None
    return {"nproc": os.cpu_count() or 1, "cpu_model": model,
            "mem_available_gb": None if mem_gb is None else round(mem_gb, 1)}


def cpu_threads(gb_per_thread=1.0):
    """Every host core, bounded by available memory (each thread replays on its
    own copy of the reference graph)."""
    info = host_info()
    n = info["nproc"]
    if info["mem_available_gb"]:
        n = min(n, max(1, int(info["mem_available_gb"] * 0.6 / gb_per_thread)))
    return max(1, n)


def run_cpu_sample(R, h, g, args, first, threads, per_thread=1):
    """Wall seconds of threads * per_thread reference simulate() calls (one
    scenario per call, one thread per call at a time); scenario durations are
    filled before the clock (their time is not counted)."""
    sc = R.OrcScenarios(seed=250409307, **scenario_kwargs(args))
    cls = g.default_scale_class()
    count = threads * per_thread
    secs, mk = h.bench_simulate(sc, first, count, cls, threads)
    return secs, count


def cpu_full_graph(args, threads):
    """Same-config reference number: the unmodified reference simulate() on the
    whole workload graph (all TP replicas), one scenario per thread."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refshim as R
    model, par, tp, _, _ = CONFIGS[args.config]
    spec = R.synth_spec(pp=par["pp"], dp=par["dp"], m=par["num_microbatches"],
                        layers=model["n_layers"], d_model=model["d_model"], d_ffn=model["d_ffn"],
                        heads=model["n_heads"])
    t0 = time.time()
    h, _ = R.generate(spec, tp=tp)
    g = h.export()
    build_s = time.time() - t0
    sc = R.OrcScenarios(seed=250409307, **scenario_kwargs(args))
    secs, mk, fill = h.bench_simulate(sc, 0, threads, g.default_scale_class(), threads,
                                      with_fill=True)
    return {"value": g.n * threads / secs, "unit": "relaxations/s", "cores": threads,
            "kind": "reference", "tasks": g.n,
            "sample": f"{threads} scenarios of the full {g.n}-task workload graph, one "
                      f"tracesim::simulate() per thread, {secs:.1f} s wall (duration fill "
                      f"{fill:.1f} s and graph build {build_s:.1f} s outside the clock)"}


def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    R, h, g = cpu_sample_graph(args)
    threads = cpu_threads(1.0)
    for w in range(args.warmup):
        run_cpu_sample(R, h, g, args, 10_000_000 + w * threads, threads)
    # each step's clock covers the parallel simulate() region only; the
    # per-thread graph copies are made before it starts (ref_shim.cpp)
    wall = 0.0
    total = 0
    for k in range(args.steps):
        secs, count = run_cpu_sample(R, h, g, args, k * threads, threads)
        wall += secs
        total += count
    relax = g.n * total / wall
    line = {"impl": "reference", "metric": METRIC, "value": relax, "unit": "relaxations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (generator graph, Philox-jittered durations)",
            "replays_per_s": total / wall,
            "config": {"workload": CONFIGS[args.config][4] + " — reference CPU replay on a "
                       "bounded sample", "sample_tasks": g.n},
            "cpu_baseline": {"value": relax, "unit": "relaxations/s", "cores": threads,
                             "kind": "reference", "host": host_info(),
                             "sample": f"{threads} scenarios per step, one per host thread, each a "
                                       f"full tracesim::simulate() of one TP replica "
                                       f"({g.n} tasks) of the workload (durations filled outside "
                                       f"the clock)"},
            "e2e": {"value": relax, "unit": "relaxations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- parity audit

def audit(args, g, dg, replay_tile, first, S_local, tile, bd_all, span_all, busy_all):
    """Bit-exact audit of the benchmarked path, outside the timed region: for
    scenario ids spread over the whole batch (first, middle and last tile,
    even and odd columns) every start / finish of every task of all TP
    replicas, the span and every per-rank breakdown row are compared with the
    unmodified reference simulate() / breakdown_by_rank() (oracle/_ref) on the
    oracle's durations of the same global (task, scenario) ids.  The reference
    replays one TP replica (the tp=1 generator graph, task-for-task identical
    to each replica's ranks) at a time, so 8 replicas x K scenarios run as
    independent CPU jobs on the host threads."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    R, h1, g1 = cpu_sample_graph(args)
    _, _, tp, _, _ = CONFIGS[args.config]
    n_tiles = S_local // tile
    picks = sorted({(0, 0), (0, 1), (n_tiles // 2, tile // 2 - 1), (n_tiles // 2, tile // 2),
                    (max(0, (2 * n_tiles) // 3), min(tile - 1, 777)), (n_tiles - 1, tile - 2),
                    (n_tiles - 1, tile - 1), (max(0, n_tiles - 2), min(tile - 1, 1501))})
    t0 = time.time()
    nr1 = int(g1.rank.max()) + 1
    of = np.searchsorted(g.rank, np.arange(nr1 * tp + 1))
    replica_idx = [np.concatenate([np.arange(of[r * tp + t], of[r * tp + t + 1])
                                   for r in range(nr1)]) for t in range(tp)]
    cls = np.zeros(g.duration.shape[0], np.uint8)
    cls[g.task_kind == 1] = 1
    cls[(g.task_kind == 1) & (g.op_class == 1)] = 2
    sc = R.OrcScenarios(seed=250409307, **scenario_kwargs(args))
    cols = {}
    for ti in sorted({p[0] for p in picks}):
        start, fin = replay_tile(ti)  # the benchmark's own call for that tile
        for t_, c in picks:
            if t_ == ti:
                cols[ti * tile + c] = (start[:, c].cpu().numpy(), fin[:, c].cpu().numpy())
    jobs = []
    for s_local, (st, fi) in cols.items():
        s = first + s_local
        dur = np.zeros(g.duration.shape[0], np.int64)
        R.orc().orc_fill_durations(C.byref(sc), s, dur.shape[0],
                                   g.duration.ctypes.data_as(R._i64p), cls.ctypes.data_as(R._u8p),
                                   dur.ctypes.data_as(R._i64p))
        for t in range(tp):
            jobs.append((s_local, t, np.ascontiguousarray(dur[replica_idx[t]])))

    def run(job):
        s_local, t, d = job
        rs, rf, rspan = h1.simulate(d)
        return s_local, t, rs, rf, rspan

    threads = max(1, min(len(jobs), os.cpu_count() or 1, 16))
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(run, jobs))
    mism = {"start": 0, "fin": 0, "span": 0, "breakdown_rows": 0}
    ends = {}
    ranks_of = np.asarray(dg.ranks)
    for s_local, t, rs, rf, rspan in res:
        st, fi = cols[s_local]
        mism["start"] += int(np.count_nonzero(st[replica_idx[t]] != rs))
        mism["fin"] += int(np.count_nonzero(fi[replica_idx[t]] != rf))
        ends[s_local] = max(ends.get(s_local, rspan[1]), rspan[1])
    W = g.window_start
    for s_local, end in ends.items():
        want = np.array([W, end, end - W], np.int64)
        mism["span"] += int(not np.array_equal(span_all[s_local], want))
    for s_local, t, rs, rf, rspan in res:
        wend = max(g.window_end, W + int(ends[s_local] - W))
        ref = h1.breakdown_by_rank(rs, rf, W, wend)
        for r1, row in ref.items():
            rr = int(np.searchsorted(ranks_of, r1 * tp + t))
            mism["breakdown_rows"] += int(tuple(bd_all[s_local, rr]) != row)
    return {"scenarios": sorted(first + s for s in cols), "replicas": tp,
            "tasks_checked": int(len(cols) * g.duration.shape[0]),
            "breakdown_rows_checked": int(len(cols) * len(ranks_of)),
            "mismatches": int(sum(mism.values())), "by_field": mism,
            "reference": "oracle/_ref tracesim::simulate + breakdown_by_rank, one TP replica "
                         "(tp=1 generator graph) per job",
            "cpu_threads": threads, "seconds": round(time.time() - t0, 1)}


# ------------------------------------------------------------------ our arm

def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2504_09307_b200 import DeviceGraph, ScenarioSpec
    from paper_2504_09307_b200 import _native as N
    from paper_2504_09307_b200.synth import SynthSpec, generate_graph

    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    model, par, tp, scenarios, label = CONFIGS[args.config]
    from paper_2504_09307_b200.shard import gather_rows, shard
    S_total = args.scenarios or scenarios
    first, S_local = shard(S_total, world, rank)
    # configs 4/5: 2,048 scenarios per call (81 / 162 GB of timestamps in HBM): wider walk and
    # K5 grids waste less of their last wave (measured: config4 235 -> 251, config5 225 -> 234
    # G relaxations/s; 512 per call drops config5 to 205)
    default_tile = {"config3": S_local, "config4": 2048, "config5": 2048}.get(args.config, 1024)
    tile = min(args.tile or default_tile, S_local)
    assert S_local % tile == 0, "scenarios per GPU must be a multiple of the tile"

    t0 = time.time()
    if args.config == "config3":
        sg = config3_graph(model, par, tp)
    else:
        sg = generate_graph(SynthSpec(tp=tp, **model, **par))
    g = sg.graph
    t_gen = time.time() - t0
    t0 = time.time()
    dg = DeviceGraph(g, device=local)
    t_compile = time.time() - t0
    n = dg.n_tasks
    R_, ST_ = dg.n_ranks, dg.n_streams

    dev = torch.device("cuda", local)
    start = torch.empty((n, tile), dtype=torch.int64, device=dev)
    fin = torch.empty((n, tile), dtype=torch.int64, device=dev)
    span = torch.empty((S_local, 3), dtype=torch.int64, device=dev)
    bd = torch.empty((S_local, R_, 5), dtype=torch.int64, device=dev)
    busy = torch.empty((S_local, ST_), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    if world > 1 and rank == 0:
        span_all = torch.empty((S_total, 3), dtype=torch.int64, device=dev)
        bd_all = torch.empty((S_total, R_, 5), dtype=torch.int64, device=dev)
        busy_all = torch.empty((S_total, ST_), dtype=torch.int64, device=dev)

    def gather():
        # the only collective: per-scenario results to rank 0 (NCCL)
        if world == 1:
            return
        gather_rows(span, world, rank, span_all if rank == 0 else None)
        gather_rows(bd, world, rank, bd_all if rank == 0 else None)
        gather_rows(busy, world, rank, busy_all if rank == 0 else None)

    def step():
        for t0_ in range(0, S_local, tile):
            spec = ScenarioSpec(count=tile, first=first + t0_, seed=250409307,
                                **scenario_kwargs(args))
            dg.replay_batch(spec, start=start, fin=fin, ld=tile, span=span[t0_:t0_ + tile],
                            rank_breakdown=bd[t0_:t0_ + tile], stream_busy=busy[t0_:t0_ + tile],
                            stream=sptr)
        gather()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # timed region
    sampler = ClockSampler(local)
    time.sleep(0.3)
    dg.profile(True)
    dg.profile_read()
    launches0 = N.lib().ts_kernel_launches()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    ms = e0.elapsed_time(e1)
    launches = (N.lib().ts_kernel_launches() - launches0) / args.steps
    prof = dg.profile_read()
    dg.profile(False)
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    relax_per_step = n * S_total
    value = relax_per_step / (ms_per_step / 1e3)

    # roofline of the dominant kernel (K1 walk): algorithmic bytes per launch =
    # start + finish rows written (16 B per task per scenario); predecessor
    # finishes are read from shared memory (0 HBM bytes) and durations are
    # generated in registers (0 HBM bytes) — DESIGN.md "Roofline".
    walk_bytes = n * tile * 16 + dg.info["program_bytes"]
    walk_avg_ms = prof["walk_ms"] / max(1, prof["walk_launches"])
    achieved = walk_bytes / (walk_avg_ms / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    traffic = walk_traffic(args.config, tile)
    step_ms_dev = (prof["walk_ms"] + prof["reduce_ms"] + prof["other_ms"]) / args.steps

    # end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        h_span = torch.empty((S_local, 3), dtype=torch.int64).pin_memory()
        h_bd = torch.empty((S_local, R_, 5), dtype=torch.int64).pin_memory()
        h_busy = torch.empty((S_local, ST_), dtype=torch.int64).pin_memory()
        sc_bytes = 0

        def e2e_step():
            nonlocal sc_bytes
            sc_bytes = 0
            for t0_ in range(0, S_local, tile):
                spec = ScenarioSpec(count=tile, first=first + t0_, seed=250409307,
                                    **scenario_kwargs(args))
                sc_bytes += 72  # the ts_scenarios descriptor read from host memory
                dg.replay_batch(spec, start=start, fin=fin, ld=tile,
                                span=h_span[t0_:t0_ + tile], rank_breakdown=h_bd[t0_:t0_ + tile],
                                stream_busy=h_busy[t0_:t0_ + tile], stream=sptr,
                                host_async=True)
            dg.wait()  # every tile's results are in host memory before the step ends
        e2e_step()
        torch.cuda.synchronize()
        barrier()
        tw = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e2e_s = (time.perf_counter() - tw) / args.steps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        d2h = (h_span.numel() + h_bd.numel() + h_busy.numel()) * 8
        e2e = {"value": relax_per_step / e2e_s, "unit": "relaxations/s",
               "h2d_bytes_per_step": sc_bytes * world, "d2h_bytes_per_step": d2h * world,
               "ms_per_step": e2e_s * 1e3,
               "note": "host scenario descriptors in, per-scenario span + per-rank breakdown + "
                       "per-stream busy copied to pinned host memory every step (each tile's "
                       "copy overlaps the next tile's kernels, host_async; the step ends after "
                       "ts_graph_wait); timestamps stay in device memory"}

    # scenarios the exact event-driven path re-ran (failed sync certificates),
    # counted on one extra step outside the timed region
    fixups = 0
    nfix = np.zeros(1, np.int32)
    for t0_ in range(0, S_local, tile):
        spec = ScenarioSpec(count=tile, first=first + t0_, seed=250409307, **scenario_kwargs(args))
        dg.replay_batch(spec, start=start, fin=fin, ld=tile, span=span[t0_:t0_ + tile],
                        rank_breakdown=bd[t0_:t0_ + tile], stream_busy=busy[t0_:t0_ + tile],
                        stream=sptr, n_fixups=nfix)
        fixups += int(nfix[0])
    if world > 1:
        t = torch.tensor([fixups], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        fixups = int(t.item())

    # parity audit of the benchmarked kernels (N = 1, outside the timed region)
    audit_res = None
    if rank == 0 and world == 1 and not args.no_audit and args.config in ("config5", "config4"):
        def replay_tile(ti):
            spec = ScenarioSpec(count=tile, first=first + ti * tile, seed=250409307,
                                **scenario_kwargs(args))
            dg.replay_batch(spec, start=start, fin=fin, ld=tile, span=span[ti * tile:(ti + 1) * tile],
                            rank_breakdown=bd[ti * tile:(ti + 1) * tile],
                            stream_busy=busy[ti * tile:(ti + 1) * tile], stream=sptr)
            torch.cuda.synchronize()
            return start, fin
        try:
            audit_res = audit(args, g, dg, replay_tile, first, S_local, tile,
                              bd.cpu().numpy(), span.cpu().numpy(), busy.cpu().numpy())
        except Exception as exc:  # the checker is test infrastructure
            audit_res = {"error": repr(exc)}

    # CPU baseline (rank 0, N = 1 only): the reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            R, h, cg = cpu_sample_graph(args)
            threads = cpu_threads(1.0)
            secs, count = run_cpu_sample(R, h, cg, args, 0, threads, per_thread=1)
            cpu = {"value": cg.n * count / secs, "unit": "relaxations/s", "cores": threads,
                   "kind": "reference", "host": host_info(),
                   "sample": f"{count} scenarios ({threads} threads x 1), each a full "
                             f"tracesim::simulate() of one TP replica ({cg.n} tasks) of the "
                             f"workload, {secs:.1f} s wall (durations filled outside the clock)"}
            # one thread too (two scenarios back to back)
            secs1, count1 = run_cpu_sample(R, h, cg, args, 1_000_000, 1, per_thread=2)
            cpu["single_thread"] = {"value": cg.n * count1 / secs1, "cores": 1,
                                    "sample": f"{count1} scenarios of one TP replica on 1 "
                                              f"thread, {secs1:.2f} s"}
            del h
            if not args.no_cpu_full and args.config in ("config5", "config4"):
                # the whole 4.95 M-task graph: ~5 GB and ~50 s per replay per thread
                cpu["same_config"] = cpu_full_graph(args, cpu_threads(7.0))
        except Exception as exc:  # the oracle library is test infrastructure
            cpu = {"value": None, "unit": "relaxations/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "relaxations/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (GPT-3 generator graph, random-free base durations from the "
                    "reference cost formulas; Philox-drawn scenario durations)",
            "replays_per_s": S_total / (ms_per_step / 1e3),
            "config": {"workload": f"{args.config}: {label}, {S_total}-scenario "
                                   f"{workload_kind(args)}",
                       "tasks": n, "edges": int(g.edge_from.shape[0]), "ranks": R_,
                       "scenarios": S_total, "tile": tile, "parallelism": f"scenario-shard x{world}",
                       "outputs": "start+finish of every task x scenario (HBM), span, per-rank "
                                  "breakdown, per-stream busy",
                       "l2": "no flush needed: each tile writes 16 B x tasks x tile "
                             f"= {n * tile * 16 / 1e9:.0f} GB >> 126 MB L2",
                       "graph_gen_s": round(t_gen, 2), "compile_s": round(t_compile, 2)},
            "gpu_launches": launches,
            "device_ms_per_step": {"walk": prof["walk_ms"] / args.steps,
                                   "reduce": prof["reduce_ms"] / args.steps,
                                   "other": prof["other_ms"] / args.steps,
                                   "sum": step_ms_dev},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("cluster_walk (K1x)" if args.config == "config3"
                                    else "replay_walk (K1)"), "bytes_per_launch": walk_bytes,
                         "launch_ms": walk_avg_ms, "peak_source": peak_src,
                         # also against the 8 TB/s spec figure
                         "peak_spec": 8000.0, "frac_spec": achieved / 8000.0},
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "audit": audit_res,
            "fixups_per_step": fixups,
            "wall_s": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
