"""Trace-ingest speed (development tool): writes the reference generator's
per-rank Chrome traces of a GPT-3 175B pp4 dp16 m32 iteration (64 ranks,
~620k events) to a temp directory, then times the native parallel ingest
(ts_ingest_traces) against the reference's own sequential path
(load_multirank + build_graph + merge_ranks) and checks they agree.
Usage: python tools/ingest_probe.py [threads]"""
import glob
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import refshim as R  # noqa: E402
from paper_2504_09307_b200.synth import ingest_traces  # noqa: E402


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    d = tempfile.mkdtemp()
    t = time.time()
    k = R.write_rank_traces(R.synth_spec(pp=4, dp=16, m=32, layers=96, d_model=12288,
                                         d_ffn=49152, heads=96), d)
    paths = sorted(glob.glob(os.path.join(d, "rank_*.json")))
    mb = sum(os.path.getsize(p) for p in paths) / 1e6
    print(f"{k} rank traces, {mb:.0f} MB JSON, written in {time.time() - t:.1f} s", flush=True)
    t = time.time()
    g = ingest_traces(paths, threads=threads)
    ours = time.time() - t
    t = time.time()
    h = R.ingest_traces(paths)
    ref = time.time() - t
    r = h.export()
    same = all(np.array_equal(getattr(g, f), getattr(r, f))
               for f in ("duration", "original_start", "edge_from", "edge_to", "lane", "rank"))
    print(f"native ingest ({threads or os.cpu_count()} threads): {ours:.2f} s; reference "
          f"(sequential): {ref:.2f} s; speed-up {ref / ours:.1f}x; {g.n} tasks; identical: {same}")
    for p in paths:
        os.unlink(p)
    os.rmdir(d)


if __name__ == "__main__":
    main()
