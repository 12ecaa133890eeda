"""Bulk-frontier microbenchmark: one hop of sample + compact over a frontier
of 10^6 .. 4*10^6 dst vertices, so the kernels' memory throughput shows without the
per-batch latency chain that dominates at batch ~1k.  Labelled separately from bench.py.

    EG_TRACE=1 python profiles/bulk_frontier.py [--config C4] [--sizes 1000000 4000000]

Per size: device time of each phase kernel of the hop (EG_TRACE in-kernel stamps,
phases serialised), and the algorithmic bytes of SURVEY §8d's model:
16 B per (dst, r) visit (indptr pair) + 16 B per sampled edge (4 B index read, 4 B src
+ 8 B eid written) + 24 B per edge of compaction traffic, divided by the hop's kernel
time (seed split excluded: it is the batch's entry, not the hop), vs the measured HBM
peak.  Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--sizes", type=int, nargs="+", default=[1000000, 4000000])
    ap.add_argument("--fanout", type=int, default=15)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    assert os.environ.get("EG_TRACE") == "1", "run with EG_TRACE=1 (per-kernel stamps)"
    import numpy as np
    import torch

    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6450.0))
    cfg = synth.config(args.config)
    g = synth.build_host_graph(cfg, materialize_indices=True)
    ctx = Context(0, 1, 0)
    load_context(ctx, g, 1, 0, "cuda:0", features=False)
    ctx.set_profiling(True)   # trace stamps are read back for timed launches
    fo = [[args.fanout] * cfg.n_rel]
    rs = np.random.default_rng(7)
    n_t = cfg.vt_counts[cfg.seed_vt]
    off = int(cfg.offsets[cfg.seed_vt])
    out = []
    for n in args.sizes:
        seeds = torch.from_numpy(off + rs.choice(n_t, size=n, replace=False).astype(np.int64)).cuda()
        b = ctx.sample_minibatch(seeds, fo, 1, features=False)   # warm-up: plan + graph
        b.free()
        before = ctx.trace()   # accumulators are per context: deltas below
        visits = edges = 0
        for i in range(args.reps):
            b = ctx.sample_minibatch(seeds, fo, 100 + i, features=False)
            tot, _ = b.stats()
            edges += tot
            visits += n * sum(1 for r in cfg.rels if r[2] == cfg.seed_vt)
            b.free()
        after = ctx.trace()
        stages = {}
        for k, (ms, cnt) in after.items():
            ms0, c0 = before.get(k, (0.0, 0))
            if cnt > c0:
                stages[k] = 1e3 * (ms - ms0) / (cnt - c0)   # us per launch
        hop_keys = [k for k in stages if k.startswith("k.h0.") or k == "k.relabel"]
        hop_us = sum(stages[k] for k in hop_keys)
        e = edges / args.reps
        v = visits / args.reps
        alg = 16 * v + 16 * e + 24 * e
        gbs = alg / (hop_us * 1e-6) / 1e9
        out.append({"frontier": n, "edges": int(e), "hop_us": round(hop_us, 1),
                    "stages_us": {k: round(stages[k], 1) for k in hop_keys},
                    "seed_split_us": round(stages.get("k.seed", 0.0), 1),
                    "algorithmic_bytes": int(alg), "algorithmic_GBps": round(gbs, 1),
                    "frac_of_hbm_peak": round(gbs / hbm, 3),
                    "edges_per_s": round(e / (hop_us * 1e-6), 1)})
        print(json.dumps(out[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"bench": "bulk_frontier", "config": args.config, "fanout": args.fanout,
                      "hbm_peak_GBps": hbm, "model": "16 B/visit + 16 B/edge + 24 B/edge (SURVEY 8d)",
                      "results": out}))


if __name__ == "__main__":
    main()
