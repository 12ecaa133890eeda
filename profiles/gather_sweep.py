"""Gather bandwidth vs batch size (one GPU, pipeline depth 1).

    EG_GATHER=tma|ldg python profiles/gather_sweep.py [--config C2] [--batches 1024 4096 16384]

For each batch size, times the gather node of the batch graph with the library's
CUDA events and reports algorithmic GB/s (2 * row bytes + 8 B per input row) --
separating the kernel's asymptotic throughput from its ramp / tail at small sizes.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batches", type=int, nargs="+", default=[1024, 4096, 16384, 65536])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context

    cfg = synth.config(args.config)
    g = synth.build_host_graph(cfg)
    ctx = Context(0, 1, 0)
    shard = load_context(ctx, g, 1, 0, "cuda:0")
    out = []
    for B in args.batches:
        seeds = [torch.from_numpy(synth.batch_seeds(cfg, i, batch=B)).cuda() for i in range(args.reps + 2)]
        rows_bytes = 0
        for i in range(2):
            ctx.sample_minibatch(seeds[i], cfg.fanouts, i, features=True).free()
        ctx.profile()
        ctx.set_profiling(True)
        for i in range(2, args.reps + 2):
            b = ctx.sample_minibatch(seeds[i], cfg.fanouts, i, features=True)
            rows_bytes += sum(b.n_inputs(u) * (2 * cfg.row_bytes(u) + 8) for u in cfg.feats)
            b.free()
        ctx.set_profiling(False)
        p = ctx.profile()
        ms = p["gather_ms"] / p["n_gather"]
        gbps = rows_bytes / args.reps / (ms / 1e3) / 1e9
        out.append({"batch": B, "gather_ms": ms, "bytes_per_launch": rows_bytes / args.reps, "GBps": gbps,
                    "sample_ms": p["sample_ms"] / p["n_sample"]})
        print(json.dumps(out[-1]), flush=True)
    ctx.close()
    del shard
    print(json.dumps({"config": args.config, "mode": os.environ.get("EG_GATHER", "tma"), "sweep": out}))


if __name__ == "__main__":
    main()
