"""Gather launches of the bench workload, for ncu (the 60 % gather bar is
measured on the local gather kernel at P=1 on C4 and C3).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        -k regex:gather_ldg --csv --log-file gpurun_out/gather_probe.csv \\
        python profiles/gather_probe.py --configs C3 C4

Per config: --launches bundles of 8 batches (the bench's bundle), each one gather
launch; prints the algorithmic bytes of each launch (2 * row bytes + 8 B per input row)
so that the ncu DRAM bytes and duration can be set beside them.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["C3", "C4"])
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--bundle", type=int, default=8)
    args = ap.parse_args()
    import torch

    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context

    for name in args.configs:
        cfg = synth.config(name)
        g = synth.build_host_graph(cfg, materialize_indices=True)
        ctx = Context(0, 1, 0)
        shard = load_context(ctx, g, 1, 0, "cuda:0", features=True)
        ctx.set_pipeline(1, args.bundle)
        for L in range(args.launches):
            idx = [L * args.bundle + j for j in range(args.bundle)]
            dev = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in idx]
            bls = ctx.sample_bundle(dev, cfg.fanouts, [synth.rng_seed(cfg, i) for i in idx], features=True)
            alg = 0
            for b in bls:
                _, n_in = b.stats()
                alg += sum(n_in[u] * (2 * cfg.row_bytes(u) + 8) for u in range(cfg.n_vt) if cfg.row_bytes(u))
                b.free()
            print(json.dumps({"config": name, "launch": L, "algorithmic_bytes": alg}), flush=True)
        ctx.close()
        del shard


if __name__ == "__main__":
    main()
