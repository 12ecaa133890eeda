"""How many of a launch's input rows repeat across the mini-batches of a bundle (C4 / C3 / C2):
rows gathered per launch vs distinct vertices among them (an upper bound on what a
bundle-level dedup of (remote) row reads could save).

    python profiles/dup_probe.py [--config C4] [--bundle 32]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--bundle", type=int, default=32)
    a = ap.parse_args()
    import torch

    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    cfg = synth.config(a.config)
    g = synth.build_host_graph(cfg, materialize_indices=cfg.name in ("C1", "C2", "C3"))
    ctx = Context(0, 1, 0)
    shard = load_context(ctx, g, 1, 0, "cuda:0", features=False)
    ctx.set_pipeline(1, a.bundle)
    dev = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in range(a.bundle)]
    bls = ctx.sample_bundle(dev, cfg.fanouts, [synth.rng_seed(cfg, i) for i in range(a.bundle)], features=False)
    out = {"config": cfg.name, "bundle": a.bundle, "types": {}}
    for u in range(cfg.n_vt):
        if u not in cfg.feats:
            continue
        ids = torch.cat([b[b.n_hops - 1].src_nodes[u] for b in bls])
        n, d = int(ids.numel()), int(torch.unique(ids).numel())
        out["types"][cfg.vtypes[u][0]] = {"rows": n, "distinct": d, "dup_share": 1 - d / max(1, n),
                                           "rows_per_batch": n / a.bundle}
    for b in bls:
        b.free()
    print(json.dumps(out))
    ctx.close()
    del shard


if __name__ == "__main__":
    main()
