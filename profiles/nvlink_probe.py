"""NVLink counters of the multi-GPU path, in ONE process (so ncu can profile it): two
ranks of a world-2 partition on cuda:0 and cuda:1 (eg_attach_peer with peer access over
NVLink), rank 0 samples bundles of its global batches with features; half of the CSC rows
it visits and half of the feature rows it gathers live on cuda:1.

    python profiles/nvlink_probe.py [--config C4] [--launches 6] [--bundle 16]
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,... python profiles/nvlink_probe.py

Prints the batches' parity vs the oracle for the first launch (C1-C3: all rows; C4: blocks +
rows of one batch)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--bundle", type=int, default=16)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    cfg = synth.config(a.config)
    g = synth.build_host_graph(cfg, materialize_indices=a.check)
    ctxs = []
    for p in range(2):
        torch.cuda.set_device(p)
        c = Context(p, 2, p)
        c._shard = load_context(c, g, 2, p, f"cuda:{p}")
        ctxs.append(c)
    ctxs[0].attach_peer(ctxs[1])
    ctxs[1].attach_peer(ctxs[0])
    torch.cuda.set_device(0)
    ctx = ctxs[0]
    ctx.set_pipeline(1, a.bundle)
    B = a.bundle
    for l in range(a.launches):
        gis = [2 * (l * B + i) for i in range(B)]   # rank 0's global batches
        seeds = [torch.from_numpy(synth.batch_seeds(cfg, x)).cuda(0) for x in gis]
        bls = ctx.sample_bundle(seeds, cfg.fanouts, [synth.rng_seed(cfg, x) for x in gis], features=True)
        if l == 0 and a.check:
            import oracle
            from gpu_util import assert_same_batch, assert_same_features
            rows = ({u: synth.host_features(cfg, u) for u in cfg.feats} if cfg.name in ("C1", "C2", "C3")
                    else {u: synth.LazyRows(cfg, u) for u in cfg.feats})
            for x, b in list(zip(gis, bls))[:2]:
                res = oracle.sample(g, synth.batch_seeds(cfg, x), cfg.fanouts, synth.rng_seed(cfg, x))
                assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
                assert_same_features(res, [b.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)],
                                     cfg, rows)
            print("parity ok (2 batches of the first launch, rank 0 of a 2-GPU world)", flush=True)
        for b in bls:
            b.free()
    torch.cuda.synchronize(0)
    print(f"nvlink probe done: {a.config}, {a.launches} launches x {B} batches on cuda:0 with peer cuda:1", flush=True)
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    main()
