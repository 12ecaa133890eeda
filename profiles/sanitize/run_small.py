"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
C1 node batches (single, bundled on 2 lanes), link-prediction batches, the standalone
gather, emulated world 2 with peer reads, both compaction paths (EG_COMPACT=bitmap via a
second process), each batch compared with the oracle.  Exit 0 iff everything matched."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import assert_same_batch, assert_same_features  # noqa: E402
from paper_2112_15345_b200 import Context  # noqa: E402
from synth.device import load_context  # noqa: E402


def ctx_of(g, world=1, rank=0):
    c = Context(rank, world, 0)
    c._shard = load_context(c, g, world, rank, "cuda:0")
    return c


def feats(b, cfg):
    return [b.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)]


def main():
    cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C1")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    n = 0
    ctx = ctx_of(g)
    for gi in range(2):   # single batches + standalone gather
        seeds, rs = synth.batch_seeds(cfg, gi), synth.rng_seed(cfg, gi)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, feats(b, cfg), cfg, rows)
        assert_same_features(res, ctx.gather_features(b), cfg, rows)
        b.free()
        n += 1
    ctx.set_pipeline(2, 4)   # bundles on 2 lanes, async
    gis = list(range(10, 18))
    dev = [torch.from_numpy(synth.batch_seeds(cfg, x)).cuda() for x in gis]
    ls = [ctx.sample_bundle(dev[i:i + 4], cfg.fanouts, [synth.rng_seed(cfg, x) for x in gis[i:i + 4]],
                            features=True, async_=True) for i in (0, 4)]
    for li, bls in enumerate(ls):
        for j, b in enumerate(bls):
            x = gis[4 * li + j]
            res = oracle.sample(g, synth.batch_seeds(cfg, x), cfg.fanouts, synth.rng_seed(cfg, x))
            assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
            assert_same_features(res, feats(b, cfg), cfg, rows)
            b.free()
            n += 1
    rel = synth.lp_rel(cfg)   # link prediction
    src, dst = synth.lp_positives(cfg, g, rel, 3, 64)
    res, lpt = oracle.sample_lp(g, src, dst, rel, 2, 77, cfg.fanouts, 78)
    b = ctx.sample_lp(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), rel, 2, 77, cfg.fanouts, 78)
    assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
    b.free()
    n += 1
    ctx.close()
    ctxs = [ctx_of(g, 2, p) for p in range(2)]   # emulated world 2: peer CSC rows and feature rows
    ctxs[0].attach_peer(ctxs[1])
    ctxs[1].attach_peer(ctxs[0])
    for p in range(2):
        seeds, rs = synth.batch_seeds(cfg, 30 + p), synth.rng_seed(cfg, 30 + p)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        b = ctxs[p].sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, feats(b, cfg), cfg, rows)
        b.free()
        n += 1
    for c in ctxs:
        c.close()
    torch.cuda.synchronize()
    print(f"sanitize workload OK: {cfg.name}, {n} batches bit-exact, EG_COMPACT={os.environ.get('EG_COMPACT', 'default')}",
          flush=True)


if __name__ == "__main__":
    main()
