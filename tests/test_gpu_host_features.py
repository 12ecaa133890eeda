"""Feature rows in pinned host memory, gathered zero-copy over PCIe (SURVEY §8f NEXT-4 ii;
the paper keeps graph data in CPU memory): the gathered bytes equal
the oracle's, for node and link-prediction batches, bundled and single; the library
rejects pageable host rows and host rows at world > 1."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_same_batch, assert_same_features

pytestmark = pytest.mark.gpu


def _ctx(graph, features, world=1, rank=0):
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    ctx = Context(rank, world, 0)
    ctx._shard = load_context(ctx, graph, world, rank, "cuda:0", features=features)
    return ctx


def _features_of(blocks, cfg):
    return [blocks.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)]


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_host_feature_rows_match_oracle(name):
    import torch
    cfg = synth.config(name)
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    ctx = _ctx(g, "host")
    assert all(ctx._shard["feats"][u].is_pinned() for u in cfg.feats)
    for gi in (0, 1):
        seeds = synth.batch_seeds(cfg, gi)
        rs = synth.rng_seed(cfg, gi)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        # the standalone gather entry point reads the same host rows
        outs = ctx.gather_features(b)
        assert_same_features(res, outs, cfg, rows)
        b.free()
    # a bundle of 3 on 2 lanes, async
    ctx.set_pipeline(2, 4)
    idx = [10, 11, 12]
    dev = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in idx]
    bls = ctx.sample_bundle(dev, cfg.fanouts, [synth.rng_seed(cfg, i) for i in idx], features=True, async_=True)
    for i, b in zip(idx, bls):
        res = oracle.sample(g, synth.batch_seeds(cfg, i), cfg.fanouts, synth.rng_seed(cfg, i))
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        b.free()
    # link prediction over host rows
    rel = synth.lp_rel(cfg)
    s, d = synth.lp_positives(cfg, g, rel, 3, 256)
    res, _ = oracle.sample_lp(g, s, d, rel, 1, 7, synth.lp_fanouts(cfg), 8)
    b = ctx.sample_lp(s, d, rel, 1, 7, synth.lp_fanouts(cfg), 8, features=True)
    assert_same_features(res, _features_of(b, cfg), cfg, rows)
    b.free()
    ctx.close()


def test_pageable_host_rows_rejected():
    import torch
    from paper_2112_15345_b200 import Context, EgError
    from synth.device import device_shard
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    sh = device_shard(g, 1, 0, "cuda:0", features=True)
    sh["feats"] = [f.cpu() if f is not None else None for f in sh["feats"]]   # pageable
    ctx = Context(0, 1, 0)
    with pytest.raises(EgError) as e:
        ctx.load_partition(sh["vt_counts"], sh["rels"], sh["feats"], bounds=sh["bounds"])
    assert e.value.code == -1
    ctx.close()


def test_host_rows_need_world_1():
    from paper_2112_15345_b200 import EgError
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    with pytest.raises(EgError) as e:
        _ctx(g, "host", world=2, rank=0)
    assert e.value.code == -1
