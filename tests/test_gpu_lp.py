"""GPU parity of link-prediction mini-batches (NEXT-3) through the C ABI: the CUDA path
(eg_sample_lp_bundle) against the oracle (og_lp_targets + og_sample), element by
element on the same seeded inputs: seeds, every block, features, negatives and pairs."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_same_batch, assert_same_features

pytestmark = pytest.mark.gpu


def _ctx(graph, world=1, rank=0, features=True):
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    ctx = Context(rank, world, 0)
    ctx._shard = load_context(ctx, graph, world, rank, "cuda:0", features=features)
    return ctx


def _features_of(blocks, cfg):
    return [blocks.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)]


def compare_lp(ctx, g, cfg, src, dst, rel, n_neg, neg_seed, fanouts, rng, rows=None, device_inputs=True,
               blocks=None):
    import torch
    res, t = oracle.sample_lp(g, src, dst, rel, n_neg, neg_seed, fanouts, rng)
    if blocks is None:
        a, b = (torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()) if device_inputs else (src, dst)
        blocks = ctx.sample_lp(a, b, rel, n_neg, neg_seed, fanouts, rng, features=rows is not None)
    assert_same_batch(res, blocks, cfg.n_vt, cfg.n_rel)
    lp = blocks.lp()
    assert lp["n_pos"] == len(src) and lp["n_neg"] == n_neg and lp["rel"] == rel
    np.testing.assert_array_equal(lp["neg_dst_gid"].cpu().numpy(), t.neg_dst)
    np.testing.assert_array_equal(lp["pos_src"].cpu().numpy(), t.pos_src)
    np.testing.assert_array_equal(lp["pos_dst"].cpu().numpy(), t.pos_dst)
    np.testing.assert_array_equal(lp["neg_src"].cpu().numpy(), t.neg_src)
    np.testing.assert_array_equal(lp["neg_dst"].cpu().numpy(), t.neg_dst_local)
    if rows is not None:
        assert_same_features(res, _features_of(blocks, cfg), cfg, rows)
    blocks.free()


@pytest.fixture(scope="module")
def c1():
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    return cfg, g, rows, _ctx(g)


@pytest.mark.parametrize("rel", [0, 1, 2])
@pytest.mark.parametrize("n_neg", [0, 1, 3])
def test_c1_lp_all_relations(c1, rel, n_neg):
    cfg, g, rows, ctx = c1
    src, dst = synth.lp_positives(cfg, g, rel, 10 * rel + n_neg, 64)
    compare_lp(ctx, g, cfg, src, dst, rel, n_neg, 1000 + rel, cfg.fanouts, 77 + n_neg, rows)


def test_c1_lp_host_inputs_and_edge_cases(c1):
    cfg, g, rows, ctx = c1
    src, dst = synth.lp_positives(cfg, g, 0, 5, 100)
    compare_lp(ctx, g, cfg, src, dst, 0, 2, 9, cfg.fanouts, 3, rows, device_inputs=False)   # pageable host
    compare_lp(ctx, g, cfg, src[:1], dst[:1], 0, 1, 9, cfg.fanouts, 3, rows)                # one positive
    compare_lp(ctx, g, cfg, src[:0], dst[:0], 0, 1, 9, cfg.fanouts, 3, rows)                # empty batch
    rep = np.repeat(src[:4], 5), np.repeat(dst[:4], 5)                                      # repeated positives
    compare_lp(ctx, g, cfg, rep[0], rep[1], 0, 4, 9, [[2, 0, -1], [1, 1, 1]], 3, rows)
    compare_lp(ctx, g, cfg, src, dst, 0, 64, 9, cfg.fanouts, 3, rows)                       # EG_MAX_NEG


def test_c1_lp_errors_then_recovers(c1):
    from paper_2112_15345_b200 import EgError
    import torch
    cfg, g, rows, ctx = c1
    src, dst = synth.lp_positives(cfg, g, 1, 7, 16)          # r1: A -> B
    bad = src.copy()
    bad[3] = int(cfg.offsets[1])                             # a type-B gid as the src of A -> B
    with pytest.raises(EgError) as e:
        ctx.sample_lp(torch.from_numpy(bad).cuda(), torch.from_numpy(dst).cuda(), 1, 1, 5, cfg.fanouts, 1)
    assert e.value.code == -2                                # EG_ERANGE
    with pytest.raises(EgError) as e:
        ctx.sample_lp(src, dst, 7, 1, 5, cfg.fanouts, 1)     # no relation 7
    assert e.value.code == -1
    with pytest.raises(EgError) as e:
        ctx.sample_lp(src, dst, 1, 65, 5, cfg.fanouts, 1)    # n_neg > EG_MAX_NEG
    assert e.value.code == -1
    compare_lp(ctx, g, cfg, src, dst, 1, 2, 5, cfg.fanouts, 1, rows)


def test_c1_node_batch_has_no_lp_view(c1):
    from paper_2112_15345_b200 import EgError
    cfg, g, rows, ctx = c1
    b = ctx.sample_minibatch(synth.batch_seeds(cfg, 0), cfg.fanouts, 1, features=False)
    with pytest.raises(EgError):
        b.lp()
    b.free()


@pytest.mark.parametrize("mode", ["default", "bitmap"])
def test_c1_lp_compaction_variants(c1, mode, monkeypatch):
    cfg, g, rows, _ = c1
    monkeypatch.setenv("EG_COMPACT", mode)
    ctx = _ctx(g)
    src, dst = synth.lp_positives(cfg, g, 2, 40, 64)
    compare_lp(ctx, g, cfg, src, dst, 2, 2, 41, cfg.fanouts, 42, rows)
    ctx.close()


def test_c1_lp_world4_invariance(c1):
    """Outputs are independent of the partition (4 ranks emulated on one GPU)."""
    cfg, g, rows, _ = c1
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    ctxs = []
    for p in range(4):
        ctx = Context(p, 4, 0)
        ctx._shard = load_context(ctx, g, 4, p, "cuda:0")
        ctxs.append(ctx)
    for a in ctxs:
        for b in ctxs:
            if a is not b:
                a.attach_peer(b)
    src, dst = synth.lp_positives(cfg, g, 0, 50, 64)
    for p in (0, 3):
        compare_lp(ctxs[p], g, cfg, src, dst, 0, 2, 51 + p, cfg.fanouts, 52, rows)


def test_c2_lp_bundle_pipelined():
    """ogbn-mag-shaped: LP fanout [25, 15], 1024 positives x 1 negative, bundles
    of 4 on 2 lanes, async: every batch bit-exact."""
    import torch
    cfg = synth.config("C2")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    ctx = _ctx(g)
    ctx.set_pipeline(2, 4)
    rel, fo = synth.lp_rel(cfg), synth.lp_fanouts(cfg)
    pend = []
    for rnd in range(3):
        idx = [4 * rnd + j for j in range(4)]
        pos = [synth.lp_positives(cfg, g, rel, i, 1024) for i in idx]
        dev = [(torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()) for s, d in pos]
        bls = ctx.sample_lp_bundle([a for a, _ in dev], [b for _, b in dev], rel, 1, [500 + i for i in idx], fo,
                                   [synth.rng_seed(cfg, i) for i in idx], features=True, async_=True)
        pend.append((idx, pos, dev, bls))
        if len(pend) == 2 or rnd == 2:
            while pend:
                idx_, pos_, _, bls_ = pend.pop(0)
                for i, (s, d), b in zip(idx_, pos_, bls_):
                    compare_lp(ctx, g, cfg, s, d, rel, 1, 500 + i, fo, synth.rng_seed(cfg, i), rows, blocks=b)
    ctx.close()


def test_c4_lp_full_size():
    """papers100M-shaped (111M vertices): 1024 positives x 1 negative, fanout [25, 15]."""
    cfg = synth.config("C4")
    g = synth.build_host_graph(cfg, materialize_indices=True)
    ctx = _ctx(g)
    rows = {0: synth.LazyRows(cfg, 0)}
    rel, fo = synth.lp_rel(cfg), synth.lp_fanouts(cfg)
    for gi in (0, 1):
        s, d = synth.lp_positives(cfg, g, rel, gi, 1024)
        compare_lp(ctx, g, cfg, s, d, rel, 1, 900 + gi, fo, synth.rng_seed(cfg, gi), rows)
    ctx.close()
