"""GPU parity of the consumer step (NEXT-4 i): eg_sage_mean_layer (tcgen05 tensor cores)
against the fp64 oracle (oracle.sage_mean_layer) on the oracle's own blocks, with the
tolerance of DESIGN.md §3 reading C2: |z_gpu - z| <= 2^-8 * (|W_self| |x_dst| +
|W_neigh| mean|x_src|) + 1e-6 per element (bf16 operands, fp32 accumulation)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_same_batch

pytestmark = pytest.mark.gpu


def _ctx(graph):
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    ctx = Context(0, 1, 0)
    ctx._shard = load_context(ctx, graph, 1, 0, "cuda:0")
    return ctx


def _bf16_weights(rng, H, K):
    import torch
    return torch.from_numpy(rng.standard_normal((H, K)).astype(np.float32) / np.sqrt(K)).to(torch.bfloat16).cuda()


def _check(z_gpu, blk, xs, xd, w, extra=None):
    """z_gpu vs the oracle layer on the oracle block `blk` (+ `extra` terms)."""
    wf = w.float().cpu().numpy().astype(np.float64)
    z = oracle.sage_mean_layer(blk.indptr, blk.indices, xs, xd, wf)
    bound = oracle.sage_mean_layer(blk.indptr, blk.indices, np.abs(xs), None if xd is None else np.abs(xd), np.abs(wf))
    if extra is not None:
        for (b2, xs2, w2) in extra:
            w2f = w2.float().cpu().numpy().astype(np.float64)
            z += oracle.sage_mean_layer(b2.indptr, b2.indices, xs2, None, w2f)
            bound += oracle.sage_mean_layer(b2.indptr, b2.indices, np.abs(xs2), None, np.abs(w2f))
    got = z_gpu.cpu().numpy().astype(np.float64)
    assert got.shape == z.shape
    err = np.abs(got - z)
    tol = 2.0 ** -8 * bound + 1e-6
    assert np.all(err <= tol), f"max err {err.max():.3e}, worst ratio {(err / tol).max():.3f}"
    return float((err / tol).max())


def _batch(ctx, g, cfg, gi, fanouts=None):
    import torch
    fo = cfg.fanouts if fanouts is None else fanouts
    seeds = synth.batch_seeds(cfg, gi)
    rs = synth.rng_seed(cfg, gi)
    res = oracle.sample(g, seeds, fo, rs)
    b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), fo, rs, features=True)
    assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
    return res, b


def test_c1_sage_all_relations_f16_features_fp32():
    """C1: 16-d fp32 rows (F padded to 64), H = 32 / 48; every relation of the input
    layer, with and without the self term."""
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    ctx = _ctx(g)
    res, b = _batch(ctx, g, cfg, 0)
    L = len(cfg.fanouts)
    rng = np.random.default_rng(0)
    for r, (_, s, t, _) in enumerate(cfg.rels):
        xs_t = b.features(s)
        xd_t = b.features(t)[:b[L - 1].n_dst[t]]
        xs = oracle.gather(res, cfg.vt_counts, s, rows[s]).astype(np.float64)
        xd = oracle.gather(res, cfg.vt_counts, t, rows[t])[:len(res.dst_nodes(L - 1, t))].astype(np.float64)
        for H in (32, 48):
            w = _bf16_weights(rng, H, 2 * 16)
            z = ctx.sage_mean_layer(b, L - 1, r, xs_t, w, x_dst=xd_t)
            _check(z, res.blocks[L - 1][r], xs, xd, w)
            w1 = _bf16_weights(rng, H, 16)
            z1 = ctx.sage_mean_layer(b, L - 1, r, xs_t, w1)
            _check(z1, res.blocks[L - 1][r], xs, None, w1)
    b.free()
    ctx.close()


def test_c2_sage_rgcn_sum_fp32_and_bf16():
    """C2 (ogbn-mag-shaped, 128-d fp32): paper dst of the input layer, H = 256:
    z = SAGE(cites, self) + SAGE(writes, no self, accumulate) -- the RGCN-style sum over
    relations into one type; again with bf16 inputs."""
    import torch
    cfg = synth.config("C2")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    ctx = _ctx(g)
    res, b = _batch(ctx, g, cfg, 1)
    L = len(cfg.fanouts)
    rng = np.random.default_rng(1)
    paper, author = 0, 1
    r_cites, r_writes = 0, 1
    xs_p = oracle.gather(res, cfg.vt_counts, paper, rows[paper]).astype(np.float64)
    xs_a = oracle.gather(res, cfg.vt_counts, author, rows[author]).astype(np.float64)
    n_dst = len(res.dst_nodes(L - 1, paper))
    w = _bf16_weights(rng, 256, 256)
    w2 = _bf16_weights(rng, 256, 128)
    for dt in (torch.float32, torch.bfloat16):
        fp, fa = b.features(paper).to(dt), b.features(author).to(dt)
        z = ctx.sage_mean_layer(b, L - 1, r_cites, fp, w, x_dst=fp[:n_dst])
        ctx.sage_mean_layer(b, L - 1, r_writes, fa, w2, out=z, accumulate=True)
        xp = fp.float().cpu().numpy().astype(np.float64)
        xa = fa.float().cpu().numpy().astype(np.float64)
        if dt == torch.float32:
            assert np.array_equal(xp, xs_p) and np.array_equal(xa, xs_a)
        _check(z, res.blocks[L - 1][r_cites], xp, xp[:n_dst], w, extra=[(res.blocks[L - 1][r_writes], xa, w2)])
    # hop 0 (the seeds' block): dst = the seeds, src = level 1
    w0 = _bf16_weights(rng, 128, 256)
    x1 = torch.from_numpy(rng.standard_normal((b[0].n_src[paper], 128)).astype(np.float32)).cuda()
    z0 = ctx.sage_mean_layer(b, 0, r_cites, x1, w0, x_dst=x1[:b[0].n_dst[paper]])
    x1n = x1.cpu().numpy().astype(np.float64)
    _check(z0, res.blocks[0][r_cites], x1n, x1n[:len(res.dst_nodes(0, paper))], w0)
    b.free()
    ctx.close()


def test_c4_sage_fp16_input_layer():
    """C4 (papers100M-shaped, 128-d fp16 rows): the input layer of a full batch, H = 128."""
    import torch
    cfg = synth.config("C4")
    g = synth.build_host_graph(cfg, materialize_indices=True)
    ctx = _ctx(g)
    res, b = _batch(ctx, g, cfg, 0)
    L = len(cfg.fanouts)
    xs_t = b.features(0)
    n_dst = b[L - 1].n_dst[0]
    xs = synth.LazyRows(cfg, 0).take(res.input_nodes(0)).astype(np.float64)
    assert np.array_equal(xs_t.float().cpu().numpy().astype(np.float64), xs)
    w = _bf16_weights(np.random.default_rng(4), 128, 256)
    z = ctx.sage_mean_layer(b, L - 1, 0, xs_t, w, x_dst=xs_t[:n_dst])
    _check(z, res.blocks[L - 1][0], xs, xs[:n_dst], w)
    b.free()
    ctx.close()


def test_sage_argument_errors():
    import torch
    from paper_2112_15345_b200 import EgError
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    ctx = _ctx(g)
    res, b = _batch(ctx, g, cfg, 2)
    x = b.features(0)
    with pytest.raises(EgError):
        ctx.sage_mean_layer(b, 0, 0, x, _bf16_weights(np.random.default_rng(0), 24, 32), x_dst=x)   # H % 16
    with pytest.raises(EgError):
        ctx.sage_mean_layer(b, 5, 0, x, _bf16_weights(np.random.default_rng(0), 32, 32), x_dst=x)   # hop
    b.free()
    ctx.close()
