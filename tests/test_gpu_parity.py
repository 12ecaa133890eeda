"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle, bit-exact.

Sampled edge lists (eids + relabelled src ids), block CSCs, node lists and
gathered feature bytes are compared element by element on the same seeded
inputs (synth/), for the configs' own shapes and fanouts and for the edge cases
of the method (fanout -1 / 0, d <= k, k > the fast-path limit, hubs, empty and
mixed-type seeds, errors), and at world sizes 1..8 (P-invariance, DESIGN §3 #13).
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_same_batch, assert_same_features, run_and_compare

pytestmark = pytest.mark.gpu


def _ctx(graph, world=1, rank=0, features=True, replicate="none"):
    from paper_2112_15345_b200 import Context
    from synth.device import load_context
    ctx = Context(rank, world, 0)
    shard = load_context(ctx, graph, world, rank, "cuda:0", features=features, replicate=replicate)
    ctx._shard = shard
    return ctx


def _world(graph, world, features=True, replicate="none"):
    """All ranks of a world in this process on one GPU, mapped to each other."""
    ctxs = [_ctx(graph, world, p, features, replicate) for p in range(world)]
    for a in ctxs:
        for b in ctxs:
            if a is not b:
                a.attach_peer(b)
    return ctxs


@pytest.fixture(scope="module")
def c1():
    cfg = synth.config("C1")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    return cfg, g, rows, _ctx(g)


@pytest.fixture(scope="module")
def c2():
    cfg = synth.config("C2")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    return cfg, g, rows, _ctx(g)


# ----------------------------------------------------------------------------- C1

@pytest.mark.parametrize("g_idx", range(6))
def test_c1_batches(c1, g_idx):
    cfg, g, rows, ctx = c1
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, g_idx), cfg.fanouts, synth.rng_seed(cfg, g_idx), rows,
                    check_invariants=True)


@pytest.mark.parametrize("fanouts", [
    [[-1, -1, -1], [-1, -1, -1]],          # full neighbourhoods (BFS closed form)
    [[0, 0, 0]],                           # no edges
    [[-1, 3, 0], [2, -1, 5]],              # mixed
    [[1, 1, 1], [1, 1, 1], [1, 1, 1]],     # 3 hops of k = 1
    [[150, 150, 150]],                     # k > fast-path limit (generic selection)
    [[113, 40, 112]],                      # around the fast-path boundary
    [[2, 1, 2]] * 8,                       # EG_MAX_HOPS hops
    [[33, 32, 31], [5, 4, 6]],             # around the lower half of a tiny item (d <= 32)
    [[65, 64, 63], [40, 33, 20]],          # around the tiny-selection bound (d <= 64)
])
def test_c1_fanouts(c1, fanouts):
    cfg, g, rows, ctx = c1
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 3)[:32], fanouts, 777, rows, check_invariants=True)


def test_c1_mixed_type_seeds_and_order(c1):
    cfg, g, rows, ctx = c1
    seeds = np.array([6000 + 5, 17, 6000 + 1, 3, 5999, 6000 + 3999, 0], np.int64)
    run_and_compare(ctx, g, cfg, seeds, cfg.fanouts, 9, rows, check_invariants=True)


def test_c1_empty_and_single(c1):
    cfg, g, rows, ctx = c1
    run_and_compare(ctx, g, cfg, np.zeros(0, np.int64), cfg.fanouts, 1, rows)
    run_and_compare(ctx, g, cfg, np.array([42], np.int64), cfg.fanouts, 2, rows)


def test_c1_large_batch_all_type_a(c1):
    # every type-A vertex as a seed: many tiles in every kernel
    cfg, g, rows, ctx = c1
    seeds = np.random.default_rng(0).permutation(6000).astype(np.int64)
    run_and_compare(ctx, g, cfg, seeds, cfg.fanouts, 31337, rows, check_invariants=True)


def test_c1_errors_then_recovers(c1):
    from paper_2112_15345_b200 import EgError
    import torch
    cfg, g, rows, ctx = c1
    with pytest.raises(EgError) as e:
        ctx.sample_blocks(torch.tensor([5, 10_000], device="cuda:0"), cfg.fanouts, 0)
    assert e.value.code == -2                                  # EG_ERANGE
    with pytest.raises(EgError) as e:
        ctx.sample_blocks(torch.tensor([5, 7, 5], device="cuda:0"), cfg.fanouts, 0)
    assert e.value.code == -1                                  # EG_EINVAL (duplicate)
    with pytest.raises(EgError):
        ctx.sample_blocks(torch.tensor([5], device="cuda:0"), [[5, -2, 5]], 0)
    # the per-context compaction state is clean again
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 1), cfg.fanouts, synth.rng_seed(cfg, 1), rows)


def test_c1_host_seeds_and_host_output(c1):
    cfg, g, rows, ctx = c1
    seeds = synth.batch_seeds(cfg, 4)
    rs = synth.rng_seed(cfg, 4)
    res = oracle.sample(g, seeds, cfg.fanouts, rs)
    blocks = ctx.sample_blocks(seeds, cfg.fanouts, rs)            # numpy host seeds
    assert_same_batch(res, blocks, cfg.n_vt, cfg.n_rel)
    outs = [np.empty((blocks.n_inputs(u), 16), np.float32) for u in range(2)]
    ctx.gather_features(blocks, out=outs)                          # host outputs
    for u in range(2):
        assert outs[u].tobytes() == oracle.gather(res, cfg.vt_counts, u, rows[u]).tobytes()


def test_c1_deterministic(c1):
    import torch
    cfg, g, rows, ctx = c1
    s = torch.from_numpy(synth.batch_seeds(cfg, 5)).cuda()
    a = ctx.sample_blocks(s, cfg.fanouts, 5)
    b = ctx.sample_blocks(s, cfg.fanouts, 5)
    for h in range(2):
        for r in range(3):
            assert torch.equal(a[h].eids[r], b[h].eids[r]) and torch.equal(a[h].indices[r], b[h].indices[r])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_c1_world_invariance(c1, world):
    cfg, g, rows, _ = c1
    ctxs = _world(g, world)
    for p, ctx in enumerate(ctxs):
        gi = p + 10
        run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, gi), cfg.fanouts, synth.rng_seed(cfg, gi), rows)


# ----------------------------------------------------------------------------- C2 (bench workload)

@pytest.mark.parametrize("g_idx", range(3))
def test_c2_full_batches(c2, g_idx):
    cfg, g, rows, ctx = c2
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, g_idx), cfg.fanouts, synth.rng_seed(cfg, g_idx), rows,
                    check_invariants=(g_idx == 0))


def test_c2_world4_invariance(c2):
    cfg, g, rows, _ = c2
    ctxs = _world(g, 4)
    for p in (0, 3):
        run_and_compare(ctxs[p], g, cfg, synth.batch_seeds(cfg, 20 + p), cfg.fanouts, synth.rng_seed(cfg, 20 + p),
                        rows)


# ----------------------------------------------------------------------------- replicated feature types

@pytest.mark.parametrize("world", [2, 4])
def test_c2_replicated_small_types(c2, world):
    """Replicated partition policy for the small types (institution, field):
    same bytes as the sharded policy, standalone gather and the graph path."""
    import torch
    from synth.device import replica_types
    cfg, g, rows, _ = c2
    assert replica_types(cfg, world) == [2, 3]
    ctxs = _world(g, world, replicate="auto")
    for p in (0, world - 1):
        gi = 40 + p
        seeds, rs = synth.batch_seeds(cfg, gi), synth.rng_seed(cfg, gi)
        run_and_compare(ctxs[p], g, cfg, seeds, cfg.fanouts, rs, rows)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        b = ctxs[p].sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        b.free()

def test_c2_replicated_fit_all_types(c2):
    """The "fit" policy replicates every C2 feature table (0.99 GB): the gather reads only local
    rows at world 2 and the bytes equal the oracle's."""
    from synth.device import replica_types
    cfg, g, rows, _ = c2
    assert replica_types(cfg, 2, "fit") == [0, 1, 2, 3]
    ctxs = _world(g, 2, replicate="fit")
    for p in (0, 1):
        gi = 60 + p
        run_and_compare(ctxs[p], g, cfg, synth.batch_seeds(cfg, gi), cfg.fanouts, synth.rng_seed(cfg, gi), rows)



def test_replica_is_what_the_gather_reads(c1):
    """Negative control: a replica whose bytes differ from the shards shows up in the
    output for that type only (so the policy is really applied), and the API errors."""
    import torch
    from paper_2112_15345_b200 import EgError
    cfg, g, rows, _ = c1
    ctxs = _world(g, 2)
    n0 = int(cfg.vt_counts[0])
    fake = torch.full((n0, cfg.feats[0][0]), 7.0, dtype=torch.float32, device="cuda:0")
    with pytest.raises(EgError):
        ctxs[0].set_feature_replica(0, fake[:-1])                    # not all N_t rows
    with pytest.raises(EgError):
        ctxs[0].set_feature_replica(0, fake.cpu())                   # not device memory
    with pytest.raises(EgError):
        ctxs[0].set_feature_replica(5, fake)                         # type out of range
    ctxs[0].set_feature_replica(0, fake)
    seeds, rs = synth.batch_seeds(cfg, 3), synth.rng_seed(cfg, 3)
    res = oracle.sample(g, seeds, cfg.fanouts, rs)
    b = ctxs[0].sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
    f = _features_of(b, cfg)
    assert torch.all(f[0] == 7.0) and f[0].shape[0] == len(res.input_nodes(0))
    want1 = oracle.gather(res, cfg.vt_counts, 1, rows[1])
    assert f[1].cpu().numpy().tobytes() == want1.tobytes()
    b.free()
    with pytest.raises(EgError):
        ctxs[0].set_feature_replica(0, None)                         # after the first sampling call


def test_gather_kernel_choice(c1, c2):
    """The default gather is the TMA kernel (tile::gather4) wherever every requested type
    has a local table with a gather4 map, and at world > 1 (peer rows by bulk copies);
    its output was compared with the oracle by the tests above / below."""
    import os

    import torch
    if os.environ.get("EG_GATHER", "auto") != "auto":
        pytest.skip("gather kernel forced by EG_GATHER")
    for cfg, g, rows, ctx in (c1, c2):
        seeds, rs = synth.batch_seeds(cfg, 5), synth.rng_seed(cfg, 5)
        b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        b.free()
        assert ctx.gather_path() == "tma", cfg.name
    cfg, g, rows, _ = c2
    ctxs = _world(g, 2)
    seeds, rs = synth.batch_seeds(cfg, 6), synth.rng_seed(cfg, 6)
    b = ctxs[1].sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
    assert_same_features(oracle.sample(g, seeds, cfg.fanouts, rs), _features_of(b, cfg), cfg, rows)
    b.free()
    assert ctxs[1].gather_path() == "tma"


# ----------------------------------------------------------------------------- C3 (3 hops, hub of degree 618k)

def test_c3_full_batch():
    cfg = synth.config("C3")
    g = synth.build_host_graph(cfg)
    rows = {0: synth.host_features(cfg, 0)}
    ctx = _ctx(g)
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 0), cfg.fanouts, synth.rng_seed(cfg, 0), rows)
    # the hub (max in-degree) as a seed: selection over 6e5 keys
    hub = int(np.argmax(np.diff(g.indptr[0])))
    run_and_compare(ctx, g, cfg, np.array([hub, 1, 2], np.int64), cfg.fanouts, 123, rows)


def test_device_features_match_host_generator():
    import torch
    from synth.device import feature_shard
    for name in ("C1", "C4"):
        cfg = synth.config(name)
        t = feature_shard(cfg, 0, 1000, 3000, "cuda:0")
        torch.cuda.synchronize()
        assert t.cpu().numpy().tobytes() == synth.host_features(cfg, 0, 1000, 3000).tobytes()


# ----------------------------------------------------------------------------- one-graph mini-batch path

def _features_of(blocks, cfg):
    return [blocks.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)]


@pytest.mark.parametrize("g_idx", range(3))
def test_c1_minibatch_graph_with_features(c1, g_idx):
    cfg, g, rows, ctx = c1
    seeds = synth.batch_seeds(cfg, g_idx)
    rs = synth.rng_seed(cfg, g_idx)
    res = oracle.sample(g, seeds, cfg.fanouts, rs)
    import torch
    b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
    assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
    assert_same_features(res, _features_of(b, cfg), cfg, rows)
    b.free()


def test_c2_async_pipeline(c2):
    """Several batches in flight (EG_ASYNC), each bit-exact; slots are reused."""
    import torch
    cfg, g, rows, ctx = c2
    idx = list(range(30, 36))
    seeds = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in idx]
    pend = [ctx.sample_minibatch(s, cfg.fanouts, synth.rng_seed(cfg, i), features=True, async_=True)
            for s, i in zip(seeds[:3], idx[:3])]
    for k, i in enumerate(idx):
        b = pend.pop(0)
        res = oracle.sample(g, synth.batch_seeds(cfg, i), cfg.fanouts, synth.rng_seed(cfg, i))
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        b.free()
        if k + 3 < len(idx):
            pend.append(ctx.sample_minibatch(seeds[k + 3], cfg.fanouts, synth.rng_seed(cfg, idx[k + 3]),
                                             features=True, async_=True))


def test_c1_async_error_reported_at_wait(c1):
    from paper_2112_15345_b200 import EgError
    import torch
    cfg, g, rows, ctx = c1
    bad = torch.tensor([3, 99999], device="cuda:0")
    b = ctx.sample_minibatch(bad, cfg.fanouts, 1, async_=True)
    with pytest.raises(EgError) as e:
        b.wait()
    assert e.value.code == -2
    b.free()
    run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 2), cfg.fanouts, synth.rng_seed(cfg, 2), rows)


def test_c1_batch_sizes_share_and_split_plans(c1):
    """Different seed counts / fanouts use different plans; results stay exact."""
    cfg, g, rows, ctx = c1
    for n, fo in [(1, cfg.fanouts), (63, cfg.fanouts), (65, cfg.fanouts), (200, [[2, 3, 4], [4, 3, 2]]),
                  (64, cfg.fanouts)]:
        run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 7, batch=n), fo, 1000 + n, rows)


def test_c2_pipeline_depth4_concurrent_lanes(c2):
    """Four batches in flight on four lanes (streams + compaction state): each bit-exact."""
    import torch
    cfg, g, rows, ctx = c2
    ctx.set_pipeline(4)
    try:
        idx = list(range(40, 52))
        seeds = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in idx]
        pend = []
        for k, i in enumerate(idx):
            pend.append((i, ctx.sample_minibatch(seeds[k], cfg.fanouts, synth.rng_seed(cfg, i), features=True,
                                                 async_=True)))
            if len(pend) == 4 or k == len(idx) - 1:
                while pend:
                    j, b = pend.pop(0)
                    res = oracle.sample(g, synth.batch_seeds(cfg, j), cfg.fanouts, synth.rng_seed(cfg, j))
                    assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
                    assert_same_features(res, _features_of(b, cfg), cfg, rows)
                    b.free()
    finally:
        ctx.set_pipeline(1)


# ----------------------------------------------------------------------------- the bench's launch configuration

@pytest.mark.parametrize("name", ["C2", "C4"])
@pytest.mark.parametrize("depth,bundle", [(4, 8), (4, 32), (6, 32)])
def test_bench_launch_configuration(name, depth, bundle):
    """Exactly what bench.py times: `depth` lanes x bundles of `bundle`, async, `depth`
    launches in flight; batches g = 0..depth*bundle-1 as the bench draws them (rank 0 of
    world 1), each checked against the oracle (C2: all with features; C4: one batch per
    bundle, blocks + features via the generator formula)."""
    import torch
    cfg = synth.config(name)
    g = synth.build_host_graph(cfg, materialize_indices=True)
    rows = ({u: synth.host_features(cfg, u) for u in cfg.feats} if name == "C2"
            else {0: synth.LazyRows(cfg, 0)})
    ctx = _ctx(g)
    ctx.set_pipeline(depth, bundle)
    n = depth * bundle
    seeds = [torch.from_numpy(synth.batch_seeds(cfg, b)).cuda() for b in range(n)]
    rngs = [synth.rng_seed(cfg, b) for b in range(n)]
    launches = [ctx.sample_bundle(seeds[b0:b0 + bundle], cfg.fanouts, rngs[b0:b0 + bundle], features=True,
                                  async_=True)
                for b0 in range(0, n, bundle)]                  # `depth` launches in flight on `depth` lanes
    for k, bls in enumerate(launches):
        for j, b in enumerate(bls):
            gi = bundle * k + j
            if name == "C2" or j == k:
                res = oracle.sample(g, synth.batch_seeds(cfg, gi), cfg.fanouts, rngs[gi])
                assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
                assert_same_features(res, _features_of(b, cfg), cfg, rows)
            b.free()
    ctx.close()
    del launches, ctx


# ----------------------------------------------------------------------------- compaction variants

@pytest.mark.parametrize("mode", ["default", "bitmap"])
def test_compaction_variant_forced(c1, c2, mode, monkeypatch):
    """Both compaction paths (compact.cuh: runs of small buckets sorted in shared memory,
    big buckets by a per-warp bitmap; EG_COMPACT=bitmap makes every bucket a task of its own
    on the bitmap path) give the oracle's blocks on C1 and C2, alone and in a bundle of 3."""
    import torch
    monkeypatch.setenv("EG_COMPACT", mode)   # read at context creation
    for cfg, g, rows, _ in (c1, c2):
        ctx = _ctx(g)
        for gi in (0, 1):
            run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 100 + gi), cfg.fanouts, synth.rng_seed(cfg, 100 + gi),
                            rows, check_invariants=(gi == 0))
        ctx.set_pipeline(1, 4)
        idx = [110, 111, 112]
        seeds = [synth.batch_seeds(cfg, i) for i in idx]
        rs = [synth.rng_seed(cfg, i) for i in idx]
        dev = [torch.from_numpy(x).cuda() for x in seeds]
        bls = ctx.sample_bundle(dev, cfg.fanouts, rs, features=True)
        for x, r, b in zip(seeds, rs, bls):
            res = oracle.sample(g, x, cfg.fanouts, r)
            assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
            assert_same_features(res, _features_of(b, cfg), cfg, rows)
            b.free()
        ctx.close()


@pytest.mark.parametrize("bshift", ["10", "11", "13"])
def test_bucket_width_override(c1, c2, bshift, monkeypatch):
    """Compaction bucket widths other than the load-time rule's (C1 2^10, C2 2^12): narrow
    buckets (many per type, most tasks on the sort path) and wide ones (2^13, more big buckets
    on the bitmap path) give the oracle's blocks, alone and in a bundle of 3 (EG_BSHIFT)."""
    import torch
    monkeypatch.setenv("EG_BSHIFT", bshift)   # read at eg_load_partition
    for cfg, g, rows, _ in (c1, c2):
        ctx = _ctx(g)
        for gi in (0, 1):
            run_and_compare(ctx, g, cfg, synth.batch_seeds(cfg, 120 + gi), cfg.fanouts, synth.rng_seed(cfg, 120 + gi),
                            rows, check_invariants=(gi == 0))
        ctx.set_pipeline(1, 4)
        idx = [130, 131, 132]
        dev = [torch.from_numpy(synth.batch_seeds(cfg, i)).cuda() for i in idx]
        bls = ctx.sample_bundle(dev, cfg.fanouts, [synth.rng_seed(cfg, i) for i in idx], features=True)
        for i, b in zip(idx, bls):
            res = oracle.sample(g, synth.batch_seeds(cfg, i), cfg.fanouts, synth.rng_seed(cfg, i))
            assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
            assert_same_features(res, _features_of(b, cfg), cfg, rows)
            b.free()
        ctx.close()


# ----------------------------------------------------------------------------- planted communities (NEXT-2)

def test_c1l_planted_world2_confined_seeds():
    """C1L (planted communities) at world 2 with each rank's seeds confined to its own
    range: every batch bit-exact (the locality-aware partition changes inputs, not the
    method)."""
    cfg = synth.config("C1L")
    g = synth.build_host_graph(cfg)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats}
    ctxs = _world(g, 2)
    for p in range(2):
        for b in range(3):
            seeds = synth.batch_seeds_confined(cfg, b, p, 2)
            run_and_compare(ctxs[p], g, cfg, seeds, cfg.fanouts, synth.rng_seed(cfg, 2 * b + p), rows,
                            check_invariants=(b == 0))


# ----------------------------------------------------------------------------- C4 / C5 (full size)

def test_c4_full_size_batches():
    """ogbn-papers100M-shaped: 111M vertices, 1.6B edges, 3 hops, 256-B fp16 rows (28 GB on
    the GPU).  Blocks bit-exact vs the oracle; feature bytes vs the generator formula."""
    import torch
    cfg = synth.config("C4")
    g = synth.build_host_graph(cfg, materialize_indices=True)
    ctx = _ctx(g)
    rows = {0: synth.LazyRows(cfg, 0)}
    for gi in (0, 1):
        seeds = synth.batch_seeds(cfg, gi)
        rs = synth.rng_seed(cfg, gi)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=True)
        assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, _features_of(b, cfg), cfg, rows)
        b.free()
    hub = int(np.argmax(np.diff(g.indptr[0])))     # in-degree 2^20: selection over 1M keys
    run_and_compare(ctx, g, cfg, np.array([hub, 7, 11], np.int64), cfg.fanouts, 99, rows)
    ctx.close()


def test_c5_full_size_sampling_single_gpu():
    """MAG240M-shaped (244M vertices, 1.7B edges, 3 types): blocks bit-exact on one GPU.
    Its 187 GB of paper features need >= 2 GPUs: checked by tests/dist_gpu_parity.py."""
    import torch
    cfg = synth.config("C5")
    g = synth.build_host_graph(cfg, materialize_indices=True)
    ctx = _ctx(g, features=False)
    seeds = synth.batch_seeds(cfg, 0)
    rs = synth.rng_seed(cfg, 0)
    res = oracle.sample(g, seeds, cfg.fanouts, rs)
    b = ctx.sample_minibatch(torch.from_numpy(seeds).cuda(), cfg.fanouts, rs, features=False)
    assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
    b.free()
    ctx.close()


def test_device_indices_match_host_generator():
    import ctypes
    import torch
    cfg = synth.config("C4")
    lo, hi = 1_000_000_000, 1_000_100_000
    t = torch.empty(hi - lo, dtype=torch.int32, device="cuda:0")
    synth.dev_lib().sy_indices_dev(cfg.gen_seed, 0, int(cfg.vt_counts[0]), lo, hi, ctypes.c_void_p(t.data_ptr()),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), synth.gen_indices(cfg, 0, lo, hi))


def test_c2_bundles_of_4_on_2_lanes(c2):
    """Bundled launches (4 mini-batches per graph launch, grid.y = batch) on 2 lanes,
    including an empty batch and a smaller one: every batch bit-exact."""
    import torch
    cfg, g, rows, ctx = c2
    ctx.set_pipeline(2, 4)
    try:
        for rnd in range(3):
            idx = [60 + 4 * rnd + j for j in range(4)]
            seeds = [synth.batch_seeds(cfg, i) for i in idx]
            seeds[1] = seeds[1][:100] if rnd == 1 else seeds[1]
            seeds[2] = seeds[2][:0] if rnd == 2 else seeds[2]
            rs = [synth.rng_seed(cfg, i) for i in idx]
            dev = [torch.from_numpy(s).cuda() for s in seeds]   # read in place: keep alive until resolved
            bls = ctx.sample_bundle(dev, cfg.fanouts, rs, features=True, async_=(rnd != 0))
            for s, r, b in zip(seeds, rs, bls):
                res = oracle.sample(g, s, cfg.fanouts, r)
                assert_same_batch(res, b, cfg.n_vt, cfg.n_rel)
                assert_same_features(res, _features_of(b, cfg), cfg, rows)
                b.free()
        # a partial bundle (3 of 4) and a bad batch inside an async bundle
        dev = [torch.from_numpy(synth.batch_seeds(cfg, 90)).cuda(), torch.tensor([1, 99999999], device="cuda:0"),
               torch.from_numpy(synth.batch_seeds(cfg, 91)).cuda()]
        bls = ctx.sample_bundle(dev, cfg.fanouts, [5, 6, 7], async_=True)
        from paper_2112_15345_b200 import EgError
        with pytest.raises(EgError):
            bls[1].wait()
        res = oracle.sample(g, synth.batch_seeds(cfg, 91), cfg.fanouts, 7)
        assert_same_batch(res, bls[2], cfg.n_vt, cfg.n_rel)
        for b in bls:
            b.free()
    finally:
        ctx.set_pipeline(1, 1)


def test_c3_heavy_items_split_and_not():
    """Hubs (d > 2048) are split into chunk tasks over several warps when k <= 48 and take
    the one-warp paths otherwise; both bit-exact (k = 48 / 49 / 1 / 5 on C3's hubs)."""
    cfg = synth.config("C3")
    g = synth.build_host_graph(cfg)
    rows = {0: synth.host_features(cfg, 0)}
    ctx = _ctx(g)
    deg = np.diff(g.indptr[0])
    hubs = np.argsort(deg)[-40:].astype(np.int64)          # the 40 largest in-degrees
    for fo in ([[48]], [[49]], [[1], [2]], [[5], [48], [3]]):
        run_and_compare(ctx, g, cfg, hubs, fo, 4242, rows)
    ctx.close()
