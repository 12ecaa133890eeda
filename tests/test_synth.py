"""The seeded input generator: exact edge counts, ranges, sharding (host only)."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_graph_shape(name):
    cfg = synth.config(name)
    g = synth.build_host_graph(cfg)
    for r, (_, s, t, ne) in enumerate(cfg.rels):
        ip = g.indptr[r]
        assert len(ip) == cfg.vt_counts[t] + 1 and ip[0] == 0 and ip[-1] == ne   # exact |E_r|
        deg = np.diff(ip)
        assert deg.min() >= 0 and deg.max() <= cfg.dmax(r)
        ix = g.indices[r]
        assert ix.min() >= 0 and ix.max() < cfg.vt_counts[s]
        assert abs(deg.mean() - ne / cfg.vt_counts[t]) < 1e-9


def test_degree_law_heavy_tail():
    cfg = synth.config("C2")
    ip = synth.gen_indptr(cfg, 0)
    deg = np.diff(ip)
    # heavy tail: the max is orders of magnitude above the mean, most vertices below it
    assert deg.max() > 100 * deg.mean()
    assert np.median(deg) < deg.mean()


def test_deterministic_and_slices():
    cfg = synth.config("C1")
    a = synth.build_host_graph(cfg)
    b = synth.build_host_graph(cfg)
    for r in range(cfg.n_rel):
        assert np.array_equal(a.indptr[r], b.indptr[r]) and np.array_equal(a.indices[r], b.indices[r])
        assert np.array_equal(synth.gen_indices(cfg, r, 100, 200), a.indices[r][100:200])
    f = synth.host_features(cfg, 1)
    assert np.array_equal(synth.host_features(cfg, 1, 10, 20), f[10:20])
    assert f.dtype == np.float32 and np.all((f >= 1) & (f < 2))


def test_fp16_features_in_range():
    cfg = synth.config("C4")
    f = synth.host_features(cfg, 0, 0, 1000)
    assert f.dtype == np.float16 and np.all((f >= 1) & (f < 2))
    assert len(np.unique(f)) > 500


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shards_cover_graph(c1_graph, world):
    cfg = synth.config("C1")
    parts = [synth.shard(c1_graph, world, p) for p in range(world)]
    for r in range(cfg.n_rel):
        t = cfg.rels[r][2]
        ips, ixs = [], []
        for p, (bounds, rels) in enumerate(parts):
            rs = rels[r]
            assert rs.indptr[0] == 0 and len(rs.indptr) == bounds[t][p + 1] - bounds[t][p] + 1
            assert rs.e_hi - rs.e_lo == rs.indptr[-1]
            ips.append(rs.indptr[:-1] + rs.e_lo)
            ixs.append(rs.indices)
        assert np.array_equal(np.concatenate(ips + [[c1_graph.indptr[r][-1]]]), c1_graph.indptr[r])
        assert np.array_equal(np.concatenate(ixs), c1_graph.indices[r])


def test_range_bounds_policy():
    assert list(synth.range_bounds(10, 4)) == [0, 2, 5, 7, 10]
    assert list(synth.range_bounds(3, 8)) == [0, 0, 0, 1, 1, 1, 2, 2, 3]


def test_seeds():
    cfg = synth.config("C2")
    s0, s1 = synth.batch_seeds(cfg, 0), synth.batch_seeds(cfg, 1)
    assert len(s0) == cfg.batch and len(np.unique(s0)) == cfg.batch
    assert not np.intersect1d(s0, s1).size        # one epoch = disjoint batches
    assert np.all((s0 >= cfg.offsets[0]) & (s0 < cfg.offsets[1]))
    assert synth.rng_seed(cfg, 0) != synth.rng_seed(cfg, 1)


# ----------------------------------------------------------------------------- planted communities (NEXT-2)

def test_planted_generator_locality_and_identity():
    """C1L: the fraction of edges whose src lies in the dst's community is q + (1-q)/8
    (a uniform draw lands in the right block 1/8 of the time); q = 0 reproduces the
    uniform generator byte for byte; LP positives of a planted graph are real edges."""
    import dataclasses
    cfg = synth.config("C1L")
    g = synth.build_host_graph(cfg)
    for r, (_, s, t, _) in enumerate(cfg.rels):
        ip, ix = g.indptr[r], g.indices[r]
        n_s, n_t = int(cfg.vt_counts[s]), int(cfg.vt_counts[t])
        dst = np.repeat(np.arange(n_t), np.diff(ip))
        same = (dst * cfg.n_comm // n_t) == np.searchsorted(
            [(c * n_s) // cfg.n_comm for c in range(1, cfg.n_comm + 1)], ix, side="right")
        want = cfg.locality + (1 - cfg.locality) / cfg.n_comm
        assert abs(same.mean() - want) < 0.01, (r, same.mean(), want)
    base = synth.config("C1")
    zero = dataclasses.replace(base, locality=1e-15)          # q_thr == 0: only the uniform branch
    assert zero.q_thr == 0
    gz = synth.build_host_graph(zero)
    gb = synth.build_host_graph(base)
    for r in range(base.n_rel):
        assert np.array_equal(gz.indices[r], gb.indices[r])
    rel = synth.lp_rel(cfg)
    src, dst = synth.lp_positives(cfg, g, rel, 0, 200)
    off_s, off_t = int(cfg.offsets[cfg.rels[rel][1]]), int(cfg.offsets[cfg.rels[rel][2]])
    ip = g.indptr[rel]
    for a, b in zip(src, dst):
        x = b - off_t
        assert (g.indices[rel][ip[x]:ip[x + 1]] + off_s == a).any()


def test_confined_seeds_stay_in_the_rank_range():
    cfg = synth.config("C2L")
    n = int(cfg.vt_counts[cfg.seed_vt])
    for world in (2, 4):
        for p in range(world):
            lo, hi = (p * n) // world, ((p + 1) * n) // world
            s = synth.batch_seeds_confined(cfg, 3, p, world) - int(cfg.offsets[cfg.seed_vt])
            assert len(s) == cfg.batch and len(set(s.tolist())) == len(s)
            assert s.min() >= lo and s.max() < hi


def test_replica_policies_select_whole_tables():
    """Replicated partition policy: "auto" takes the small types only, "fit" whole
    tables smallest first within FIT_BUDGET (C2-C4 fit a quarter of a B200's HBM, C5 does not);
    nothing is replicated on one GPU."""
    from synth.device import FIT_BUDGET, replica_types
    assert replica_types(synth.config("C2"), 2) == [2, 3]
    assert replica_types(synth.config("C2"), 2, "fit") == [0, 1, 2, 3]
    assert replica_types(synth.config("C3"), 4, "fit") == [0]
    assert replica_types(synth.config("C4"), 8, "fit") == [0]
    assert replica_types(synth.config("C5"), 2, "fit") == []
    assert replica_types(synth.config("C4"), 1, "fit") == []
    c4 = synth.config("C4")
    assert int(c4.vt_counts[0]) * c4.feats[0][0] * 2 <= FIT_BUDGET
