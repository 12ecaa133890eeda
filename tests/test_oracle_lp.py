"""Pins of the oracle's link-prediction targets (og_lp_targets, NEXT-3; -m "not gpu").

What fixes them (readings L1-L4):
  negatives  -> an independent pure-Python Philox (tests/ref_model.py) evaluated on the
                L1 counter layout, and a chi-square over the dst type's range (S:409:
                "negative dst empirical distribution uniform over type range")
  seeds      -> brute-force set of the endpoints ("seed vertex set = union of all
                endpoints"), ascending gid (L2)
  pairs      -> round trip through the per-type seed arrays (L3); S:407's trivial case
  sampling   -> identical to og_sample on the seeds (L2) and the batch invariants
"""
import numpy as np
import pytest
from scipy import stats

import oracle
import ref_model
import synth
from graphs import from_edges
from invariants import check_batch

NEG_TAG = 0x4E454721   # 'NEG!'


def _positives(cfg, g, rel, n, seed):
    """n existing edges of relation rel as (src gid, dst gid)."""
    rng = np.random.default_rng(seed)
    ip = g.indptr[rel]
    e = rng.integers(0, int(ip[-1]), n)
    dst = np.searchsorted(ip, e, side="right") - 1 + int(cfg.offsets[cfg.rels[rel][2]])
    src = g.indices[rel][e].astype(np.int64) + int(cfg.offsets[cfg.rels[rel][1]])
    return src, dst.astype(np.int64)


@pytest.mark.parametrize("rel", [0, 1, 2])
def test_negatives_match_independent_philox(c1_graph, rel):
    cfg = synth.config("C1")
    src, dst = _positives(cfg, c1_graph, rel, 40, rel)
    n_neg, neg_seed = 3, 0x0123456789ABCDEF
    t = oracle.lp_targets(c1_graph, src, dst, rel, n_neg, neg_seed)
    dvt = cfg.rels[rel][2]
    off, n_t = int(cfg.offsets[dvt]), int(cfg.vt_counts[dvt])
    want = []
    for i in range(len(src)):
        for q in range(n_neg):
            w = ref_model.philox([i, q, 0, NEG_TAG], [neg_seed & 0xFFFFFFFF, neg_seed >> 32])[0]
            want.append(off + ((w * n_t) >> 32))
    assert t.neg_dst.tolist() == want
    assert np.all((t.neg_dst >= off) & (t.neg_dst < off + n_t))   # S:408 range


def test_negatives_uniform_chi_square():
    """uniform over the dst type's range.  10-vertex dst type, 20k draws."""
    g = from_edges([5, 10], [(0, 1, [(0, 0), (1, 1)])])   # r0: type 0 -> type 1
    n = 4000
    src = np.zeros(n, np.int64)                            # gid 0 (type 0)
    dst = np.full(n, 5, np.int64)                          # gid 5 (type 1, tid 0)
    t = oracle.lp_targets(g, src, dst, 0, 5, 77)
    counts = np.bincount(t.neg_dst - 5, minlength=10)
    assert counts.sum() == n * 5
    chi2 = ((counts - n * 5 / 10) ** 2 / (n * 5 / 10)).sum()
    assert stats.chi2.sf(chi2, 9) > 0.001


def test_seeds_union_and_pairs_round_trip(c1_graph):
    cfg = synth.config("C1")
    for rel in range(cfg.n_rel):
        src, dst = _positives(cfg, c1_graph, rel, 64, 10 + rel)
        t = oracle.lp_targets(c1_graph, src, dst, rel, 2, 5 + rel)
        assert t.seeds.tolist() == sorted(set(src.tolist()) | set(dst.tolist()) | set(t.neg_dst.tolist()))
        per = {u: [x for x in t.seeds.tolist() if cfg.offsets[u] <= x < cfg.offsets[u + 1]] for u in range(cfg.n_vt)}
        svt, dvt = cfg.rels[rel][1], cfg.rels[rel][2]
        assert [per[svt][i] for i in t.pos_src] == src.tolist()
        assert [per[dvt][i] for i in t.pos_dst] == dst.tolist()
        assert [per[dvt][i] for i in t.neg_dst_local] == t.neg_dst.tolist()
        assert t.neg_src.tolist() == np.repeat(t.pos_src, 2).tolist()


def test_spec_trivial_one_positive_one_negative():
    """1 positive, 1 negative -> 2 pairs, 2-3 unique seed vertices."""
    g = from_edges([4, 3], [(0, 1, [(0, 0), (1, 0), (2, 1)])])
    t = oracle.lp_targets(g, [1], [4], 0, 1, 3)
    assert len(t.pos_src) + len(t.neg_src) == 2
    assert 2 <= len(t.seeds) <= 3
    assert t.seeds.tolist() == sorted({1, 4, int(t.neg_dst[0])})


def test_no_negatives_and_empty():
    g = from_edges([4, 3], [(0, 1, [(0, 0), (1, 0), (2, 1)])])
    t = oracle.lp_targets(g, [2, 1], [5, 4], 0, 0, 3)
    assert t.seeds.tolist() == [1, 2, 4, 5] and len(t.neg_dst) == 0
    assert t.pos_src.tolist() == [1, 0] and t.pos_dst.tolist() == [1, 0]
    t = oracle.lp_targets(g, [], [], 0, 4, 3)
    assert len(t.seeds) == 0


def test_range_errors():
    g = from_edges([4, 3], [(0, 1, [(0, 0), (1, 0), (2, 1)])])
    with pytest.raises(oracle.OracleError) as e:
        oracle.lp_targets(g, [4], [4], 0, 1, 3)            # src of the wrong type
    assert e.value.code == oracle.OG_ERANGE
    with pytest.raises(oracle.OracleError) as e:
        oracle.lp_targets(g, [0], [7], 0, 1, 3)            # dst out of range
    assert e.value.code == oracle.OG_ERANGE
    with pytest.raises(oracle.OracleError) as e:
        oracle.lp_targets(g, [0], [4], 1, 1, 3)            # no such relation
    assert e.value.code == oracle.OG_EINVAL


def test_sample_lp_is_sample_on_the_seeds(c1_graph):
    cfg = synth.config("C1")
    src, dst = _positives(cfg, c1_graph, 1, 32, 3)
    res, t = oracle.sample_lp(c1_graph, src, dst, 1, 2, 11, cfg.fanouts, 42)
    ref = oracle.sample(c1_graph, t.seeds, cfg.fanouts, 42)
    for lvl in range(len(cfg.fanouts) + 1):
        for u in range(cfg.n_vt):
            assert np.array_equal(res.levels[lvl][u], ref.levels[lvl][u])
    check_batch(c1_graph, t.seeds, cfg.fanouts, res.levels, res.blocks)
