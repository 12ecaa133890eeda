"""Checks of the paper's definitions on one sampled mini-batch.

These are the pins of the oracle (and, on the GPU, extra checks of the CUDA
output): they follow from the paper's text, not from either implementation.

  every sampled edge exists in its relation      P:284-285 ("neighbor vertices")
  count = min(d, k) per (dst, relation)           P:284-285 ("at most K")
  full neighbourhood when d <= k
  no duplicate edge per (dst, relation)           without replacement (DESIGN §3 #3)
  dst prefix: src_nodes starts with dst_nodes     DGL to_block convention (DESIGN §3 #6)
  new sources unique, sorted by gid, not in dst   P:698-700 ("unique set"), DESIGN §3 #7
  block ids round-trip to global ids              P:704-707 ("relabel vertices")
  every new source is used by some edge           P:706-707 ("remove empty vertices")
"""
import numpy as np


def check_batch(graph, seeds, fanouts, levels, blocks):
    """levels[l][u] node arrays (l=0 seeds), blocks[h][r] with indptr/indices/eids.
    graph: global CSC (vt_counts, rel_src, rel_dst, indptr, indices)."""
    vtc = np.asarray(graph.vt_counts, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(vtc)])
    V, R = len(vtc), len(graph.indptr)
    seeds = np.asarray(seeds, dtype=np.int64)
    for u in range(V):   # level 0 = seeds of type u in caller order
        m = (seeds >= off[u]) & (seeds < off[u + 1])
        assert np.array_equal(np.asarray(levels[0][u]), seeds[m])
    for h, fo in enumerate(fanouts):
        for u in range(V):
            F, S = np.asarray(levels[h][u], np.int64), np.asarray(levels[h + 1][u], np.int64)
            assert np.array_equal(S[:len(F)], F), "dst prefix"
            new = S[len(F):]
            assert np.all(np.diff(new) > 0), "new sources sorted + unique"
            assert not np.isin(new, F).any(), "new sources not in dst"
            assert np.all((S >= off[u]) & (S < off[u + 1])), "type range"
            used = np.zeros(len(S), bool)
            for r in range(R):
                if int(graph.rel_src[r]) == u:
                    used[np.asarray(blocks[h][r]["indices"] if isinstance(blocks[h][r], dict)
                                    else blocks[h][r].indices, np.int64)] = True
            assert used[len(F):].all(), "every new source has an edge"
        for r in range(R):
            s, t = int(graph.rel_src[r]), int(graph.rel_dst[r])
            b = blocks[h][r]
            get = (lambda k: np.asarray(b[k])) if isinstance(b, dict) else (lambda k: np.asarray(getattr(b, k)))
            ip, ix, ei = get("indptr").astype(np.int64), get("indices").astype(np.int64), get("eids").astype(np.int64)
            F = np.asarray(levels[h][t], np.int64)
            S = np.asarray(levels[h + 1][s], np.int64)
            assert len(ip) == len(F) + 1 and ip[0] == 0 and np.all(np.diff(ip) >= 0)
            assert ip[-1] == len(ix) == len(ei)
            gip, gix = graph.indptr[r], graph.indices[r]
            k = int(fo[r])
            x = F - off[t]
            lo, hi = gip[x], gip[x + 1]
            d = hi - lo
            want = d if k == -1 else np.minimum(d, k)
            assert np.array_equal(np.diff(ip), want), "count = min(d, k)"
            dst_of_edge = np.repeat(np.arange(len(F)), np.diff(ip))
            assert np.all(ei >= lo[dst_of_edge]) and np.all(ei < hi[dst_of_edge]), "edge exists"
            if len(ix):
                assert np.all(ix < len(S)), "local id range"
                assert np.array_equal(S[ix], off[s] + gix[ei].astype(np.int64)), "round trip"
            for i in range(len(F)):   # ascending offsets => no duplicates; full when d <= k
                e = ei[ip[i]:ip[i + 1]]
                assert np.all(np.diff(e) > 0)
                if k == -1 or d[i] <= k:
                    assert np.array_equal(e, np.arange(lo[i], hi[i]))
