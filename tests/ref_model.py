"""Independent pure-Python model of the method, for TINY inputs only.

A second, separately written reading of the same definition,
used to cross-check the C oracle on small cases.  It shares nothing with
oracle/ or the CUDA path.  Python loops: only for tiny graphs.
"""
M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox(ctr, key, rounds=10):
    c0, c1, c2, c3 = [x & MASK for x in ctr]
    k0, k1 = [x & MASK for x in key]
    for i in range(rounds):
        if i:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
        p0, p1 = M0 * c0, M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c3 ^ k1) & MASK, p0 & MASK
    return [c0, c1, c2, c3]


def key32(seed, h, r, v, j):
    w = philox([j >> 2, v & MASK, v >> 32, (h << 16) | r], [seed & MASK, (seed >> 32) & MASK])
    return w[j & 3]


def sample(vt_counts, rels, seeds, fanouts, rng_seed):
    """rels: list of (src_vt, dst_vt, indptr, indices) global in-CSC.
    Returns (levels, blocks) like oracle.OracleResult."""
    off = [0]
    for n in vt_counts:
        off.append(off[-1] + int(n))

    def vt_of(g):
        for t in range(len(vt_counts)):
            if off[t] <= g < off[t + 1]:
                return t
        raise ValueError(g)

    V = len(vt_counts)
    F = [[int(s) for s in seeds if vt_of(int(s)) == t] for t in range(V)]
    levels = [[list(x) for x in F]]
    blocks = []
    for h, fo in enumerate(fanouts):
        hop = []
        srcs_by_type = [set() for _ in range(V)]
        raw = []
        for r, (s, t, indptr, indices) in enumerate(rels):
            k = int(fo[r])
            ptr, eids, src = [0], [], []
            for v in F[t]:
                x = v - off[t]
                lo, hi = int(indptr[x]), int(indptr[x + 1])
                d = hi - lo
                if k == -1 or d <= k:
                    js = list(range(d))
                else:
                    js = sorted(sorted(range(d), key=lambda j: (key32(rng_seed, h, r, v, j), j))[:k])
                for j in js:
                    eids.append(lo + j)
                    src.append(off[s] + int(indices[lo + j]))
                ptr.append(len(eids))
            raw.append((ptr, eids, src))
            srcs_by_type[s].update(src)
        S = [F[u] + sorted(srcs_by_type[u] - set(F[u])) for u in range(V)]
        index = [{g: i for i, g in enumerate(S[u])} for u in range(V)]
        for r, (s, t, _, _) in enumerate(rels):
            ptr, eids, src = raw[r]
            hop.append({"indptr": ptr, "indices": [index[s][g] for g in src], "eids": eids, "src_gid": src})
        blocks.append(hop)
        levels.append([list(x) for x in S])
        F = S
    return levels, blocks
