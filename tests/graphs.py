"""Tiny hand-built graphs for tests (test code, not the method)."""
from dataclasses import dataclass

import numpy as np


@dataclass
class TinyGraph:
    vt_counts: np.ndarray
    rel_src: np.ndarray
    rel_dst: np.ndarray
    indptr: list
    indices: list


def from_edges(vt_counts, rels):
    """rels: list of (src_vt, dst_vt, [(src_tid, dst_tid), ...]); CSC neighbour
    order = input order (stable by dst)."""
    vt_counts = np.asarray(vt_counts, dtype=np.int64)
    indptr, indices = [], []
    for s, t, edges in rels:
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        order = np.argsort(e[:, 1], kind="stable")
        e = e[order]
        deg = np.bincount(e[:, 1], minlength=int(vt_counts[t])) if len(e) else np.zeros(int(vt_counts[t]), np.int64)
        ip = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        indptr.append(ip)
        indices.append(e[:, 0].astype(np.int32))
    return TinyGraph(vt_counts, np.array([r[0] for r in rels], np.int32),
                     np.array([r[1] for r in rels], np.int32), indptr, indices)


def star(n_dst, degree, n_src=None):
    """one vertex type? no: two types; every dst (type 1) has `degree` in-edges
    from distinct srcs (type 0) at offsets j -> src (i*degree + j) % n_src."""
    n_src = n_src or n_dst * degree
    edges = [((i * degree + j) % n_src, i) for i in range(n_dst) for j in range(degree)]
    return from_edges([n_src, n_dst], [(0, 1, edges)])
