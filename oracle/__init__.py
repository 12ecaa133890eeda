"""CPU oracle for mini-batch ego-network generation (DistDGLv2, arxiv 2112.15345).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2112_15345_b200``) never imports it and
shares no code with it.

This is a thin ctypes marshaller over ``oracle.c`` (plain single-threaded C; see
its header for the passage each step follows).  Every function here only moves
numpy arrays in and out; all of the method's arithmetic is in ``oracle.c``.

Parity status of each oracle function (pins are in ``tests/test_oracle_*.py``):
  og_philox4x32_10  pinned: Random123 known-answer vectors
  og_key32          pinned: counter-layout golden values + chi-square / inclusion
  og_sample         pinned: paper invariants (existence, min(d,k), no duplicates,
                    full neighbourhood, dst prefix, sorted new, round trip),
                    BFS closed form at fanout -1, worked example, uniformity
  og_gather         pinned: numpy.take on the same rows
  sage_mean_layer   pinned: dense-matrix form (D^-1 A X W^T via numpy matmul), closed
                    forms (constant inputs, isolated dsts), neighbour-order invariance
  og_lp_targets     pinned: negatives vs an independent pure-Python Philox and a
                    chi-square over the dst range; seeds = brute-force set of the
                    endpoints; every pair round-trips through the seeds
  exact sampled sets vs the paper: parity unpinned (the paper fixes only the
                    distribution; bit-exactness is relative to key32)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

OG_OK, OG_EINVAL, OG_ERANGE = 0, -1, -2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11, no CUDA)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-o", tmp, _SRC]
        )
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER
        L.og_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.og_key32.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64]
        L.og_key32.restype = ctypes.c_uint32
        L.og_sample.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_void_p, ctypes.c_uint64, P(ctypes.c_void_p)]
        L.og_gather.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.og_free.argtypes = [ctypes.c_void_p]
        L.og_n_nodes.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
        L.og_n_nodes.restype = ctypes.c_int64
        L.og_nodes.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
        L.og_nodes.restype = P(ctypes.c_int64)
        L.og_lp_targets.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_void_p, P(ctypes.c_int64), ctypes.c_void_p]
        L.og_block.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64),
                               P(ctypes.c_int64), P(P(ctypes.c_int32)), P(P(ctypes.c_int32)),
                               P(P(ctypes.c_int64)), P(P(ctypes.c_int64))]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__({OG_EINVAL: "EINVAL", OG_ERANGE: "ERANGE"}.get(code, str(code)))
        self.code = code


def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().og_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def key32(seed: int, h: int, r: int, v: int, j: int) -> int:
    return int(lib().og_key32(seed & (2**64 - 1), h, r, v, j))


@dataclass
class RelBlock:
    indptr: np.ndarray   # int32 [n_dst+1]
    indices: np.ndarray  # int32 local src ids
    eids: np.ndarray     # int64
    src_gid: np.ndarray  # int64 sampled edge list (global src ids)


@dataclass
class OracleResult:
    n_hops: int
    n_vt: int
    n_rel: int
    levels: list = field(default_factory=list)  # levels[l][u] int64 arrays; l=0 seeds, l=h+1 S_h
    blocks: list = field(default_factory=list)  # blocks[h][r] RelBlock

    def dst_nodes(self, h, u):
        return self.levels[h][u]

    def src_nodes(self, h, u):
        return self.levels[h + 1][u]

    def input_nodes(self, u):
        return self.levels[self.n_hops][u]


class _Graph:
    """Keeps the ctypes view of a host graph (and the arrays it points to) alive."""

    def __init__(self, graph):
        self.vt_counts = np.ascontiguousarray(graph.vt_counts, dtype=np.int64)
        self.src = np.ascontiguousarray(graph.rel_src, dtype=np.int32)
        self.dst = np.ascontiguousarray(graph.rel_dst, dtype=np.int32)
        self.indptr = [np.ascontiguousarray(a, dtype=np.int64) for a in graph.indptr]
        self.indices = [np.ascontiguousarray(a, dtype=np.int32) for a in graph.indices]
        R = len(self.indptr)
        self.ip_ptrs = (ctypes.c_void_p * R)(*[a.ctypes.data for a in self.indptr])
        self.ix_ptrs = (ctypes.c_void_p * R)(*[a.ctypes.data for a in self.indices])

        class OgGraph(ctypes.Structure):
            _fields_ = [("n_vt", ctypes.c_int32), ("vt_count", ctypes.c_void_p),
                        ("n_rel", ctypes.c_int32), ("rel_src_vt", ctypes.c_void_p),
                        ("rel_dst_vt", ctypes.c_void_p), ("indptr", ctypes.c_void_p),
                        ("indices", ctypes.c_void_p)]

        self.c = OgGraph(len(self.vt_counts), self.vt_counts.ctypes.data, R,
                         self.src.ctypes.data, self.dst.ctypes.data,
                         ctypes.cast(self.ip_ptrs, ctypes.c_void_p),
                         ctypes.cast(self.ix_ptrs, ctypes.c_void_p))


def sample(graph, seeds, fanouts, rng_seed: int) -> OracleResult:
    """Run og_sample.  ``graph`` has vt_counts, rel_src, rel_dst, indptr[r], indices[r]
    (global in-CSC per relation).  ``fanouts`` is [hop][relation]."""
    L = lib()
    g = _Graph(graph)
    seeds = np.ascontiguousarray(seeds, dtype=np.int64)
    fo = np.ascontiguousarray(fanouts, dtype=np.int32)
    n_hops = fo.shape[0]
    R = len(g.indptr)
    assert fo.shape == (n_hops, R)
    res = ctypes.c_void_p()
    rc = L.og_sample(ctypes.addressof(g.c), seeds.ctypes.data, len(seeds), n_hops,
                     fo.ctypes.data, rng_seed & (2**64 - 1), ctypes.byref(res))
    if rc != OG_OK:
        raise OracleError(rc)
    try:
        V = len(g.vt_counts)
        out = OracleResult(n_hops, V, R)
        for lvl in range(n_hops + 1):
            row = []
            for u in range(V):
                n = L.og_n_nodes(res, lvl, u)
                p = L.og_nodes(res, lvl, u)
                row.append(np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.int64))
            out.levels.append(row)
        for h in range(n_hops):
            row = []
            for r in range(R):
                nd, nz = ctypes.c_int64(), ctypes.c_int64()
                ip, ix = ctypes.POINTER(ctypes.c_int32)(), ctypes.POINTER(ctypes.c_int32)()
                ei, sg = ctypes.POINTER(ctypes.c_int64)(), ctypes.POINTER(ctypes.c_int64)()
                L.og_block(res, h, r, ctypes.byref(nd), ctypes.byref(nz), ctypes.byref(ip),
                           ctypes.byref(ix), ctypes.byref(ei), ctypes.byref(sg))
                nd, nz = nd.value, nz.value
                row.append(RelBlock(
                    np.ctypeslib.as_array(ip, shape=(nd + 1,)).copy(),
                    np.ctypeslib.as_array(ix, shape=(nz,)).copy() if nz else np.zeros(0, np.int32),
                    np.ctypeslib.as_array(ei, shape=(nz,)).copy() if nz else np.zeros(0, np.int64),
                    np.ctypeslib.as_array(sg, shape=(nz,)).copy() if nz else np.zeros(0, np.int64)))
            out.blocks.append(row)
        return out
    finally:
        L.og_free(res)


@dataclass
class LpTargets:
    """Link-prediction targets of one mini-batch (og_lp_targets)."""
    seeds: np.ndarray     # int64 distinct endpoints, ascending gid
    neg_dst: np.ndarray   # int64 [n_pos * n_neg] corrupted dst gids
    pos_src: np.ndarray   # int32 local ids (index among the seeds of the endpoint's type)
    pos_dst: np.ndarray
    neg_src: np.ndarray
    neg_dst_local: np.ndarray


def lp_targets(graph, src, dst, rel: int, n_neg: int, neg_seed: int) -> LpTargets:
    g = _Graph(graph)
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    n = len(src)
    assert len(dst) == n
    neg = np.zeros(max(1, n * n_neg), np.int64)
    seeds = np.zeros(max(1, n * (2 + n_neg)), np.int64)
    pairs = np.zeros(max(1, 2 * n + 2 * n * n_neg), np.int32)
    ns = ctypes.c_int64()
    rc = lib().og_lp_targets(ctypes.addressof(g.c), src.ctypes.data, dst.ctypes.data, n, rel, n_neg,
                             neg_seed & (2**64 - 1), neg.ctypes.data, seeds.ctypes.data, ctypes.byref(ns),
                             pairs.ctypes.data)
    if rc != OG_OK:
        raise OracleError(rc)
    m = n * n_neg
    return LpTargets(seeds[:ns.value].copy(), neg[:m].copy(), pairs[:n].copy(), pairs[n:2 * n].copy(),
                     pairs[2 * n:2 * n + m].copy(), pairs[2 * n + m:2 * n + 2 * m].copy())


def sample_lp(graph, src, dst, rel: int, n_neg: int, neg_seed: int, fanouts, rng_seed: int):
    """A link-prediction mini-batch: its targets, then og_sample from their seeds."""
    t = lp_targets(graph, src, dst, rel, n_neg, neg_seed)
    return sample(graph, t.seeds, fanouts, rng_seed), t


def gather(result: OracleResult, vt_counts, u: int, rows: np.ndarray) -> np.ndarray:
    """Feature rows of the input vertices of type u (result.input_nodes(u)),
    verbatim bytes, via og_gather.  ``rows`` is the full [N_u, ...] host array."""
    return gather_ids(result.input_nodes(u), vt_counts, u, rows)


def gather_ids(ids, vt_counts, u: int, rows: np.ndarray) -> np.ndarray:
    rows = np.ascontiguousarray(rows)
    row_bytes = rows.strides[0] if rows.ndim > 1 else rows.itemsize
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    vtc = np.asarray(vt_counts, dtype=np.int64)
    off_u = int(vtc[:u].sum())
    out = np.empty((len(ids),) + rows.shape[1:], dtype=rows.dtype)
    rc = lib().og_gather(ids.ctypes.data, len(ids), off_u, int(vtc[u]), rows.ctypes.data,
                         row_bytes, out.ctypes.data)
    if rc != OG_OK:
        raise OracleError(rc)
    return out


# ----------------------------------------------------------------------------- consumer step (NEXT-4 i)

def sage_mean_layer(indptr, indices, x_src, x_dst, w):
    """GraphSAGE-mean layer over one block relation, pre-activation, in fp64 -- the
    paper's message passing h_v' = g(h_v, (+)_{u in N(v)} f(h_u, ...)) (Eq. 1)
    with f = identity, (+) = mean over the block's sampled in-edges of v (an edge sampled
    twice counts twice; no in-edge -> 0), g(a, b) = W_self a + W_neigh b (GraphSAGE,
    P:964; DESIGN.md §3 reading C1).  x_src [n_src, F] (rows = the block's src nodes),
    x_dst [n_dst, F] or None (no self term), w [H, 2F] = [W_self | W_neigh] (or [H, F]
    = W_neigh without a self term).  Returns z [n_dst, H] float64.  Plain loop over the
    dst vertices in the definition's order."""
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    xs = np.asarray(x_src, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    n_dst, F = len(indptr) - 1, xs.shape[1]
    self_term = x_dst is not None
    w_self, w_neigh = (w[:, :F], w[:, F:]) if self_term else (None, w)
    z = np.zeros((n_dst, w.shape[0]), dtype=np.float64)
    xd = np.asarray(x_dst, dtype=np.float64) if self_term else None
    for v in range(n_dst):
        nb = indices[indptr[v]:indptr[v + 1]]
        m = xs[nb].mean(axis=0) if len(nb) else np.zeros(F)
        z[v] = w_neigh @ m
        if self_term:
            z[v] += w_self @ xd[v]
    return z

