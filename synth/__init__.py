"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONE place both sides take inputs from: the oracle (tests,
cpu baseline) and the CUDA path (tests, bench) both read the graphs, feature
bytes, seeds and rng seeds built here.  It holds none of the sampling method's
arithmetic (no Philox, no selection, no compaction, no gather); its hash is
splitmix64 (synth_hash.h).

Config shapes: BASELINE.json ``configs``; vertex/edge counts per type are the
OGB statistics, consistent with the paper's Table 1
(tbl:dataset).  Fanouts are [hop][relation], hop 0 at the seeds
(reading 1).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_DEV_SO = os.path.join(_HERE, "libsynth_dev.so")
_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(so, srcs):
    return not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(s) for s in srcs)


def build(force: bool = False) -> None:
    srcs = [os.path.join(_HERE, f) for f in ("synth.c", "synth_hash.h")]
    if force or _stale(_SO, srcs):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", tmp,
                               srcs[0], "-lm"])
        os.replace(tmp, _SO)
    dsrcs = [os.path.join(_HERE, f) for f in ("synth_dev.cu", "synth_hash.h")]
    if force or _stale(_DEV_SO, dsrcs):
        tmp = _DEV_SO + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", *_ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               "-o", tmp, dsrcs[0]])
        os.replace(tmp, _DEV_SO)


_lib = None
_dev = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        c = ctypes
        L.sy_indptr.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_int64, c.c_double, c.c_void_p]
        L.sy_indptr.restype = c.c_int
        L.sy_indices.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_int64, c.c_void_p]
        L.sy_indices_at.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_void_p, c.c_int64, c.c_void_p]
        L.sy_indices_loc.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_void_p, c.c_int64, c.c_int64,
                                     c.c_uint32, c.c_int32, c.c_void_p]
        L.sy_indices_at_loc.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_void_p, c.c_void_p,
                                        c.c_int64, c.c_uint32, c.c_int32, c.c_void_p]
        L.sy_features.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_int64, c.c_int32, c.c_void_p]
        L.sy_features_ids.argtypes = [c.c_uint64, c.c_int32, c.c_void_p, c.c_int64, c.c_int64, c.c_int32, c.c_void_p]
        L.sy_select_train.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_uint64, c.c_void_p, c.c_int64]
        L.sy_select_train.restype = c.c_int64
        L.sy_perm_keys.argtypes = [c.c_uint64, c.c_int64, c.c_void_p, c.c_int64, c.c_void_p]
        L.sy_mix.argtypes = [c.c_uint64]
        L.sy_mix.restype = c.c_uint64
        L.sy_degree_table.argtypes = [c.c_double, c.c_int64, c.c_double, c.c_void_p, c.POINTER(c.c_double)]
        L.sy_degree_table.restype = c.c_int
        _lib = L
    return _lib


def dev_lib():
    global _dev
    if _dev is None:
        build()
        L = ctypes.CDLL(_DEV_SO)
        c = ctypes
        L.sy_indices_dev.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_int64, c.c_void_p, c.c_void_p]
        L.sy_features_dev.argtypes = [c.c_uint64, c.c_int32, c.c_int64, c.c_int64, c.c_int64, c.c_int32,
                                      c.c_void_p, c.c_void_p]
        _dev = L
    return _dev


# ----------------------------------------------------------------------------- configs

F32, F16 = 0, 1
DTYPE_BYTES = {F32: 4, F16: 2}
NP_DTYPE = {F32: np.float32, F16: np.float16}


@dataclass
class Config:
    name: str
    vtypes: list            # [(name, count)]
    rels: list              # [(name, src_vt, dst_vt, n_edges)]
    feats: dict             # vt -> (dim, dtype)
    seed_vt: int
    batch: int
    fanouts: list           # [hop][rel]
    train_count: int
    gen_seed: int = 0x5EED_2112_15345
    alpha: float = 2.5
    base_rng: int = 0xD15_7D61_0002
    min_gpus: int = 1
    description: str = ""
    locality: float = 0.0   # planted communities (NEXT-2): P(src from the dst's community)
    n_comm: int = 8         # contiguous communities per vertex type

    @property
    def q_thr(self) -> int:
        return int(min(2**32 - 1, round(self.locality * 2**32)))

    @property
    def n_vt(self):
        return len(self.vtypes)

    @property
    def n_rel(self):
        return len(self.rels)

    @property
    def vt_counts(self):
        return np.array([c for _, c in self.vtypes], dtype=np.int64)

    @property
    def offsets(self):
        return np.concatenate([[0], np.cumsum(self.vt_counts)]).astype(np.int64)

    @property
    def n_hops(self):
        return len(self.fanouts)

    def dmax(self, r):
        return int(min(1 << 20, -(-self.rels[r][3] // 100)))

    def row_bytes(self, u):
        if u not in self.feats:
            return 0
        dim, dt = self.feats[u]
        return dim * DTYPE_BYTES[dt]


def _c1():
    return Config("C1", [("A", 6000), ("B", 4000)],
                  [("r0", 0, 0, 40000), ("r1", 0, 1, 30000), ("r2", 1, 0, 30000)],
                  {0: (16, F32), 1: (16, F32)}, seed_vt=0, batch=64,
                  fanouts=[[5, 5, 5], [5, 5, 5]], train_count=6000,
                  description="tiny synthetic hetero graph: 2 vertex types, 3 edge types, 10k vertices, "
                              "100k edges, fanout [5,5], batch 64, feat dim 16")


def _c2():
    return Config("C2", [("paper", 736389), ("author", 1134649), ("institution", 8740), ("field", 59965)],
                  [("cites", 0, 0, 5416271), ("writes", 1, 0, 7145660),
                   ("rev_has_topic", 3, 0, 7505078), ("rev_affiliated_with", 2, 1, 1043998)],
                  {u: (128, F32) for u in range(4)}, seed_vt=0, batch=1024,
                  fanouts=[[25] * 4, [20] * 4], train_count=629571,
                  description="ogbn-mag-shaped synthetic: 4 vertex types, 4 relations, 1.9M vertices, "
                              "21M edges, fanout [25,20], batch 1024, 128-d fp32")


def _c3():
    return Config("C3", [("product", 2449029)], [("also_bought", 0, 0, 61859140)],
                  {0: (100, F32)}, seed_vt=0, batch=1000, fanouts=[[15], [10], [5]],
                  train_count=196615,
                  description="ogbn-products-shaped synthetic homogeneous: 2.4M vertices, 62M edges, "
                              "fanout [15,10,5], batch 1000, 100-d fp32")


def _c4():
    return Config("C4", [("paper", 111059956)], [("cites", 0, 0, 1615685872)],
                  {0: (128, F16)}, seed_vt=0, batch=1024, fanouts=[[15], [10], [5]],
                  train_count=1207179,
                  description="ogbn-papers100M-shaped synthetic: 111M vertices, 1.6B edges, "
                              "fanout [15,10,5], batch 1024, 128-d fp16")


def _c5():
    return Config("C5", [("paper", 121751666), ("author", 122383112), ("institution", 25721)],
                  [("cites", 0, 0, 1297748926), ("writes", 1, 0, 386022720),
                   ("rev_affiliated_with", 2, 1, 44592586)],
                  {0: (768, F16)}, seed_vt=0, batch=1024, fanouts=[[25] * 3, [15] * 3],
                  train_count=1112392, min_gpus=2,
                  description="MAG240M-shaped synthetic hetero: 244M vertices, 3 types, 1.7B edges, "
                              "fanout [25,15], batch 1024, 768-d fp16 on paper vertices")


def _planted(base, q=0.9):
    """NEXT-2: the same shape with planted communities (8 contiguous blocks per type,
    sources from the dst's block with probability q), for the locality-aware partition
    (P:421-437): per-GPU ranges aligned with the blocks at P = 1, 2, 4, 8."""
    def make():
        c = base()
        c.name = c.name + "L"
        c.locality = q
        c.description = c.description + f"; planted communities (8 per type, p_local={q})"
        return c
    return make


CONFIGS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5,
           "C1L": _planted(_c1), "C2L": _planted(_c2), "C4L": _planted(_c4)}


def config(name: str) -> Config:
    return CONFIGS[name]()


# ----------------------------------------------------------------------------- host graph

@dataclass
class HostGraph:
    """Global (unsharded) in-CSC per relation.  indices may be None when not
    materialised (huge configs); then use ``indices_slice``."""
    cfg: Config
    vt_counts: np.ndarray
    rel_src: np.ndarray
    rel_dst: np.ndarray
    indptr: list
    indices: list = field(default_factory=list)

    def indices_slice(self, r, e_lo, e_hi):
        if self.indices and self.indices[r] is not None:
            return self.indices[r][e_lo:e_hi]
        return gen_indices(self.cfg, r, e_lo, e_hi, self.indptr[r])


def gen_indptr(cfg: Config, r: int) -> np.ndarray:
    _, s, t, ne = cfg.rels[r]
    n_dst = int(cfg.vt_counts[t])
    ip = np.empty(n_dst + 1, dtype=np.int64)
    rc = lib().sy_indptr(cfg.gen_seed, r, n_dst, ne, cfg.dmax(r), cfg.alpha, ip.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"sy_indptr failed ({rc}) for {cfg.name} r{r}")
    return ip


def gen_indices(cfg: Config, r: int, e_lo: int, e_hi: int, indptr=None) -> np.ndarray:
    _, s, t, ne = cfg.rels[r]
    out = np.empty(max(0, e_hi - e_lo), dtype=np.int32)
    if cfg.locality > 0:   # planted communities: the source depends on the dst's community
        ip = np.ascontiguousarray(gen_indptr(cfg, r) if indptr is None else indptr, np.int64)
        lib().sy_indices_loc(cfg.gen_seed, r, int(cfg.vt_counts[s]), int(cfg.vt_counts[t]), ip.ctypes.data,
                             e_lo, e_hi, cfg.q_thr, cfg.n_comm, out.ctypes.data)
    else:
        lib().sy_indices(cfg.gen_seed, r, int(cfg.vt_counts[s]), e_lo, e_hi, out.ctypes.data)
    return out


def build_host_graph(cfg: Config, materialize_indices: bool = True) -> HostGraph:
    indptr = [gen_indptr(cfg, r) for r in range(cfg.n_rel)]
    materialize_indices = materialize_indices or cfg.locality > 0   # (no device generator for these)
    indices = [gen_indices(cfg, r, 0, int(indptr[r][-1]), indptr[r]) if materialize_indices else None
               for r in range(cfg.n_rel)]
    return HostGraph(cfg, cfg.vt_counts, np.array([s for _, s, _, _ in cfg.rels], np.int32),
                     np.array([t for _, _, t, _ in cfg.rels], np.int32), indptr, indices)


def host_features(cfg: Config, u: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
    dim, dt = cfg.feats[u]
    hi = int(cfg.vt_counts[u]) if hi is None else hi
    out = np.empty((hi - lo, dim), dtype=NP_DTYPE[dt])
    lib().sy_features(cfg.gen_seed, u, lo, hi, dim, dt, out.ctypes.data)
    return out


def host_features_ids(cfg: Config, u: int, tids) -> np.ndarray:
    """Feature rows of the given type-local ids (no full materialisation)."""
    dim, dt = cfg.feats[u]
    tids = np.ascontiguousarray(tids, dtype=np.int64)
    out = np.empty((len(tids), dim), dtype=NP_DTYPE[dt])
    lib().sy_features_ids(cfg.gen_seed, u, tids.ctypes.data, len(tids), dim, dt, out.ctypes.data)
    return out


class LazyRows:
    """Stands in for a [N_u, dim] host feature array: rows[tids] computed on demand."""

    def __init__(self, cfg: Config, u: int):
        self.cfg, self.u = cfg, u

    def take(self, tids):
        return host_features_ids(self.cfg, self.u, tids)


# ----------------------------------------------------------------------------- partition

def range_bounds(n: int, world: int) -> np.ndarray:
    """bounds[p] = floor(p * n / world): the fixed per-type vertex-range policy."""
    return np.array([(p * n) // world for p in range(world + 1)], dtype=np.int64)


@dataclass
class RelShard:
    src_vt: int
    dst_vt: int
    indptr: np.ndarray     # local, starts at 0, n_local_dst + 1
    e_lo: int              # global CSC position of local edge 0 (edge_base)
    e_hi: int
    indices: np.ndarray | None = None   # host copy (None => generate on device)


def shard(graph: HostGraph, world: int, rank: int, with_indices: bool = True):
    """Rank `rank`'s shard: relation CSC rows of the dst vertices it owns (edge
    ownership = dst owner) and the bounds of every type."""
    cfg = graph.cfg
    bounds = np.stack([range_bounds(int(n), world) for n in cfg.vt_counts])
    rels = []
    for r in range(cfg.n_rel):
        _, s, t, _ = cfg.rels[r]
        lo, hi = int(bounds[t][rank]), int(bounds[t][rank + 1])
        ip = graph.indptr[r]
        e_lo, e_hi = int(ip[lo]), int(ip[hi])
        local = (ip[lo:hi + 1] - e_lo).astype(np.int64)
        rels.append(RelShard(s, t, local, e_lo, e_hi,
                             graph.indices_slice(r, e_lo, e_hi) if with_indices else None))
    return bounds, rels


# ----------------------------------------------------------------------------- seeds

_train_cache: dict = {}


def train_ids(cfg: Config) -> np.ndarray:
    key = (cfg.name, cfg.gen_seed)
    if key not in _train_cache:
        n = int(cfg.vt_counts[cfg.seed_vt])
        if cfg.train_count >= n:
            ids = np.arange(n, dtype=np.int64)
        else:
            thresh = int(min(2**64 - 1, (cfg.train_count / n) * 2**64))
            cap = int(cfg.train_count * 1.1) + 1024
            out = np.empty(cap, dtype=np.int64)
            m = lib().sy_select_train(cfg.gen_seed, cfg.seed_vt, n, thresh, out.ctypes.data, cap)
            ids = out[:min(m, cap)].copy()
        _train_cache[key] = ids
    return _train_cache[key]


_perm_cache: dict = {}


def batch_seeds(cfg: Config, g: int, batch: int | None = None) -> np.ndarray:
    """Seeds (gids) of global batch g: a seeded epoch permutation of the train
    ids, sliced.  Rank p's b-th batch is g = b * world + p."""
    B = cfg.batch if batch is None else batch
    ids = train_ids(cfg)
    per_epoch = max(1, len(ids) // B)
    epoch, k = divmod(g, per_epoch)
    pk = (cfg.name, epoch)
    if pk not in _perm_cache:
        keys = np.empty(len(ids), dtype=np.uint64)
        lib().sy_perm_keys(cfg.gen_seed, epoch, ids.ctypes.data, len(ids), keys.ctypes.data)
        _perm_cache.clear()
        _perm_cache[pk] = ids[np.argsort(keys, kind="stable")]
    perm = _perm_cache[pk]
    return (perm[k * B:(k + 1) * B] + int(cfg.offsets[cfg.seed_vt])).astype(np.int64)


# link-prediction inputs (NEXT-3): the paper trains LP on all edges with
# fanout 25, 15; a batch is a seeded uniform draw of existing edges.
LP_TAG = 0x4C50   # 'LP'


def lp_fanouts(cfg: Config) -> list:
    return [[25] * cfg.n_rel, [15] * cfg.n_rel]


def lp_rel(cfg: Config) -> int:
    """The relation LP batches train on: the first one into the seed type."""
    return next(r for r, x in enumerate(cfg.rels) if x[2] == cfg.seed_vt)


def lp_positives(cfg: Config, graph, rel: int, g: int, n: int | None = None):
    """Positive edges (src gid, dst gid) of global LP batch g: n uniformly drawn edge
    positions of relation rel (with repetition), their dst from the CSC row and their
    src from the generator's source formula (no host copy of the indices needed)."""
    n = cfg.batch if n is None else n
    ip = graph.indptr[rel]
    E = int(ip[-1])
    rng = np.random.default_rng([int(cfg.gen_seed & 0xFFFFFFFF), LP_TAG, rel, g])
    e = rng.integers(0, E, n).astype(np.int64)
    _, s, t, _ = cfg.rels[rel]
    dst = np.searchsorted(ip, e, side="right") - 1 + int(cfg.offsets[t])
    tid = np.empty(n, np.int32)
    if cfg.locality > 0:
        dt = np.ascontiguousarray(dst - int(cfg.offsets[t]), np.int64)
        lib().sy_indices_at_loc(cfg.gen_seed, rel, int(cfg.vt_counts[s]), int(cfg.vt_counts[t]), e.ctypes.data,
                                dt.ctypes.data, n, cfg.q_thr, cfg.n_comm, tid.ctypes.data)
    else:
        lib().sy_indices_at(cfg.gen_seed, rel, int(cfg.vt_counts[s]), e.ctypes.data, n, tid.ctypes.data)
    src = tid.astype(np.int64) + int(cfg.offsets[s])
    return src, dst.astype(np.int64)


def batch_seeds_confined(cfg: Config, b: int, rank: int, world: int, batch: int | None = None) -> np.ndarray:
    """Seed confinement (NEXT-2: "split the training set accordingly ... a
    trainer samples target vertices ... from the local second-level partition"): rank p's
    b-th batch is slice b of a seeded epoch permutation of the train ids inside p's own
    vertex range [floor(p*N/P), floor((p+1)*N/P)) of the seed type."""
    B = cfg.batch if batch is None else batch
    n = int(cfg.vt_counts[cfg.seed_vt])
    lo, hi = (rank * n) // world, ((rank + 1) * n) // world
    ids = train_ids(cfg)
    ids = ids[(ids >= lo) & (ids < hi)]
    per_epoch = max(1, len(ids) // B)
    epoch, k = divmod(b, per_epoch)
    pk = (cfg.name, "confined", rank, world, epoch)
    if pk not in _perm_cache:
        keys = np.empty(len(ids), dtype=np.uint64)
        lib().sy_perm_keys(cfg.gen_seed, epoch, ids.ctypes.data, len(ids), keys.ctypes.data)
        _perm_cache.clear()
        _perm_cache[pk] = ids[np.argsort(keys, kind="stable")]
    perm = _perm_cache[pk]
    return (perm[k * B:(k + 1) * B] + int(cfg.offsets[cfg.seed_vt])).astype(np.int64)


def rng_seed(cfg: Config, g: int) -> int:
    return int(lib().sy_mix(cfg.base_rng ^ g))


def fanout_array(cfg: Config) -> np.ndarray:
    return np.array(cfg.fanouts, dtype=np.int32)
