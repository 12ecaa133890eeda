"""Python binding of the egonet C ABI (include/egonet.h).

Argument marshalling only: every step of the hot path runs in libegonet.so's
sm_100a kernels.  PyTorch provides device memory (shards, outputs), streams and
the process group used to all-gather the peer-shard blobs.  There is no CPU
fallback: if libegonet.so cannot be loaded, or no B200 is visible, calls fail.
"""
from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_PKG, "libegonet.so")

EG_MAX_VT = 8
EG_MAX_REL = 8
EG_MAX_RANKS = 8
EG_MAX_HOPS = 8

STATUS = {0: "EG_OK", -1: "EG_EINVAL", -2: "EG_ERANGE", -3: "EG_ENOMEM", -4: "EG_ECUDA", -6: "EG_EPEER",
          -7: "EG_ESTATE"}

ABI_SYMBOLS = [
    "eg_version", "eg_create", "eg_set_stream", "eg_load_partition", "eg_export_shard", "eg_import_shards",
    "eg_sample_blocks", "eg_block_view_get", "eg_blocks_n_hops", "eg_blocks_n_inputs", "eg_gather_features",
    "eg_blocks_free", "eg_destroy", "eg_last_error", "eg_set_profiling", "eg_get_profile", "eg_kernel_launches",
    "eg_range_bounds", "eg_batch_caps", "eg_attach_peer", "eg_sample_minibatch", "eg_blocks_wait",
    "eg_blocks_features", "eg_check_shard_metas", "eg_trace_get", "eg_set_pipeline", "eg_sample_bundle",
    "eg_blocks_stats", "eg_sample_lp_bundle", "eg_lp_view_get", "eg_sage_mean_layer", "eg_set_feature_replica",
    "eg_gather_path", "eg_counter_bytes", "eg_blocks_copy_features",
]

EG_FEATURES = 1
EG_ASYNC = 2


class EgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Relation(ctypes.Structure):
    _fields_ = [("src_vt", ctypes.c_int32), ("dst_vt", ctypes.c_int32), ("indptr", ctypes.c_void_p),
                ("indices", ctypes.c_void_p), ("n_local_edges", ctypes.c_int64), ("edge_base", ctypes.c_int64)]


class Features(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_void_p), ("row_bytes", ctypes.c_int64)]


class ShardMeta(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("n_vt", ctypes.c_int32), ("n_rel", ctypes.c_int32),
                ("vt_counts", ctypes.c_int64 * EG_MAX_VT),
                ("bounds", (ctypes.c_int64 * (EG_MAX_RANKS + 1)) * EG_MAX_VT),
                ("rel_src_vt", ctypes.c_int32 * EG_MAX_REL), ("rel_dst_vt", ctypes.c_int32 * EG_MAX_REL),
                ("rel_n_local_edges", ctypes.c_int64 * EG_MAX_REL), ("rel_edge_base", ctypes.c_int64 * EG_MAX_REL),
                ("rel_max_degree", ctypes.c_int64 * EG_MAX_REL), ("row_bytes", ctypes.c_int64 * EG_MAX_VT)]


def shard_meta(rank, world, vt_counts, bounds, rels, row_bytes):
    """Build an eg_shard_meta (host only).  rels: list of dicts with src_vt, dst_vt,
    n_local_edges, edge_base, max_degree."""
    m = ShardMeta()
    m.rank, m.world, m.n_vt, m.n_rel = rank, world, len(vt_counts), len(rels)
    for t, n in enumerate(vt_counts):
        m.vt_counts[t] = int(n)
        m.row_bytes[t] = int(row_bytes[t])
        for q in range(world + 1):
            m.bounds[t][q] = int(bounds[t][q])
    for r, d in enumerate(rels):
        m.rel_src_vt[r], m.rel_dst_vt[r] = int(d["src_vt"]), int(d["dst_vt"])
        m.rel_n_local_edges[r], m.rel_edge_base[r] = int(d["n_local_edges"]), int(d["edge_base"])
        m.rel_max_degree[r] = int(d.get("max_degree", 0))
    return m


def check_shard_metas(metas):
    """eg_check_shard_metas over a list of ShardMeta (rank order); returns
    (rel_edges, rel_max_degree) or raises EgError(EG_EPEER)."""
    world = len(metas)
    arr = (ShardMeta * world)(*metas)
    edges = np.zeros(EG_MAX_REL, np.int64)
    mx = np.zeros(EG_MAX_REL, np.int64)
    msg = ctypes.create_string_buffer(256)
    rc = lib().eg_check_shard_metas(world, ctypes.cast(arr, ctypes.c_void_p), edges.ctypes.data, mx.ctypes.data,
                                    msg, 256)
    if rc:
        raise EgError(rc, msg.value.decode())
    n_rel = metas[0].n_rel
    return edges[:n_rel], mx[:n_rel]


class BlockView(ctypes.Structure):
    _fields_ = [("hop", ctypes.c_int32), ("n_vt", ctypes.c_int32), ("n_rel", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("dst_nodes", ctypes.c_void_p * EG_MAX_VT), ("n_dst", ctypes.c_int64 * EG_MAX_VT),
                ("src_nodes", ctypes.c_void_p * EG_MAX_VT), ("n_src", ctypes.c_int64 * EG_MAX_VT),
                ("indptr", ctypes.c_void_p * EG_MAX_REL), ("indices", ctypes.c_void_p * EG_MAX_REL),
                ("eids", ctypes.c_void_p * EG_MAX_REL), ("nnz", ctypes.c_int64 * EG_MAX_REL)]


class LpView(ctypes.Structure):
    _fields_ = [("n_pos", ctypes.c_int64), ("n_neg", ctypes.c_int32), ("rel", ctypes.c_int32),
                ("pos_src", ctypes.c_void_p), ("pos_dst", ctypes.c_void_p), ("neg_src", ctypes.c_void_p),
                ("neg_dst", ctypes.c_void_p), ("neg_dst_gid", ctypes.c_void_p)]


_lib = None


def lib(build_if_missing: bool = True):
    """Load libegonet.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        alt = os.environ.get("EG_LIB")   # A/B experiments: another build of the same library
        if build_if_missing and not alt:
            from . import build as _b
            _b.build()
        so = alt or _SO
        if not os.path.exists(so):
            raise RuntimeError(f"{so} missing: run paper_2112_15345_b200/build.py (no CPU fallback exists)")
        L = ctypes.CDLL(so)
        c = ctypes
        P = c.POINTER
        vp = c.c_void_p
        L.eg_version.restype = c.c_char_p
        L.eg_counter_bytes.restype = c.c_int64
        L.eg_last_error.argtypes = [vp]
        L.eg_last_error.restype = c.c_char_p
        L.eg_create.argtypes = [c.c_int32, c.c_int32, c.c_int32, vp, P(vp)]
        L.eg_set_stream.argtypes = [vp, vp]
        L.eg_load_partition.argtypes = [vp, c.c_int32, vp, vp, c.c_int32, vp, vp]
        L.eg_export_shard.argtypes = [vp, vp, P(c.c_size_t)]
        L.eg_import_shards.argtypes = [vp, vp, c.c_size_t]
        L.eg_attach_peer.argtypes = [vp, vp]
        L.eg_set_feature_replica.argtypes = [vp, c.c_int32, vp, c.c_int64]
        L.eg_gather_path.argtypes = [vp]
        L.eg_gather_path.restype = c.c_int32
        L.eg_set_pipeline.argtypes = [vp, c.c_int32, c.c_int32]
        L.eg_sample_bundle.argtypes = [vp, c.c_int32, vp, vp, c.c_int32, vp, vp, c.c_int32, vp]
        L.eg_sample_lp_bundle.argtypes = [vp, c.c_int32, vp, vp, vp, c.c_int32, c.c_int32, vp, c.c_int32, vp, vp,
                                          c.c_int32, vp]
        L.eg_lp_view_get.argtypes = [vp, P(LpView)]
        L.eg_sage_mean_layer.argtypes = [vp, vp, c.c_int32, c.c_int32, vp, c.c_int32, c.c_int64, vp, c.c_int64,
                                         c.c_int32, vp, c.c_int32, vp, c.c_int64, c.c_int32]
        L.eg_trace_get.argtypes = [vp, c.c_int32, c.c_char_p, c.c_size_t, P(c.c_double), P(c.c_int64)]
        L.eg_trace_get.restype = c.c_int32
        L.eg_check_shard_metas.argtypes = [c.c_int32, vp, vp, vp, c.c_char_p, c.c_size_t]
        L.eg_sample_blocks.argtypes = [vp, vp, c.c_int64, c.c_int32, vp, c.c_uint64, P(vp)]
        L.eg_block_view_get.argtypes = [vp, c.c_int32, P(BlockView)]
        L.eg_sample_minibatch.argtypes = [vp, vp, c.c_int64, c.c_int32, vp, c.c_uint64, c.c_int32, P(vp)]
        L.eg_blocks_wait.argtypes = [vp]
        L.eg_blocks_stats.argtypes = [vp, P(c.c_int64), vp]
        L.eg_blocks_features.argtypes = [vp, c.c_int32, P(vp), P(c.c_int64), P(c.c_int64)]
        L.eg_blocks_copy_features.argtypes = [vp, vp, c.c_int32]
        L.eg_blocks_n_hops.argtypes = [vp]
        L.eg_blocks_n_hops.restype = c.c_int32
        L.eg_blocks_n_inputs.argtypes = [vp, c.c_int32]
        L.eg_blocks_n_inputs.restype = c.c_int64
        L.eg_gather_features.argtypes = [vp, vp, vp]
        L.eg_blocks_free.argtypes = [vp]
        L.eg_destroy.argtypes = [vp]
        L.eg_set_profiling.argtypes = [vp, c.c_int32]
        L.eg_get_profile.argtypes = [vp, P(c.c_double)]
        L.eg_kernel_launches.argtypes = [vp]
        L.eg_kernel_launches.restype = c.c_int64
        L.eg_range_bounds.argtypes = [c.c_int64, c.c_int32, vp]
        L.eg_batch_caps.argtypes = [c.c_int32, vp, c.c_int32, vp, vp, vp, vp, c.c_int64, c.c_int32, vp, vp, vp]
        for name in ABI_SYMBOLS:
            if name not in ("eg_version", "eg_last_error", "eg_blocks_n_hops", "eg_blocks_n_inputs",
                            "eg_kernel_launches", "eg_trace_get", "eg_counter_bytes"):
                getattr(L, name).restype = c.c_int
        _lib = L
    return _lib


def version() -> str:
    return lib().eg_version().decode()


def counter_bytes() -> int:
    """Bytes of the per-batch counters read back to the host after every launch."""
    return int(lib().eg_counter_bytes())


def range_bounds(n: int, world: int) -> np.ndarray:
    out = np.empty(world + 1, dtype=np.int64)
    rc = lib().eg_range_bounds(n, world, out.ctypes.data)
    if rc:
        raise EgError(rc, "eg_range_bounds")
    return out


def batch_caps(vt_counts, rel_src, rel_dst, rel_edges, rel_maxdeg, n_seeds, fanouts):
    vtc = np.ascontiguousarray(vt_counts, np.int64)
    rs, rd = np.ascontiguousarray(rel_src, np.int32), np.ascontiguousarray(rel_dst, np.int32)
    re_, rm = np.ascontiguousarray(rel_edges, np.int64), np.ascontiguousarray(rel_maxdeg, np.int64)
    fo = np.ascontiguousarray(fanouts, np.int32)
    cn = np.empty(len(vtc), np.int64)
    ce = np.empty(fo.shape, np.int64)
    rc = lib().eg_batch_caps(len(vtc), vtc.ctypes.data, len(rs), rs.ctypes.data, rd.ctypes.data, re_.ctypes.data,
                             rm.ctypes.data, n_seeds, fo.shape[0], fo.ctypes.data, cn.ctypes.data, ce.ctypes.data)
    if rc:
        raise EgError(rc, "eg_batch_caps")
    return cn, ce


# ----------------------------------------------------------------------------- device wrappers

def _torch():
    import torch
    return torch


class _DevArray:
    """__cuda_array_interface__ over library-owned device memory; keeps the owning
    Blocks alive for as long as any tensor built from it lives."""

    def __init__(self, ptr, n, typestr, owner, device):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}
        self._owner = owner
        self._device = device


def _wrap(ptr, n, typestr, owner, device):
    torch = _torch()
    if n == 0 or not ptr:
        dt = {"<i8": torch.int64, "<i4": torch.int32}[typestr]
        return torch.empty(0, dtype=dt, device=device)
    with torch.cuda.device(device):
        return torch.as_tensor(_DevArray(ptr, n, typestr, owner, device), device=device)


class Block:
    """One hop's block: DGL-style bipartite CSC per relation (dst-in-src prefix)."""

    def __init__(self, view: BlockView, owner, device):
        self.hop = view.hop
        V, R = view.n_vt, view.n_rel
        self.n_dst = [int(view.n_dst[u]) for u in range(V)]
        self.n_src = [int(view.n_src[u]) for u in range(V)]
        self.nnz = [int(view.nnz[r]) for r in range(R)]
        self.dst_nodes = [_wrap(view.dst_nodes[u], self.n_dst[u], "<i8", owner, device) for u in range(V)]
        self.src_nodes = [_wrap(view.src_nodes[u], self.n_src[u], "<i8", owner, device) for u in range(V)]
        self.indptr = [None] * R
        self.indices = [_wrap(view.indices[r], self.nnz[r], "<i4", owner, device) for r in range(R)]
        self.eids = [_wrap(view.eids[r], self.nnz[r], "<i8", owner, device) for r in range(R)]
        self._view = view
        self._owner = owner
        self._device = device

    def set_indptr(self, rel_dst):
        for r, t in enumerate(rel_dst):
            self.indptr[r] = _wrap(self._view.indptr[r], self.n_dst[t] + 1, "<i4", self._owner, self._device)


class Blocks:
    """Handle of one sampled mini-batch (eg_blocks).  Sizes are resolved on first
    use (waiting for an EG_ASYNC batch); per-hop tensors are zero-copy views of
    library memory built lazily."""

    def __init__(self, ctx: "Context", handle: int, n_hops: int | None = None, inputs=None):
        self._ctx = ctx
        self._h = handle
        self.n_hops = lib().eg_blocks_n_hops(handle) if n_hops is None else n_hops
        self._views = None
        self._blocks = [None] * self.n_hops
        # The launch reads device / pinned seed (and positive-edge) buffers IN PLACE on the
        # library's lane stream, which torch's caching allocator does not know about: the
        # caller's tensors of the whole launch are held here until it has completed.
        self._inputs = inputs
        ctx._live.add(self)

    def wait(self):
        rc = lib().eg_blocks_wait(self._h)
        if rc:
            raise EgError(rc, lib().eg_last_error(self._ctx._h).decode())
        self._inputs = None   # the launch has completed: its inputs are no longer read
        return self

    @property
    def views(self):
        if self._views is None:
            self.wait()
            vs = []
            for h in range(self.n_hops):
                v = BlockView()
                rc = lib().eg_block_view_get(self._h, h, ctypes.byref(v))
                if rc:
                    raise EgError(rc, "eg_block_view_get")
                vs.append(v)
            self._views = vs
        return self._views

    def __getitem__(self, h) -> Block:
        if self._blocks[h] is None:
            b = Block(self.views[h], self, self._ctx.device)
            b.set_indptr(self._ctx.rel_dst)
            self._blocks[h] = b
        return self._blocks[h]

    def __len__(self):
        return self.n_hops

    def stats(self):
        """(total sampled edges, [input vertices per type]) in one call (waits if pending)."""
        e = ctypes.c_int64()
        n = np.zeros(EG_MAX_VT, np.int64)
        rc = lib().eg_blocks_stats(self._h, ctypes.byref(e), n.ctypes.data)
        if rc:
            raise EgError(rc, lib().eg_last_error(self._ctx._h).decode())
        self._inputs = None
        return int(e.value), [int(x) for x in n[:len(self._ctx.vt_counts)]]

    def nnz(self, h=None) -> int:
        vs = self.views
        hops = range(self.n_hops) if h is None else [h]
        return sum(int(vs[x].nnz[r]) for x in hops for r in range(vs[x].n_rel))

    def n_inputs(self, u) -> int:
        self.views
        return int(lib().eg_blocks_n_inputs(self._h, u))

    def lp(self):
        """Pairs of a link-prediction batch as zero-copy device tensors: pos_src,
        pos_dst [n_pos], neg_src, neg_dst [n_pos * n_neg] (int32 local ids = positions
        in block 0's dst nodes of the endpoint's type) and neg_dst_gid (int64)."""
        v = LpView()
        rc = lib().eg_lp_view_get(self._h, ctypes.byref(v))
        if rc:
            raise EgError(rc, lib().eg_last_error(self._ctx._h).decode())
        n, m = int(v.n_pos), int(v.n_pos) * int(v.n_neg)
        d = self._ctx.device
        return {"n_pos": n, "n_neg": int(v.n_neg), "rel": int(v.rel),
                "pos_src": _wrap(v.pos_src, n, "<i4", self, d), "pos_dst": _wrap(v.pos_dst, n, "<i4", self, d),
                "neg_src": _wrap(v.neg_src, m, "<i4", self, d), "neg_dst": _wrap(v.neg_dst, m, "<i4", self, d),
                "neg_dst_gid": _wrap(v.neg_dst_gid, m, "<i8", self, d)}

    def features(self, u):
        """Feature rows of the input vertices of type u gathered in the same graph
        launch (sample_minibatch(features=True)); zero-copy tensor or None."""
        torch = _torch()
        self.views
        ptr, n, rb = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        rc = lib().eg_blocks_features(self._h, u, ctypes.byref(ptr), ctypes.byref(n), ctypes.byref(rb))
        if rc:
            raise EgError(rc, "eg_blocks_features")
        if not ptr.value and n.value == 0 and not self._ctx.row_bytes[u]:
            return None
        dt, shape = self._ctx.feat_dtypes[u], self._ctx.feat_shapes[u]
        if n.value == 0:
            return torch.empty((0,) + shape, dtype=dt, device=self._ctx.device)
        raw = _wrap(ptr.value, n.value * rb.value // 4, "<i4", self, self._ctx.device)
        return raw.view(dt).view((n.value,) + shape)

    def copy_features(self, host, async_: bool = False):
        """eg_blocks_copy_features: the rows gathered in this batch's launch into caller
        memory, host[u] (pinned CPU tensors / numpy arrays with room for n_inputs(u) rows;
        None skips u).  async_: stream-ordered on the context's stream, not synchronized."""
        V = len(self._ctx.vt_counts)
        ptrs = (ctypes.c_void_p * V)()
        for u in range(V):
            o = host[u] if u < len(host) else None
            ptrs[u] = None if o is None else (o.data_ptr() if hasattr(o, "data_ptr") else o.ctypes.data)
        rc = lib().eg_blocks_copy_features(self._h, ptrs, EG_ASYNC if async_ else 0)
        if rc:
            raise EgError(rc, lib().eg_last_error(self._ctx._h).decode())
        self._inputs = None

    @property
    def handle(self):
        return self._h

    def free(self):
        """Release the batch's slot now (tensors obtained from this handle must no
        longer be used).  Otherwise it is released when the handle is garbage.  A handle
        that still holds the caller's input tensors of an unfinished launch waits for the
        launch first, so that those buffers are not recycled while it reads them."""
        if self._h:
            if self._inputs is not None:
                lib().eg_blocks_wait(self._h)   # errors are reported by the calls that read results
                self._inputs = None
            lib().eg_blocks_free(self._h)
            self._h = None
            self._ctx._live.discard(self)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One rank's view of the partitioned graph (eg_ctx)."""

    def __init__(self, rank: int = 0, world: int = 1, device: int = 0, stream=None):
        torch = _torch()
        self.rank, self.world, self.device = rank, world, device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        rc = lib().eg_create(rank, world, device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if rc:
            raise EgError(rc, "eg_create (needs an sm_100 GPU; there is no CPU fallback)")
        self._h = h
        self._keep = []
        self._live = weakref.WeakSet()   # Blocks handles not yet freed (close() frees them)
        self.rel_dst = []
        self.vt_counts = None
        self.row_bytes = []

    def _check(self, rc, what):
        if rc:
            raise EgError(rc, f"{what}: {lib().eg_last_error(self._h).decode()}")

    def set_stream(self, stream):
        self.stream = stream
        self._check(lib().eg_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)), "eg_set_stream")

    def load_partition(self, vt_counts, rels, feats, bounds=None):
        """rels: list of dicts {src_vt, dst_vt, indptr (cuda int64), indices (cuda int32), edge_base};
        feats: list (per type) of cuda tensors [n_local_rows, ...], pinned CPU tensors
        (world 1: gathered zero-copy over PCIe) or None."""
        vtc = np.ascontiguousarray(vt_counts, np.int64)
        self.vt_counts = vtc
        R = len(rels)
        carr = (Relation * R)()
        for r, d in enumerate(rels):
            ip, ix = d["indptr"], d["indices"]
            assert ip.dtype.itemsize == 8 and ix.dtype.itemsize == 4 and ip.is_cuda and ix.is_cuda
            carr[r] = Relation(d["src_vt"], d["dst_vt"], ip.data_ptr(), ix.data_ptr() if ix.numel() else None,
                               ix.numel(), int(d["edge_base"]))
            self._keep += [ip, ix]
        farr = (Features * len(vtc))()
        self.row_bytes = []
        for u in range(len(vtc)):
            t = feats[u] if feats is not None and u < len(feats) else None
            if t is None:
                farr[u] = Features(None, 0)
                self.row_bytes.append(0)
            else:
                # cuda tensors, or CPU tensors (pinned: read zero-copy over PCIe at world 1; the
                # library rejects pageable memory with EG_EINVAL)
                assert t.is_contiguous()
                rb = t.stride(0) * t.element_size() if t.dim() > 1 else t.element_size()
                farr[u] = Features(t.data_ptr() if t.numel() else None, rb)
                self.row_bytes.append(rb)
                self._keep.append(t)
        self.rel_dst = [int(d["dst_vt"]) for d in rels]
        self.rel_src = [int(d["src_vt"]) for d in rels]
        self.feat_dtypes = [None if (feats is None or u >= len(feats) or feats[u] is None) else feats[u].dtype
                            for u in range(len(vtc))]
        self.feat_shapes = [None if (feats is None or u >= len(feats) or feats[u] is None) else tuple(feats[u].shape[1:])
                            for u in range(len(vtc))]
        b = None
        if bounds is not None:
            b = np.ascontiguousarray(bounds, np.int64)
            self._keep.append(b)
        self._check(lib().eg_load_partition(self._h, len(vtc), vtc.ctypes.data, b.ctypes.data if b is not None else None,
                                            R, ctypes.cast(carr, ctypes.c_void_p), ctypes.cast(farr, ctypes.c_void_p)),
                    "eg_load_partition")

    def export_shard(self) -> bytes:
        n = ctypes.c_size_t(0)
        self._check(lib().eg_export_shard(self._h, None, ctypes.byref(n)), "eg_export_shard")
        buf = ctypes.create_string_buffer(n.value)
        self._check(lib().eg_export_shard(self._h, buf, ctypes.byref(n)), "eg_export_shard")
        return buf.raw[:n.value]

    def attach_peer(self, peer: "Context"):
        """Single-process peer mapping (another rank's context in this process)."""
        self._check(lib().eg_attach_peer(self._h, peer._h), "eg_attach_peer")

    def gather_path(self) -> str:
        """Kernel of the last enqueued feature gather: "tma" (gather4), "ldg" or "none"."""
        return {0: "tma", 1: "ldg"}.get(int(lib().eg_gather_path(self._h)), "none")

    def set_feature_replica(self, vt: int, rows):
        """Replicated partition policy for type vt's features: `rows` is the type's full
        table on this GPU (cuda tensor [N_vt, ...]); None restores the sharded policy.
        Call before the first sampling call."""
        if rows is None:
            self._check(lib().eg_set_feature_replica(self._h, vt, None, 0), "eg_set_feature_replica")
            return
        assert rows.is_contiguous()   # device memory of this GPU: checked by the library (EG_EINVAL)
        self._check(lib().eg_set_feature_replica(self._h, vt, ctypes.c_void_p(rows.data_ptr()), rows.shape[0]),
                    "eg_set_feature_replica")
        self._keep.append(rows)

    def import_shards(self, blobs):
        stride = len(blobs[0])
        assert all(len(b) == stride for b in blobs)
        joined = ctypes.create_string_buffer(b"".join(blobs), stride * len(blobs))
        self._check(lib().eg_import_shards(self._h, joined, stride), "eg_import_shards")

    def connect_peers(self, group=None):
        """All-gather the shard blobs over a torch.distributed group and map the peers."""
        import torch.distributed as dist
        blob = self.export_shard()
        blobs = [None] * self.world
        dist.all_gather_object(blobs, blob, group=group)
        self.import_shards(blobs)

    def sample_blocks(self, seeds, fanouts, rng_seed: int) -> Blocks:
        """seeds: cuda int64 tensor (or host numpy int64 / pinned tensor); fanouts [hop][rel]."""
        torch = _torch()
        fo = np.ascontiguousarray(fanouts, np.int32)
        if isinstance(seeds, np.ndarray):
            seeds = np.ascontiguousarray(seeds, np.int64)
            ptr, n = seeds.ctypes.data, len(seeds)
        else:
            assert seeds.dtype == torch.int64 and seeds.is_contiguous()
            ptr, n = seeds.data_ptr(), seeds.numel()
        h = ctypes.c_void_p()
        self._check(lib().eg_sample_blocks(self._h, ptr if n else None, n, fo.shape[0], fo.ctypes.data,
                                           rng_seed & (2**64 - 1), ctypes.byref(h)), "eg_sample_blocks")
        return Blocks(self, h.value)   # synchronous: the inputs have been read

    def sample_minibatch(self, seeds, fanouts, rng_seed: int, features: bool = True, async_: bool = False) -> Blocks:
        """One CUDA-graph launch: sample + compact every hop (+ gather features into
        library-owned buffers, Blocks.features(u)).  async_=True returns after
        enqueueing; sizes are resolved on first use."""
        torch = _torch()
        fo = np.ascontiguousarray(fanouts, np.int32)
        if isinstance(seeds, np.ndarray):
            seeds = np.ascontiguousarray(seeds, np.int64)
            ptr, n = seeds.ctypes.data, len(seeds)
        else:
            assert seeds.dtype == torch.int64 and seeds.is_contiguous()
            ptr, n = seeds.data_ptr(), seeds.numel()
        flags = (EG_FEATURES if features else 0) | (EG_ASYNC if async_ else 0)
        h = ctypes.c_void_p()
        self._check(lib().eg_sample_minibatch(self._h, ptr if n else None, n, fo.shape[0], fo.ctypes.data,
                                              rng_seed & (2**64 - 1), flags, ctypes.byref(h)), "eg_sample_minibatch")
        return Blocks(self, h.value, inputs=[seeds] if async_ else None)

    def sample_bundle(self, seeds_list, fanouts, rng_seeds, features: bool = True, async_: bool = False):
        """Several mini-batches as ONE graph launch (bundle); returns one Blocks per batch."""
        torch = _torch()
        fo = np.ascontiguousarray(fanouts, np.int32)
        n = len(seeds_list)
        ptrs = (ctypes.c_void_p * n)()
        cnts = np.zeros(n, np.int64)
        keep = []
        for i, s in enumerate(seeds_list):
            if isinstance(s, np.ndarray):
                s = np.ascontiguousarray(s, np.int64)
                keep.append(s)
                ptrs[i], cnts[i] = s.ctypes.data, len(s)
            else:
                assert s.dtype == torch.int64 and s.is_contiguous()
                keep.append(s)
                ptrs[i], cnts[i] = s.data_ptr(), s.numel()
        rs = np.ascontiguousarray([int(x) & (2**64 - 1) for x in rng_seeds], np.uint64)
        outs = (ctypes.c_void_p * n)()
        flags = (EG_FEATURES if features else 0) | (EG_ASYNC if async_ else 0)
        self._check(lib().eg_sample_bundle(self._h, n, ctypes.cast(ptrs, ctypes.c_void_p), cnts.ctypes.data,
                                           fo.shape[0], fo.ctypes.data, rs.ctypes.data, flags,
                                           ctypes.cast(outs, ctypes.c_void_p)), "eg_sample_bundle")
        L = fo.shape[0]
        held = keep if async_ else None   # every batch of the launch holds all its inputs
        return [Blocks(self, outs[i], L, inputs=held) for i in range(n)]

    def sample_lp_bundle(self, src_list, dst_list, rel: int, n_neg: int, neg_seeds, fanouts, rng_seeds,
                         features: bool = True, async_: bool = False):
        """Link-prediction mini-batches (positives (src, dst) of relation rel + n_neg
        corrupted dsts each) as ONE graph launch; one Blocks per batch, with .lp()."""
        torch = _torch()
        fo = np.ascontiguousarray(fanouts, np.int32)
        n = len(src_list)
        assert len(dst_list) == n
        sp, dp = (ctypes.c_void_p * n)(), (ctypes.c_void_p * n)()
        cnts = np.zeros(n, np.int64)
        keep = []
        for i, (a, b) in enumerate(zip(src_list, dst_list)):
            for arr, tab in ((a, sp), (b, dp)):
                if isinstance(arr, np.ndarray):
                    arr = np.ascontiguousarray(arr, np.int64)
                    keep.append(arr)
                    tab[i] = arr.ctypes.data
                    m = len(arr)
                else:
                    assert arr.dtype == torch.int64 and arr.is_contiguous()
                    keep.append(arr)
                    tab[i] = arr.data_ptr()
                    m = arr.numel()
                assert tab is sp or m == cnts[i], "src / dst lengths differ"
                cnts[i] = m
        ns = np.ascontiguousarray([int(x) & (2**64 - 1) for x in neg_seeds], np.uint64)
        rs = np.ascontiguousarray([int(x) & (2**64 - 1) for x in rng_seeds], np.uint64)
        outs = (ctypes.c_void_p * n)()
        flags = (EG_FEATURES if features else 0) | (EG_ASYNC if async_ else 0)
        self._check(lib().eg_sample_lp_bundle(self._h, n, ctypes.cast(sp, ctypes.c_void_p),
                                              ctypes.cast(dp, ctypes.c_void_p), cnts.ctypes.data, rel, n_neg,
                                              ns.ctypes.data, fo.shape[0], fo.ctypes.data, rs.ctypes.data, flags,
                                              ctypes.cast(outs, ctypes.c_void_p)), "eg_sample_lp_bundle")
        held = keep if async_ else None
        return [Blocks(self, outs[i], fo.shape[0], inputs=held) for i in range(n)]

    def sample_lp(self, src, dst, rel: int, n_neg: int, neg_seed: int, fanouts, rng_seed: int,
                  features: bool = True, async_: bool = False) -> Blocks:
        """One link-prediction mini-batch (eg_sample_lp_bundle with one batch)."""
        return self.sample_lp_bundle([src], [dst], rel, n_neg, [neg_seed], fanouts, [rng_seed], features, async_)[0]

    def sage_mean_layer(self, blocks: Blocks, hop: int, rel: int, x_src, w, x_dst=None, out=None,
                        accumulate: bool = False):
        """The consumer step (NEXT-4 i): one GraphSAGE-mean layer over relation rel of block
        hop on the tensor cores -- out = W_self x_dst + W_neigh mean(x_src over sampled
        in-edges), pre-activation, fp32 [n_dst, H].  x_src / x_dst: cuda fp32 / fp16 /
        bf16 [rows, F]; w: cuda bf16 [H, 2F] ([W_self | W_neigh]) or [H, F] without x_dst."""
        torch = _torch()
        dt = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}[x_src.dtype]
        F = x_src.shape[1]
        assert w.dtype == torch.bfloat16 and w.is_contiguous()
        H = w.shape[0]
        ok = 0 <= hop < blocks.n_hops and 0 <= rel < len(self.rel_dst)   # else the library reports EG_EINVAL
        n_dst = blocks[hop].n_dst[self.rel_dst[rel]] if ok else 0
        if out is None:
            out = (torch.zeros if accumulate else torch.empty)((n_dst, H), dtype=torch.float32, device=self.device)
        if x_dst is not None:
            assert x_dst.dtype == x_src.dtype and x_dst.shape[1] == F
        self._check(lib().eg_sage_mean_layer(self._h, blocks.handle, hop, rel, x_src.data_ptr(), dt, x_src.stride(0),
                                             x_dst.data_ptr() if x_dst is not None else None,
                                             x_dst.stride(0) if x_dst is not None else 0, F, w.data_ptr(), H,
                                             out.data_ptr(), out.stride(0), 1 if accumulate else 0),
                    "eg_sage_mean_layer")
        return out

    def gather_features(self, blocks: Blocks, out=None, types=None):
        """Feature rows of the input vertices per type (None for types without
        features).  `out` may give preallocated (device or host) tensors / arrays."""
        torch = _torch()
        V = len(self.vt_counts)
        types = range(V) if types is None else types
        outs = [None] * V
        ptrs = (ctypes.c_void_p * V)()
        for u in types:
            if not self.row_bytes[u]:
                continue
            if out is not None and out[u] is not None:
                o = out[u]
            else:
                o = torch.empty((blocks.n_inputs(u),) + self.feat_shapes[u], dtype=self.feat_dtypes[u],
                                device=self.device)
            outs[u] = o
            ptrs[u] = o.data_ptr() if hasattr(o, "data_ptr") else o.ctypes.data
        self._check(lib().eg_gather_features(self._h, blocks.handle, ptrs), "eg_gather_features")
        return outs

    def set_pipeline(self, depth: int, bundle: int = 1):
        """Up to `depth` launches in flight (independent lanes / streams), each carrying up
        to `bundle` mini-batches (sample_bundle)."""
        self._check(lib().eg_set_pipeline(self._h, depth, bundle), "eg_set_pipeline")
        self.bundle = bundle

    def set_profiling(self, on: bool):
        self._check(lib().eg_set_profiling(self._h, 1 if on else 0), "eg_set_profiling")

    def profile(self):
        out = (ctypes.c_double * 4)()
        self._check(lib().eg_get_profile(self._h, out), "eg_get_profile")
        return {"sample_ms": out[0], "gather_ms": out[1], "n_sample": int(out[2]), "n_gather": int(out[3])}

    def trace(self):
        """Per-stage device time accumulated with EG_TRACE=1 (ms total, count)."""
        n = lib().eg_trace_get(self._h, -1, None, 0, None, None)
        out = {}
        for i in range(n):
            name = ctypes.create_string_buffer(64)
            ms, cnt = ctypes.c_double(), ctypes.c_int64()
            lib().eg_trace_get(self._h, i, name, 64, ctypes.byref(ms), ctypes.byref(cnt))
            out[name.value.decode()] = (ms.value, cnt.value)
        return out

    def kernel_launches(self) -> int:
        return int(lib().eg_kernel_launches(self._h))

    def close(self):
        """Destroy the library context, then drop the buffers it borrowed (the shard
        tensors kept alive for it), so that their device memory is released now rather
        than whenever this object is collected."""
        if self._h:
            for b in list(self._live):   # before the library frees their slots
                b.free()
            lib().eg_destroy(self._h)
            self._h = None
        self._keep = []
        self.__dict__.pop("_shard", None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
