"""Put a rank's shard of a synthetic graph on its GPU (input plumbing, untimed).

CSC rows come from the host generator (sliced per rank); src tids of huge
relations and all feature rows are generated directly on the device by
synth_dev.cu with the same formulas as the host (byte-identical, tested).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import (HostGraph, NP_DTYPE, Config, dev_lib, shard)


def _torch():
    import torch
    return torch


def feature_shard(cfg: Config, u: int, lo: int, hi: int, device):
    torch = _torch()
    dim, dt = cfg.feats[u]
    tdt = torch.float32 if dt == 0 else torch.float16
    t = torch.empty((hi - lo, dim), dtype=tdt, device=device)
    if hi > lo:
        s = torch.cuda.current_stream(device)
        rc = dev_lib().sy_features_dev(cfg.gen_seed, u, lo, hi, dim, dt, ctypes.c_void_p(t.data_ptr()),
                                       ctypes.c_void_p(s.cuda_stream))
        if rc:
            raise RuntimeError(f"sy_features_dev failed: {rc}")
    return t


def host_feature_shard(cfg: Config, u: int, lo: int, hi: int):
    """The same rows in pinned host memory (NEXT-4 ii: features in CPU memory, read
    zero-copy by the gather kernel over PCIe)."""
    from . import lib
    torch = _torch()
    dim, dt = cfg.feats[u]
    tdt = torch.float32 if dt == 0 else torch.float16
    t = torch.empty((hi - lo, dim), dtype=tdt, pin_memory=True)
    step = 1 << 22   # rows per generator call (OpenMP inside)
    base = t.data_ptr()
    rb = t.element_size() * dim
    for a in range(lo, hi, step):
        b = min(hi, a + step)
        lib().sy_features(cfg.gen_seed, u, a, b, dim, dt, ctypes.c_void_p(base + (a - lo) * rb))
    return t


def device_shard(graph: HostGraph, world: int, rank: int, device, features=True):
    """Returns dict(vt_counts, bounds, rels=[{src_vt,dst_vt,indptr,indices,edge_base}], feats=[tensor|None])."""
    torch = _torch()
    cfg = graph.cfg
    materialized = bool(graph.indices) and all(x is not None for x in graph.indices)
    bounds, rels = shard(graph, world, rank, with_indices=materialized)
    out_rels = []
    s = torch.cuda.current_stream(device)
    for r, rs in enumerate(rels):
        ip = torch.from_numpy(rs.indptr).to(device)
        if rs.indices is not None:
            ix = torch.from_numpy(np.ascontiguousarray(rs.indices, np.int32)).to(device)
        else:
            ix = torch.empty(rs.e_hi - rs.e_lo, dtype=torch.int32, device=device)
            if rs.e_hi > rs.e_lo:
                n_src = int(cfg.vt_counts[rs.src_vt])
                rc = dev_lib().sy_indices_dev(cfg.gen_seed, r, n_src, rs.e_lo, rs.e_hi,
                                              ctypes.c_void_p(ix.data_ptr()), ctypes.c_void_p(s.cuda_stream))
                if rc:
                    raise RuntimeError(f"sy_indices_dev failed: {rc}")
        out_rels.append({"src_vt": rs.src_vt, "dst_vt": rs.dst_vt, "indptr": ip, "indices": ix,
                         "edge_base": rs.e_lo})
    feats = []
    for u in range(cfg.n_vt):
        if features == "host" and u in cfg.feats:
            feats.append(host_feature_shard(cfg, u, int(bounds[u][rank]), int(bounds[u][rank + 1])))
        elif features and u in cfg.feats:
            feats.append(feature_shard(cfg, u, int(bounds[u][rank]), int(bounds[u][rank + 1]), device))
        else:
            feats.append(None)
    torch.cuda.synchronize(device)
    return {"vt_counts": cfg.vt_counts, "bounds": bounds, "rels": out_rels, "feats": feats}


REPLICA_BUDGET = 64 << 20   # bytes: "auto" replicates feature types whose full table is this small
FIT_BUDGET = 45 << 30       # bytes: "fit" replicates types (smallest first) up to a quarter of a B200's HBM


def replica_types(cfg: Config, world: int, spec="auto", budget: int = REPLICA_BUDGET):
    """Vertex types whose features follow the replicated partition policy.
    spec: "auto" (world > 1: every type whose full table is <= budget bytes), "fit" (world > 1:
    whole tables, smallest first, while their sum stays <= FIT_BUDGET), "none", or an
    iterable of type indices."""
    if spec is None or spec == "none":
        return []
    if spec == "fit":
        if world <= 1:
            return []
        sizes = sorted((int(cfg.vt_counts[u]) * dim * (4 if dt == 0 else 2), u) for u, (dim, dt) in cfg.feats.items())
        out, tot = [], 0
        for b, u in sizes:
            if tot + b > FIT_BUDGET:
                break
            out.append(u)
            tot += b
        return sorted(out)
    if spec == "auto":
        if world <= 1:
            return []
        out = []
        for u, (dim, dt) in cfg.feats.items():
            rb = dim * (4 if dt == 0 else 2)
            if int(cfg.vt_counts[u]) * rb <= budget:
                out.append(u)
        return sorted(out)
    return sorted(int(u) for u in spec)


def load_context(ctx, graph: HostGraph, world: int, rank: int, device, features=True, replicate="none"):
    """device_shard + Context.load_partition; returns the shard dict (keep it alive).
    features: True (rows on the GPU), False (none) or "host" (pinned host memory).
    replicate: see replica_types; each replicated type's full table is generated on this
    GPU (same formula as the shards) and handed to Context.set_feature_replica."""
    sh = device_shard(graph, world, rank, device, features)
    ctx.load_partition(sh["vt_counts"], sh["rels"], sh["feats"], bounds=sh["bounds"])
    cfg = graph.cfg
    sh["replicas"] = {}
    if features is True:
        for u in replica_types(cfg, world, replicate):
            t = feature_shard(cfg, u, 0, int(cfg.vt_counts[u]), device)
            _torch().cuda.synchronize(device)
            ctx.set_feature_replica(u, t)
            sh["replicas"][u] = t
    return sh
