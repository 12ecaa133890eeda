"""World-size-2 host logic of the multi-GPU path, on CPU with the gloo backend.

Each rank builds its shard of the same seeded graph (per-type range partition,
edge owner = dst owner S:178), publishes its shard metadata, all-gathers it, and
runs the library's partition check (eg_check_shard_metas, the same check
eg_import_shards runs before mapping peers over NVLink).  Also: the shards
reassemble the global CSC, and the ranks' batches of one epoch are disjoint.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _metas(world, rank, graph):
    import synth
    from paper_2112_15345_b200 import shard_meta
    cfg = graph.cfg
    bounds, rels = synth.shard(graph, world, rank)
    rd = [{"src_vt": r.src_vt, "dst_vt": r.dst_vt, "n_local_edges": r.e_hi - r.e_lo, "edge_base": r.e_lo,
           "max_degree": int(np.diff(r.indptr).max()) if len(r.indptr) > 1 else 0} for r in rels]
    return bounds, rels, shard_meta(rank, world, cfg.vt_counts, bounds, rd,
                                    [cfg.row_bytes(u) for u in range(cfg.n_vt)])


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from paper_2112_15345_b200 import EgError, check_shard_metas
        cfg = synth.config("C1")
        g = synth.build_host_graph(cfg)
        bounds, rels, meta = _metas(world, rank, g)
        blobs = [None] * world
        dist.all_gather_object(blobs, bytes(meta))
        from paper_2112_15345_b200.egonet import ShardMeta
        metas = [ShardMeta.from_buffer_copy(b) for b in blobs]
        edges, mx = check_shard_metas(metas)
        assert list(edges) == [r[3] for r in cfg.rels]
        assert list(mx) == [int(np.diff(ip).max()) for ip in g.indptr]
        # a rank whose shard does not start where the previous one ended is rejected
        bad = [ShardMeta.from_buffer_copy(b) for b in blobs]
        bad[1].rel_edge_base[0] += 1
        try:
            check_shard_metas(bad)
            raise AssertionError("inconsistent edge bases accepted")
        except EgError as e:
            assert e.code == -6 and "edge bases" in str(e)
        bad = [ShardMeta.from_buffer_copy(b) for b in blobs]
        bad[0].bounds[0][1] -= 1
        try:
            check_shard_metas(bad)
            raise AssertionError("inconsistent bounds accepted")
        except EgError as e:
            assert e.code == -6
        # the shards reassemble the global CSC
        parts = [None] * world
        dist.all_gather_object(parts, [(r.indptr, r.indices, r.e_lo) for r in rels])
        for r in range(cfg.n_rel):
            ip = np.concatenate([parts[p][r][0][:-1] + parts[p][r][2] for p in range(world)] + [[g.indptr[r][-1]]])
            ix = np.concatenate([parts[p][r][1] for p in range(world)])
            assert np.array_equal(ip, g.indptr[r]) and np.array_equal(ix, g.indices[r])
        # rank p's b-th batch is global batch b * world + p: disjoint within an epoch
        mine = np.concatenate([synth.batch_seeds(cfg, b * world + rank) for b in range(5)])
        allseeds = [None] * world
        dist.all_gather_object(allseeds, mine)
        cat = np.concatenate(allseeds)
        assert len(np.unique(cat)) == len(cat)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "FAIL " + repr(e) + traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_world2_gloo_partition_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_single_process_meta_check_world3():
    import synth
    from paper_2112_15345_b200 import check_shard_metas
    g = synth.build_host_graph(synth.config("C1"))
    metas = [_metas(3, p, g)[2] for p in range(3)]
    edges, _ = check_shard_metas(metas)
    assert list(edges) == [40000, 30000, 30000]
