"""Helpers of the GPU parity tests: run the CUDA path through the C ABI and compare
it element by element with the oracle on the same seeded inputs."""
import numpy as np

import oracle
import synth
from invariants import check_batch


def gpu_levels(blocks, n_vt):
    """levels[l][u] as numpy (l = 0 seeds = dst of block 0; l = h+1 = src of block h)."""
    L = blocks.n_hops
    levels = [[blocks[0].dst_nodes[u].cpu().numpy() for u in range(n_vt)]]
    for h in range(L):
        levels.append([blocks[h].src_nodes[u].cpu().numpy() for u in range(n_vt)])
    return levels


def gpu_blocks(blocks, n_rel):
    out = []
    for h in range(blocks.n_hops):
        b = blocks[h]
        out.append([{"indptr": b.indptr[r].cpu().numpy(), "indices": b.indices[r].cpu().numpy(),
                     "eids": b.eids[r].cpu().numpy()} for r in range(n_rel)])
    return out


def assert_same_batch(res, blocks, n_vt, n_rel):
    """Bit-exact: every node list, block CSC and edge-id array."""
    lv = gpu_levels(blocks, n_vt)
    assert len(lv) == len(res.levels)
    for l in range(len(lv)):
        for u in range(n_vt):
            np.testing.assert_array_equal(lv[l][u], res.levels[l][u], err_msg=f"level {l} type {u}")
    gb = gpu_blocks(blocks, n_rel)
    for h in range(len(gb)):
        for r in range(n_rel):
            o = res.blocks[h][r]
            np.testing.assert_array_equal(gb[h][r]["indptr"], o.indptr, err_msg=f"indptr h{h} r{r}")
            np.testing.assert_array_equal(gb[h][r]["indices"], o.indices, err_msg=f"indices h{h} r{r}")
            np.testing.assert_array_equal(gb[h][r]["eids"], o.eids, err_msg=f"eids h{h} r{r}")
    return lv, gb


def assert_same_features(res, feats, cfg, host_rows):
    for u in range(cfg.n_vt):
        if u not in cfg.feats:
            assert feats[u] is None
            continue
        rows = host_rows[u]
        if isinstance(rows, synth.LazyRows):
            # huge configs: out_u[i] = rows_u[tid_i] with rows_u defined by the generator
            want = rows.take(res.input_nodes(u) - int(cfg.offsets[u]))
        else:
            want = oracle.gather(res, cfg.vt_counts, u, rows)
        got = feats[u].cpu().numpy()
        assert got.shape == want.shape
        assert got.tobytes() == want.tobytes(), f"feature bytes differ for type {u}"


def run_and_compare(ctx, graph, cfg, seeds, fanouts, rng, host_rows=None, check_invariants=False):
    import torch
    seeds = np.asarray(seeds, np.int64)
    res = oracle.sample(graph, seeds, fanouts, rng)
    blocks = ctx.sample_blocks(torch.from_numpy(seeds).to(f"cuda:{ctx.device}"), fanouts, rng)
    lv, gb = assert_same_batch(res, blocks, cfg.n_vt, cfg.n_rel)
    if check_invariants:
        check_batch(graph, seeds, fanouts, lv, gb)
    if host_rows is not None:
        feats = ctx.gather_features(blocks)
        assert_same_features(res, feats, cfg, host_rows)
    return res, blocks
