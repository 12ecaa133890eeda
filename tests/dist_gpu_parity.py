"""Multi-GPU parity (one process per GPU, peer shards mapped over NVLink via CUDA IPC).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29511 tests/dist_gpu_parity.py [--config C2] [--batches 4]

Every rank samples its own global batches g = b * N + rank with the graph and
features range-sharded over the N GPUs, and compares blocks + feature bytes with
the CPU oracle on the unsharded graph, bit-exactly (P-invariance, DESIGN §3 #13).
Exit status 0 iff every rank matched.
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--replicate", default="auto", help="replicated feature types: auto | none")
    ap.add_argument("--depth", type=int, default=2, help="pipelined check: launches in flight")
    ap.add_argument("--bundle", type=int, default=4, help="pipelined check: mini-batches per launch")
    ap.add_argument("--backend", default="nccl", help="process group for the blob all-gather (gloo: CPU)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (two processes sharing one GPU still map each other's shards "
                         "through CUDA IPC: the multi-process path, testable on a 1-GPU box)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    from gpu_util import assert_same_batch, assert_same_features
    from paper_2112_15345_b200 import Context
    from synth.device import load_context

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(args.backend)
    cfg = synth.config(args.config)
    g = synth.build_host_graph(cfg)
    ctx = Context(rank, world, local)
    shard = load_context(ctx, g, world, rank, f"cuda:{local}", replicate=args.replicate)
    ctx.connect_peers()
    small = cfg.name in ("C1", "C2", "C3")
    rows = {u: (synth.host_features(cfg, u) if small else synth.LazyRows(cfg, u)) for u in cfg.feats}
    ok = 0
    for b in range(args.batches):
        gi = b * world + rank
        seeds = synth.batch_seeds(cfg, gi)
        rs = synth.rng_seed(cfg, gi)
        res = oracle.sample(g, seeds, cfg.fanouts, rs)
        bl = ctx.sample_minibatch(torch.from_numpy(seeds).to(f"cuda:{local}"), cfg.fanouts, rs, features=True)
        assert_same_batch(res, bl, cfg.n_vt, cfg.n_rel)
        assert_same_features(res, [bl.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)], cfg, rows)
        # the separate gather entry point reads the same peer rows
        if small:
            outs = ctx.gather_features(bl)
            assert_same_features(res, outs, cfg, rows)
        bl.free()
        ok += 1
    # pipelined, bundled launches (the bench's mode) read the same peer shards
    D, B = args.depth, args.bundle
    ctx.set_pipeline(D, B)
    gis = [1000 + (b * world + rank) for b in range(D * B)]
    dev = [torch.from_numpy(synth.batch_seeds(cfg, gi)).to(f"cuda:{local}") for gi in gis]
    launches = [ctx.sample_bundle(dev[i:i + B], cfg.fanouts, [synth.rng_seed(cfg, gi) for gi in gis[i:i + B]],
                                  features=True, async_=True) for i in range(0, D * B, B)]
    for li, bls in enumerate(launches):
        for j, bl in enumerate(bls):
            gi = gis[B * li + j]
            res = oracle.sample(g, synth.batch_seeds(cfg, gi), cfg.fanouts, synth.rng_seed(cfg, gi))
            assert_same_batch(res, bl, cfg.n_vt, cfg.n_rel)
            assert_same_features(res, [bl.features(u) if u in cfg.feats else None for u in range(cfg.n_vt)], cfg,
                                 rows)
            bl.free()
            ok += 1
    t = torch.tensor([ok], device="cuda" if args.backend == "nccl" else "cpu")
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist parity OK: {args.config} world={world}, {int(t.item())} batches bit-exact vs oracle", flush=True)
    ctx.close()
    del shard
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
