"""Consumer-step benchmark (NEXT-4 i): the fused GraphSAGE-mean layer (eg_sage_mean_layer,
tcgen05) on the input layer of real mini-batches, one B200.

    python profiles/sage_bench.py [--config C4] [--hidden 256] [--reps 20]

The input layer of a batch: out[n_dst, H] = [x_dst | mean x_src] [W_self | W_neigh]^T over
relation 0 of the last block.  Reports per layer call (CUDA events, median of reps):
  algorithmic bytes = nnz * F * esz (neighbour rows) + n_dst * F * esz (self rows)
                      + n_dst * H * 4 (fp32 out) + nnz * 4 + (n_dst + 1) * 4 (CSC)
  -> GB/s vs the measured HBM peak (the bound: neighbour rows are gathered from HBM);
  flops = 2 * n_dst_padded * H * K -> TFLOP/s vs the dense bf16 peak (context only).
Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batches", type=int, default=8, help="mini-batches whose input layers are timed")
    ap.add_argument("--trace", action="store_true",
                    help="with an EG_SAGE_TRACE build: print the phase stamps of CTAs 0 / 100 of the last call")
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    from paper_2112_15345_b200 import Context
    from synth.device import load_context

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6450.0))
    bf16_tf = float(peaks.get("bf16_tflops", 1650.0))
    cfg = synth.config(args.config)
    g = synth.build_host_graph(cfg, materialize_indices=cfg.name in ("C1", "C2", "C3"))
    ctx = Context(0, 1, 0)
    shard = load_context(ctx, g, 1, 0, "cuda:0")
    L = len(cfg.fanouts)
    r = 0
    s, t = cfg.rels[r][1], cfg.rels[r][2]
    F = cfg.feats[s][0]
    H = args.hidden
    w = (torch.randn(H, 2 * F) / (2 * F) ** 0.5).to(torch.bfloat16).cuda()
    rows = []
    for gi in range(args.batches):
        b = ctx.sample_minibatch(torch.from_numpy(synth.batch_seeds(cfg, gi)).cuda(), cfg.fanouts,
                                 synth.rng_seed(cfg, gi), features=True)
        xs = b.features(s)
        xd = b.features(t)[:b[L - 1].n_dst[t]]
        nnz, n_dst = b[L - 1].nnz[r], b[L - 1].n_dst[t]
        out = torch.empty((n_dst, H), dtype=torch.float32, device="cuda")
        ctx.sage_mean_layer(b, L - 1, r, xs, w, x_dst=xd, out=out)   # warm-up
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(torch.cuda.current_stream())
            ctx.sage_mean_layer(b, L - 1, r, xs, w, x_dst=xd, out=out)
            e.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) / 1e3)
        sec = float(np.median(ts))
        if args.trace:
            st = out[:2, :20].contiguous().view(torch.int64).cpu().numpy()
            for cta, row in zip((0, 100), st):
                d = (row - row[0]) / 1e3
                print(json.dumps({"trace_cta": cta, "us": [round(float(x), 2) for x in d]}), file=sys.stderr)
        esz = xs.element_size()
        alg = nnz * F * esz + n_dst * F * esz + n_dst * H * 4 + nnz * 4 + (n_dst + 1) * 4
        flops = 2 * ((n_dst + 127) // 128 * 128) * H * 2 * ((F + 63) // 64 * 64)
        rows.append({"n_dst": n_dst, "nnz": nnz, "us": sec * 1e6, "GBps": alg / sec / 1e9,
                     "TFLOPs": flops / sec / 1e12})
        b.free()
    us = float(np.median([x["us"] for x in rows]))
    gbs = float(np.median([x["GBps"] for x in rows]))
    tf = float(np.median([x["TFLOPs"] for x in rows]))
    print(json.dumps({"bench": "sage_mean_layer", "config": cfg.name, "F": F, "H": H, "dtype_in": str(xs.dtype),
                      "layer": f"input layer (block {L - 1}, relation {cfg.rels[r][0]})",
                      "median_us": round(us, 1), "median_GBps": round(gbs, 1), "hbm_peak_GBps": hbm,
                      "frac_hbm": round(gbs / hbm, 3), "median_TFLOPs": round(tf, 2),
                      "bf16_peak_TFLOPs": bf16_tf, "per_batch": rows}))
    ctx.close()
    del shard


if __name__ == "__main__":
    main()
