#!/usr/bin/env python
"""Benchmark of the mini-batch ego-network generator (seeds -> blocks + features).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload (N=1 default): C4, the ogbn-papers100M-shaped graph (111M vertices, 1.6B
edges, 128-d fp16) -- the largest BASELINE config that fits one B200 (C5 needs two).

A step = one launch of the whole hot path over a bundle of `--bundle` (32)
mini-batches per rank: sample every hop (sampling + compaction kernels) and gather
the input vertices' feature rows, as one CUDA graph; `--depth` (6) launches are in
flight per GPU.  So `--steps 20` times 640 mini-batches per rank, and every timed
launch carries a full bundle (steady state: the warm-up captures every lane's graph).
Inputs (graph shard, feature shard, the seeds of every step) are resident in HBM
before the timed region.  Each rank samples its own batches (global batch
g = b * N + rank); the graph and features are range-sharded over the N GPUs and
peer shards are read over NVLink.  Timing: W untimed warm-up steps, then K steps
bracketed by barrier + synchronize, CUDA events on the context's stream, max over
ranks.  Rank 0 prints one JSON line.

The oracle leg (rank 0 at N=1, skipped with --no-cpu-baseline) re-runs the first
timed mini-batches through the same bundled launch after the timed region and
compares them element by element with oracle/ (parity_checked), then times the
oracle on a bounded sample (cpu_baseline).

--impl reference times the CPU oracle (oracle/, plain single-threaded C) on the
host, on the same workload and metric (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = ("sampled edges/sec + mini-batches/sec (seeds→blocks+features) at 1/2/4/8 B200; gather GB/s")
UNIT = "sampled edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32, help="timed launches (each: --bundle mini-batches per rank)")
    ap.add_argument("--warmup", type=int, default=8, help="untimed launches before the timed region")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--task", default="nc", choices=["nc", "lp"],
                    help="nc: node-classification batches (seed vertices, the headline); lp: link-prediction "
                         "batches (NEXT-3: cfg.batch positive edges + 1 negative each, fanout [25, 15])")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--confine", action="store_true",
                    help="seed confinement (NEXT-2, P:428-431): each rank draws its seeds from the train ids "
                         "of its own vertex range (use with the planted-community configs C2L / C4L)")
    ap.add_argument("--features", default="device", choices=["device", "host"],
                    help="feature rows in HBM (default) or in pinned host memory read zero-copy over PCIe "
                         "(NEXT-4 ii: the paper's placement, lets C5 run on one GPU)")
    ap.add_argument("--replicate", default="auto",
                    help="replicated feature partition policy (P:468-473) for small vertex types: auto (N > 1: "
                         "every type whose full table is <= 64 MiB gets a local copy on each GPU), none, or a "
                         "comma list of type indices, or fit (N > 1: whole tables, smallest first, up to 45 GiB per GPU; "
                         "the features of C2-C4 are then local on every GPU, DESIGN §7)")
    ap.add_argument("--depth", type=int, default=None,
                    help="launches in flight per GPU (pipeline lanes); default 6 (C5 and --task lp: 4)")
    ap.add_argument("--bundle", type=int, default=None,
                    help="mini-batches per launch (bundled kernels); default 32")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--diag-no-gather", action="store_true",
                    help="DIAGNOSTIC ONLY (not a bench line): sampling + compaction without the gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded oracle sample (cpu_baseline)")
    ap.add_argument("--parity", type=int, default=None,
                    help="timed mini-batches re-run and compared with the oracle after the timed region "
                         "(default 8 for C4/C5, 16 otherwise; 0 = none)")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    a = ap.parse_args()
    # pipeline shape: 4 lanes x bundles of 32 (round-2 sweep, profiles/r02/bundle32/,
    # bundle64/: 4 x 32 is +5-10 % over 4 x 16, 4 x 64 another +2 %)
    if a.depth is None:   # 6 lanes hide the peer (NVLink) latency at N > 1: C4 +5 % at N = 2, +2 % at N = 4,
        # ~+1 % at N = 1 (profiles/r02/depth/, knobs/).  C5 and link-prediction batches keep 4: their
        # worst-case slot sizes (C2 LP: fanout [25, 15] over 3 seeds per positive) exhaust HBM at 6 x 32
        a.depth = 4 if (a.config == "C5" or a.task == "lp") else 6
    if a.bundle is None:   # C5: 4 x 32 batches of feature outputs (~84 GB) + a 98 GB shard at N = 2 exceed HBM
        a.bundle = 16 if a.config == "C5" else 32
    if a.replicate not in ("auto", "none", "fit"):
        a.replicate = [int(x) for x in a.replicate.split(",") if x != ""]
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


LP_NEG = 1   # negatives per positive edge in --task lp
LP_NEG_KEY = 0x4E4547   # neg_seed(g) = rng_seed(g) ^ LP_NEG_KEY


def task_fanouts(cfg, task):
    import synth
    return synth.lp_fanouts(cfg) if task == "lp" else cfg.fanouts


def workload(cfg, world, task="nc"):
    import synth
    if task == "lp":
        rel = synth.lp_rel(cfg)
        return {"workload": f"{cfg.name} link prediction: {cfg.batch} positive edges of relation "
                            f"{cfg.rels[rel][0]} + {LP_NEG} uniform negative each (seeds = distinct endpoints), "
                            f"fanout [25, 15] (P:970-971); graph: {cfg.description}",
                "task": "lp", "positives_per_rank": cfg.batch, "negatives_per_positive": LP_NEG,
                "fanouts": synth.lp_fanouts(cfg), "n_vertices": int(cfg.vt_counts.sum()),
                "n_edges": int(sum(r[3] for r in cfg.rels)), "ranks": world,
                "partition": "per-type vertex range, floor(p*N_t/P)",
                "l2": "inputs larger than L2 (feature store %.2f GB, random rows)" % (
                    sum(cfg.row_bytes(u) * int(cfg.vt_counts[u]) for u in cfg.feats) / 1e9)}
    return {"workload": f"{cfg.name}: {cfg.description}", "batch_per_rank": cfg.batch, "fanouts": cfg.fanouts,
            "n_vertices": int(cfg.vt_counts.sum()), "n_edges": int(sum(r[3] for r in cfg.rels)),
            "ranks": world, "partition": "per-type vertex range, floor(p*N_t/P)",
            "l2": "inputs larger than L2 (feature store %.2f GB, random rows)" % (
                sum(cfg.row_bytes(u) * int(cfg.vt_counts[u]) for u in cfg.feats) / 1e9)}


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region.

    NVML polled every millisecond from a thread (the timed region of a default run is
    tens of ms, too short for nvidia-smi's loop); nvidia-smi -lms 50 when NVML is
    unavailable."""
    POLL_S = 0.001
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index, pci_bus_id=None):
        self.index = index
        self.pci = pci_bus_id
        self.proc = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, reasons bitmask)
        self.stop_ev = threading.Event()
        self.nvml = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (nv, h)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        try:
                            rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                        except Exception:
                            rs = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    time.sleep(self.POLL_S)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_ev.set()
            self.t.join(timeout=1)
            if not self.samples:
                return None
            reasons = sorted({n for _, rs in self.samples for n, b in self.BITS.items() if rs & b})
            return {"sm_mhz": statistics.median(sm for sm, _ in self.samples), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(self.samples), "source": "NVML, 1 ms polling"}
        if not self.proc:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi -lms 50"}


# ----------------------------------------------------------------------------- oracle timing

def time_oracle(cfg, graph, host_rows, batches, budget_s, min_batches=1, task="nc"):
    """The oracle as it stands (single-threaded C), sample + gather per batch.

    host_rows None (C4 / C5: the feature store does not fit the host): the rows of the
    batch's input vertices are generated first, outside the timed region, into a
    compact array, and the oracle gathers from that (same bytes copied per row)."""
    import numpy as np

    import oracle
    import synth
    n_edges = 0
    n = 0
    gathered = 0
    spent = 0.0
    for g in batches:
        if task == "lp":
            rel = synth.lp_rel(cfg)
            src, dst = synth.lp_positives(cfg, graph, rel, g)
            t0 = time.perf_counter()
            res, _ = oracle.sample_lp(graph, src, dst, rel, LP_NEG, synth.rng_seed(cfg, g) ^ LP_NEG_KEY,
                                      synth.lp_fanouts(cfg), synth.rng_seed(cfg, g))
            spent += time.perf_counter() - t0
        else:
            seeds = synth.batch_seeds(cfg, g)
            t0 = time.perf_counter()
            res = oracle.sample(graph, seeds, cfg.fanouts, synth.rng_seed(cfg, g))
            spent += time.perf_counter() - t0
        n_edges += sum(len(b.eids) for hop in res.blocks for b in hop)
        for u in cfg.feats:
            if host_rows is not None:
                t0 = time.perf_counter()
                gathered += oracle.gather(res, cfg.vt_counts, u, host_rows[u]).nbytes
                spent += time.perf_counter() - t0
            else:
                ids = res.input_nodes(u)
                off_u = int(cfg.offsets[u])
                rows = synth.host_features_ids(cfg, u, ids - off_u)           # untimed: input data
                local = off_u + np.arange(len(ids), dtype=np.int64)
                t0 = time.perf_counter()
                gathered += oracle.gather_ids(local, cfg.vt_counts, u, rows).nbytes
                spent += time.perf_counter() - t0
        n += 1
        if n >= min_batches and spent > budget_s:
            break
    return {"batches": n, "seconds": spent, "edges": n_edges, "bytes": gathered}


def run_reference(args, cfg, rank, world):
    """The reference arm (this tier: the oracle as it stands, on the host cores): the
    same workload, metric and step as our arm -- a step = the `--bundle` mini-batches one
    launch of ours carries (rank 0's batches g = b*N), sampled, compacted and gathered by
    the single-threaded C oracle."""
    if rank != 0:
        return
    import synth
    B = args.bundle
    graph = synth.build_host_graph(cfg, materialize_indices=True)
    rows = {u: synth.host_features(cfg, u) for u in cfg.feats} if cfg.name in ("C1", "C2", "C3") else None
    for b in range(args.warmup):
        time_oracle(cfg, graph, rows, [(b * B + i) * world for i in range(B)], float("inf"), task=args.task)
    per_step = []
    edges = 0
    nbytes = 0
    for b in range(args.warmup, args.warmup + args.steps):
        r = time_oracle(cfg, graph, rows, [(b * B + i) * world for i in range(B)], float("inf"), task=args.task)
        per_step.append(r["seconds"])
        edges += r["edges"]
        nbytes += r["bytes"]
    total = sum(per_step)
    value = edges / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32/bytes",
            "data": "synthetic", "config": dict(workload(cfg, world, args.task),
                                               step_unit=f"a bundle of {B} mini-batches (rank 0's)"),
            "minibatches_per_s": args.steps * B / total, "gather_GBps": nbytes / total / 1e9,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} steps x {B} full {cfg.name} batches (sample+compact+gather), "
                                       f"single-threaded C oracle on {cpu_model()}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(args, line)


def emit(args, line):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


# ----------------------------------------------------------------------------- our path

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# Version tag of the gather kernel the committed ncu traffic figures were captured on
# (profiles/gather_traffic.json entries carry it; a changed kernel invalidates them).
TRAFFIC_CODE = "r02"


def load_traffic(cfg_name, kernel, bundle):
    """ncu DRAM bytes (per mini-batch) and duration (per launch) of `kernel` on this
    config at this bundle size (profiles/gather_traffic.json, from one --set full capture)."""
    p = os.path.join(ROOT, "profiles", "gather_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("%s@b%d" % (kernel, bundle))
    except Exception:
        return None


def parity_check(cfg, graph, task, batches, outs, seeds_host, rngs, negs, rel):
    """Oracle leg: the CUDA path's outputs of `batches` (host copies taken from the same
    bundled launch configuration the bench times) vs oracle/, element by element:
    every node list, block CSC (indptr, relabelled src ids, eids) and gathered feature
    byte.  Raises on the first difference; returns the number of batches compared."""
    import oracle
    import synth
    rows_full = cfg.name in ("C1", "C2", "C3")
    for g, out in zip(batches, outs):
        if task == "lp":
            src, dst = seeds_host[g]
            res, _ = oracle.sample_lp(graph, src, dst, rel, LP_NEG, negs[g], synth.lp_fanouts(cfg), rngs[g])
        else:
            res = oracle.sample(graph, seeds_host[g], cfg.fanouts, rngs[g])
        for l, lv in enumerate(out["levels"]):
            for u in range(cfg.n_vt):
                if not np.array_equal(lv[u], res.levels[l][u]):
                    raise AssertionError(f"parity: batch {g} level {l} type {u} differs")
        for h, hop in enumerate(out["blocks"]):
            for r in range(cfg.n_rel):
                o = res.blocks[h][r]
                for key, want in (("indptr", o.indptr), ("indices", o.indices), ("eids", o.eids)):
                    if not np.array_equal(hop[r][key], want):
                        raise AssertionError(f"parity: batch {g} hop {h} relation {r} {key} differs")
        for u in cfg.feats:
            ids = res.input_nodes(u)
            if rows_full:
                want = oracle.gather(res, cfg.vt_counts, u, synth.host_features(cfg, u))
            else:   # the store does not fit host RAM: the rows of this batch's inputs only
                off_u = int(cfg.offsets[u])
                rows = synth.host_features_ids(cfg, u, ids - off_u)
                want = oracle.gather_ids(off_u + np.arange(len(ids), dtype=np.int64), cfg.vt_counts, u, rows)
            if out["feats"][u].tobytes() != want.tobytes():
                raise AssertionError(f"parity: batch {g} feature bytes of type {u} differ")
    return len(outs)


def host_copy(bl, cfg):
    """A batch's outputs as numpy (levels, per-hop CSCs, feature bytes)."""
    levels = [[bl[0].dst_nodes[u].cpu().numpy() for u in range(cfg.n_vt)]]
    blocks = []
    for h in range(bl.n_hops):
        b = bl[h]
        levels.append([b.src_nodes[u].cpu().numpy() for u in range(cfg.n_vt)])
        blocks.append([{"indptr": b.indptr[r].cpu().numpy(), "indices": b.indices[r].cpu().numpy(),
                        "eids": b.eids[r].cpu().numpy()} for r in range(cfg.n_rel)])
    feats = {u: bl.features(u).cpu().numpy() for u in cfg.feats}
    return {"levels": levels, "blocks": blocks, "feats": feats}


def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import synth
    from synth.device import load_context
    from paper_2112_15345_b200 import Context

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    B = args.bundle
    W, K = args.warmup, args.steps            # launches (steps); each carries B mini-batches per rank
    n_b = (W + K) * B                          # mini-batches per rank
    oracle_leg = rank == 0 and world == 1 and not args.no_cpu_baseline
    # host src ids: for the oracle leg (C4: 6.5 GB) and small configs; C5 generates on the device
    graph = synth.build_host_graph(cfg, materialize_indices=cfg.name in ("C1", "C2", "C3") or oracle_leg)
    t_load = time.perf_counter()
    ctx = Context(rank, world, local_rank, stream)
    shard = load_context(ctx, graph, world, rank, dev, features=args.features if args.features != "device" else True,
                         replicate=args.replicate if args.features == "device" else "none")
    replicas = sorted(shard["replicas"])
    if world > 1:
        ctx.connect_peers()
    ctx.set_pipeline(args.depth, B)
    t_load = time.perf_counter() - t_load
    rngs = [synth.rng_seed(cfg, b * world + rank) for b in range(n_b)]
    fanouts = np.array(task_fanouts(cfg, args.task), np.int32)
    lp = args.task == "lp"
    rel, negs = None, None
    if lp:   # link prediction: positives (src, dst) per batch; inputs[b] = (src, dst)
        rel = synth.lp_rel(cfg)
        seeds_host = [synth.lp_positives(cfg, graph, rel, b * world + rank) for b in range(n_b)]
        seeds_dev = [(torch.from_numpy(a).to(dev), torch.from_numpy(c).to(dev)) for a, c in seeds_host]
        negs = [r ^ LP_NEG_KEY for r in rngs]
    else:
        if args.confine:
            seeds_host = [synth.batch_seeds_confined(cfg, b, rank, world) for b in range(n_b)]
        else:
            seeds_host = [synth.batch_seeds(cfg, b * world + rank) for b in range(n_b)]
        seeds_dev = [torch.from_numpy(s).to(dev) for s in seeds_host]
    row_bytes = [cfg.row_bytes(u) for u in range(cfg.n_vt)]
    torch.cuda.synchronize(dev)

    def launch(b0, b1, seeds, features=True):
        # one CUDA-graph launch for batches b0..b1-1: sample + compact all hops + gather
        # features; no host sync
        if lp:
            return ctx.sample_lp_bundle([seeds[b][0] for b in range(b0, b1)], [seeds[b][1] for b in range(b0, b1)],
                                        rel, LP_NEG, negs[b0:b1], fanouts, rngs[b0:b1], features=features,
                                        async_=True)
        if b1 - b0 == 1 and B == 1:
            return [ctx.sample_minibatch(seeds[b0], fanouts, rngs[b0], features=features, async_=True)]  # noqa
        return ctx.sample_bundle([seeds[b] for b in range(b0, b1)], fanouts, rngs[b0:b1], features=features,
                                 async_=True)

    def retire(bl):
        return bl.stats()      # waits for the batch; one call

    from collections import deque

    host_t = {"launch": 0.0, "retire": 0.0}

    def run(lo, hi, seeds, on_retire):
        """Launches lo..hi-1 (launch l = batches l*B .. l*B+B-1), `depth` in flight."""
        q = deque()
        for l in range(lo, hi):
            t0 = time.perf_counter()
            q.append(launch(l * B, (l + 1) * B, seeds, features=not args.diag_no_gather))
            host_t["launch"] += time.perf_counter() - t0
            if len(q) >= args.depth:
                for bl in q.popleft():
                    t0 = time.perf_counter()
                    on_retire(bl)
                    bl.free()
                    host_t["retire"] += time.perf_counter() - t0
        while q:
            for bl in q.popleft():
                on_retire(bl)
                bl.free()

    acc = {"edges": 0, "gbytes": 0, "rbytes": 0, "inputs": 0}

    def count(bl):
        e, rows = retire(bl)
        acc["edges"] += e
        acc["inputs"] += sum(rows)
        acc["gbytes"] += sum(rows[u] * (2 * row_bytes[u] + 8) for u in cfg.feats)
        acc["rbytes"] += sum(rows[u] * row_bytes[u] for u in cfg.feats)

    pci = None
    try:
        pr = torch.cuda.get_device_properties(dev)
        pci = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
    except Exception:
        pass
    with torch.cuda.stream(stream):
        run(0, W, seeds_dev, retire)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        ctx.profile()                                   # drain
        ctx.set_profiling(True)
        clocks = ClockSampler(local_rank, pci)
        clocks.start()
        launches0 = ctx.kernel_launches()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        ev0.record(stream)
        host_t["launch"] = host_t["retire"] = 0.0
        run(W, W + K, seeds_dev, count)
        host_us = {k: 1e6 * v / (K * B) for k, v in host_t.items()}
        edges, gbytes = acc["edges"], acc["gbytes"]
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        ms = ev0.elapsed_time(ev1)
        launches = ctx.kernel_launches() - launches0
        clk = clocks.stop()
        ctx.set_profiling(False)
        prof = ctx.profile()
        trace = {k: round(1e3 * ms / max(1, n), 2) for k, (ms, n) in ctx.trace().items()}

    totals = torch.tensor([ms, float(edges), float(gbytes), float(K)], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        mx = totals.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(totals[1:], op=dist.ReduceOp.SUM)
        ms = float(mx[0])
        edges = float(totals[1])
    value = edges / (ms / 1e3)
    n_timed = world * K * B                           # mini-batches, all ranks

    # e2e: host seeds in (pinned), features out to pinned host memory, through the C ABI
    e2e = None
    if not args.no_e2e:
        if lp:
            pinned_seeds = [(torch.from_numpy(a).pin_memory(), torch.from_numpy(c).pin_memory()) for a, c in seeds_host]
        else:
            pinned_seeds = [torch.from_numpy(s).pin_memory() for s in seeds_host]
        caps_nodes, _ = __import__("paper_2112_15345_b200").batch_caps(
            cfg.vt_counts, [r[1] for r in cfg.rels], [r[2] for r in cfg.rels], [r[3] for r in cfg.rels],
            [cfg.dmax(r) for r in range(cfg.n_rel)], cfg.batch * (2 + LP_NEG) if lp else cfg.batch, fanouts)
        host_outs = [None] * cfg.n_vt
        for u in cfg.feats:
            dim, dt = cfg.feats[u]
            host_outs[u] = torch.empty((int(caps_nodes[u]), dim),
                                       dtype=torch.float32 if dt == 0 else torch.float16).pin_memory()

        def e2e_retire(bl):
            e, rows = retire(bl)
            # the batch's gathered rows to pinned host memory through the C ABI (D2H on the
            # context's stream; the timed region ends with a synchronize)
            bl.copy_features([host_outs[u] if u in cfg.feats else None for u in range(cfg.n_vt)], async_=True)
            nbytes = sum(rows[u] * row_bytes[u] for u in cfg.feats)
            return e, nbytes

        e2e_acc = {"edges": 0, "h2d": 0, "d2h": 0}
        counter_b = __import__("paper_2112_15345_b200").counter_bytes()

        def e2e_count(bl):
            e, nb = e2e_retire(bl)
            e2e_acc["edges"] += e
            e2e_acc["h2d"] += cfg.batch * (16 if lp else 8)
            e2e_acc["d2h"] += nb + counter_b   # + the per-batch counters read back (eg_counter_bytes)

        with torch.cuda.stream(stream):
            run(0, min(W, 2), pinned_seeds, e2e_retire)
            torch.cuda.synchronize(dev)
            if world > 1:
                torch.distributed.barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            run(W, W + K, pinned_seeds, e2e_count)
            t1.record(stream)
            torch.cuda.synchronize(dev)
            ems = t0.elapsed_time(t1)
        e_edges, h2d, d2h = e2e_acc["edges"], e2e_acc["h2d"], e2e_acc["d2h"]
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ems, float(e_edges)], dtype=torch.float64, device=dev)
            m = t.clone()
            dist.all_reduce(m[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
            ems, e_edges = float(m[0]), float(t[1])
        e2e = {"value": e_edges / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d // K,
               "d2h_bytes_per_step": d2h // K,
               # the bound: one GPU's PCIe link (D2H of the gathered rows, ~55-57 GB/s on Gen5 x16)
               "d2h_GBps_per_gpu": (d2h / K) / (ems / K / 1e3) / 1e9 if ems > 0 else None,
               "note": "per step (one launch of %d mini-batches): seeds from pinned host memory in (read in place "
                       "by the seed split over PCIe), gathered feature rows out to pinned host memory (D2H), "
                       "per-batch counters read back; blocks stay device-resident" % B}

    # roofline of the gather kernel (events inside the library's graph, on its stream,
    # timed region).  P = 1: HBM-bound (read row + write row + read id).  P > 1: rows owned
    # by peers cross NVLink; the remote share is measured on one extra batch.
    peak, peak_src = load_peaks()
    gather_ms = prof["gather_ms"] / max(1, prof["n_gather"])      # gather kernel node
    sample_ms = prof["sample_ms"] / max(1, prof["n_sample"])      # sampling + compaction nodes
    n_launch = max(1, prof["n_gather"])                             # one gather launch per step
    achieved = (gbytes / n_launch) / (gather_ms / 1e3) / 1e9 if gather_ms > 0 else 0.0
    gk = {"tma": "gather_tma_kernel", "ldg": "gather_ldg_kernel"}.get(ctx.gather_path(), "none")
    tr = load_traffic(cfg.name, gk, B)
    if tr and not (args.task == "nc" and world == 1 and B == tr.get("bundle") and args.features == "device"
                   and tr.get("code") == TRAFFIC_CODE):
        tr = None   # the ncu capture must be of this kernel, bundle size, task and code version
    alg_per_batch = gbytes / max(1, K * B)
    roofline = {"kernel": gk, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "traffic": (tr["dram_bytes_per_batch"] * B) if tr else None,
                "algorithmic_bytes_per_launch": gbytes / n_launch,
                "per_unit": "2*row_bytes + 8 B per input row (read row, write row, read id); one launch gathers "
                            "the rows of a bundle of %d mini-batches" % B,
                "gather_ms_per_launch": gather_ms, "sample_chain_ms_per_launch": sample_ms,
                "launches_timed": n_launch}
    if tr:
        # the same kernel in one ncu --set full capture (serialised, one launch of B batches):
        # its DRAM bytes (traffic, per batch x B) and its duration alone
        a1 = alg_per_batch * B / (tr["ncu_duration_us_per_launch"] / 1e6) / 1e9
        roofline["traffic_source"] = tr.get("source")
        roofline["traffic_over_algorithmic"] = tr["dram_bytes_per_batch"] / alg_per_batch
        roofline["alone_ncu"] = {"achieved": a1, "frac": a1 / peak, "duration_us": tr["ncu_duration_us_per_launch"]}
    frac_remote = None
    if world > 1:
        with torch.cuda.stream(stream):
            bl = launch(0, 1, seeds_dev, features=False)[0]
            bl.wait()
            remote = 0
            rows_tot = 0
            bounds = shard["bounds"]
            for u in cfg.feats:
                ids = bl[bl.n_hops - 1].src_nodes[u] - int(cfg.offsets[u])
                lo, hi = int(bounds[u][rank]), int(bounds[u][rank + 1])
                n_remote = 0 if u in replicas else int(((ids < lo) | (ids >= hi)).sum().item())
                remote += n_remote * row_bytes[u]
                rows_tot += ids.numel() * row_bytes[u]
            bl.free()
        frac_remote = remote / max(1, rows_tot)
    if frac_remote:   # some rows cross NVLink: that is the bound (else all rows are local: HBM)
        nv_bytes = (gbytes / n_launch) / 2 * frac_remote   # row bytes read over NVLink per launch
        nv_peak = 770.0
        nv_achieved = nv_bytes / (gather_ms / 1e3) / 1e9 if gather_ms > 0 else 0.0
        roofline.update({"kernel": gk, "bound": "nvlink", "achieved": nv_achieved, "peak": nv_peak,
                         "frac": nv_achieved / nv_peak,
                         "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction per GPU",
                         "per_unit": "row_bytes per input row owned by a peer (read over NVLink)",
                         "algorithmic_bytes_per_launch": nv_bytes, "remote_row_fraction": frac_remote,
                         # both directions are busy (every GPU reads from and serves its peers):
                         # profiles/micro/p2p_rw.cu measured 645 GB/s per GPU for random 512-B rows
                         "peak_bidirectional_measured": 645.0, "frac_bidirectional": nv_achieved / 645.0,
                         "hbm_view": {"achieved": achieved, "peak": peak, "frac": achieved / peak}})

    if args.features != "device":
        # rows read zero-copy over PCIe: bound = the measured pinned host -> device copy bandwidth
        src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        best = 0.0
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            with torch.cuda.stream(stream):
                dst.copy_(src, non_blocking=True)
            b.record(stream)
            torch.cuda.synchronize(dev)
            best = max(best, (1 << 30) / (a.elapsed_time(b) / 1e3) / 1e9)
        del src, dst
        pc_bytes = acc["rbytes"] / n_launch
        pc_achieved = pc_bytes / (gather_ms / 1e3) / 1e9 if gather_ms > 0 else 0.0
        roofline.update({"kernel": gk, "bound": "pcie", "achieved": pc_achieved, "peak": best,
                         "frac": pc_achieved / best if best else None,
                         "peak_source": "measured here: pinned host -> device copy of 1 GiB (best of 5, CUDA events)",
                         "per_unit": "row_bytes per input row read zero-copy from pinned host memory",
                         "algorithmic_bytes_per_launch": pc_bytes, "traffic": None,
                         "hbm_view": {"achieved": achieved, "peak": peak, "frac": achieved / peak}})

    cpu = None
    parity = None
    if oracle_leg:
        # parity: the first timed mini-batches again, through the same bundled launch
        npar = min(B, args.parity if args.parity is not None else B)
        if npar > 0:
            g0 = W * B
            with torch.cuda.stream(stream):
                bls = launch(g0, g0 + npar, seeds_dev)
                outs = [host_copy(bl, cfg) for bl in bls]
                for bl in bls:
                    bl.free()
            parity = parity_check(cfg, graph, args.task, range(g0, g0 + npar), outs, seeds_host, rngs, negs, rel)
        full = cfg.name in ("C1", "C2", "C3")
        rows_h = {u: synth.host_features(cfg, u) for u in cfg.feats} if full else None
        r = time_oracle(cfg, graph, rows_h, range(100000, 200000), args.cpu_seconds, task=args.task)
        cpu = {"value": r["edges"] / r["seconds"], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{r['batches']} full {cfg.name} batches (sample+compact+gather) in "
                         f"{r['seconds']:.1f} s, single-threaded C oracle on {cpu_model()} "
                         f"({host_cores()} cores available)"
                         + ("" if full else "; feature rows of each batch generated untimed into a compact "
                                            "host array first (the store does not fit host RAM)")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "int32 ids / raw feature bytes (%s)" % ",".join(
                    sorted({"fp32" if cfg.feats[u][1] == 0 else "fp16" for u in cfg.feats})),
                "data": "synthetic (seeded generator, synth/)", "config": dict(workload(cfg, world, args.task), seeds=(
                    "confined to the rank's vertex range (second-level partition, P:428-431)" if args.confine
                    else "global epoch permutation, batch g = b*P + p"), features_in=(
                    "pinned host memory (zero-copy over PCIe)" if args.features == "host" else "HBM"),
                    feature_replicas=[cfg.vtypes[u][0] for u in replicas],
                    step_unit=f"one launch (CUDA graph) of a bundle of {B} mini-batches per rank; {args.depth} "
                              f"launches in flight per GPU"),
                "minibatches_per_s": n_timed / (ms / 1e3),
                "gather_GBps": achieved if gather_ms > 0 else None,
                "sampled_edges_per_batch": edges / n_timed,
                "input_vertices_per_batch_rank0": acc["inputs"] / (K * B),
                "parity_checked": parity,
                "parity_note": ("the first %d timed mini-batches of rank 0, re-run through the same bundled launch "
                                "after the timed region, equal the oracle's element by element (node lists, block "
                                "CSCs, eids, feature bytes)" % parity) if parity else None,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                # lanes co-running (nsys is not in the image): the device time of one launch
                # (its sampling + compaction nodes and its gather node, CUDA events recorded
                # inside the launch's graph) against the step period
                "overlap": {"launch_device_ms": sample_ms + gather_ms, "ms_per_step": ms / K,
                            "launches_in_flight_avg": (sample_ms + gather_ms) / (ms / K) if ms > 0 else None,
                            "gather_busy_frac": gather_ms / (ms / K) if ms > 0 else None,
                            "source": "CUDA events inside each launch's graph (rank 0)"},
                "clocks": clk, "load_seconds": t_load, "stage_us": trace or None,
                "pipeline_depth": args.depth, "bundle": B, "host_us_per_batch": host_us,
                "host": {"cores": host_cores(), "cpu": cpu_model()}}
        emit(args, line)
    ctx.close()
    del shard
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if world != args.gpus:
        world = args.gpus if world == 1 and args.gpus == 1 else world
    import synth
    cfg = synth.config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
