"""BASELINE.md §5 tables from a results-sweep directory (profiles/r02_final_sweep*.sh)."""
import json
import os
import sys

D = sys.argv[1]


def load(c, t, n, tag=""):
    p = f"{D}/{c}_{t}_n{n}{tag}.json"
    return json.load(open(p)) if os.path.exists(p) else None


def row(d, base, lp=False, label=None):
    r = d["roofline"]
    n = d["n_gpus"]
    mb = d["minibatches_per_s"]
    eff = "1" if n == 1 else ("—" if base is None else f"{mb / n / base:.2f}")
    if r["bound"] == "hbm":
        rl = f"HBM {r['achieved'] / 1e3:.2f} TB/s = {r['frac']:.2f} of 6.56"
    else:
        rl = f"NVLink {r['achieved']:.0f} GB/s = {r['frac']:.2f} of 770"
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    cfg = label or d["config"]["workload"].split(":")[0]
    o = f"{cpu['value'] / 1e6:.2f} M edges/s" if cpu else ""
    if lp:
        return f"| {cfg} | {n} | {mb / 1e3:.1f}k | {d['value'] / 1e9:.2f} G | {eff} | {rl} | {o} |"
    return (f"| {cfg} | {n} | {mb / 1e3:.1f}k | {d['value'] / 1e9:.2f} G | {eff} | {rl} | "
            f"{e2e.get('value', 0) / 1e9:.3f} G/s |" + (f" {o} |" if o or n == 1 else "  |"))


out = ["| config | P | mini-batches/s (agg) | sampled edges/s (agg) | per-GPU efficiency | gather roofline (in the pipelined run) | e2e (host buffers, PCIe) | oracle, 1 core |",
       "|---|---|---|---|---|---|---|---|"]
for c in ["C1", "C2", "C3", "C4", "C5"]:
    b = load(c, "nc", 1)
    base = b["minibatches_per_s"] if b else None
    for n in (1, 2, 4):
        d = load(c, "nc", n)
        if d:
            out.append(row(d, base))
out += ["", "| config (link prediction) | P | LP mini-batches/s | sampled edges/s | per-GPU efficiency | gather roofline | oracle, 1 core |",
        "|---|---|---|---|---|---|---|"]
for c in ["C2", "C4"]:
    base = load(c, "lp", 1)["minibatches_per_s"]
    for n in (1, 2, 4):
        d = load(c, "lp", n)
        if d:
            out.append(row(d, base, lp=True, label=c))
out += ["", "| config (`--replicate fit`) | P | mini-batches/s (agg) | sampled edges/s (agg) | per-GPU efficiency | gather roofline | e2e |",
        "|---|---|---|---|---|---|---|"]
for c, t in [("C2", "nc"), ("C3", "nc"), ("C4", "nc"), ("C4", "lp")]:
    base = load(c, t, 1)["minibatches_per_s"]
    for n in (2, 4):
        d = load(c, t, n, "_fit")
        if d:
            out.append(row(d, base, label=c + (" (LP)" if t == "lp" else "")).rstrip(" |").rstrip() + " |")
print("\n".join(out))
