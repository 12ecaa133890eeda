"""One summary row of a bench.py JSON line (profiles/r02_final_sweep.sh)."""
import json
import sys

d = json.load(open(sys.argv[1]))
r = d["roofline"]
cfg = d["config"]["workload"].split(":")[0]
task = d["config"].get("task", "nc")
e2e = d.get("e2e") or {}
cpu = d.get("cpu_baseline") or {}
print(f"{cfg:4s} {task} N={d['n_gpus']}  {d['minibatches_per_s']:9.0f} mb/s  {d['value'] / 1e9:6.2f} G edges/s  "
      f"{r['bound']} {r['achieved']:7.0f} {r['unit']} = {r['frac']:.2f} of {r['peak']:.0f}  "
      f"e2e {e2e.get('value', 0) / 1e9:6.3f} G/s  parity {d.get('parity_checked')}  "
      f"oracle {cpu.get('value', 0) / 1e6:.2f} M/s")
