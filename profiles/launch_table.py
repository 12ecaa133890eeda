"""Per-kernel table of an ncu launch list (csv of gpu__time_duration / dram bytes / ...):
kernels of the same name are split by their occurrence inside one launch of the batch
graph (e.g. k_compact #0 = level 0 ... #3 = level 3), averaged over the launches seen.

    python profiles/launch_table.py launches.csv [kernels_per_launch_marker=gather]
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (int(r[ii]), r[ki].split("(")[0].replace("void ", "").split("<")[0])
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            v = 0.0
        if r[mi] == "gpu__time_duration.sum":
            v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)
        per.setdefault(key, {})[r[mi]] = v
    return per


def main():
    per = load(sys.argv[1])
    seq = [(k[1], m) for k, m in sorted(per.items()) if k[1].startswith("eg::") and "max_degree" not in k[1]]
    # split into launches: a launch ends with the gather (or starts with k_seed / k_lp_mark)
    launches, cur = [], []
    for n, m in seq:
        if n in ("eg::k_seed", "eg::k_lp_mark") and cur:
            launches.append(cur)
            cur = []
        cur.append((n, m))
    if cur:
        launches.append(cur)
    agg = collections.OrderedDict()
    for L in launches:
        occ = collections.Counter()
        for n, m in L:
            key = f"{n}#{occ[n]}"
            occ[n] += 1
            a = agg.setdefault(key, collections.defaultdict(float))
            a["n"] += 1
            for k, v in m.items():
                a[k] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    print(f"{len(launches)} launches, {tot / max(1, len(launches)):.1f} us per launch (ncu: serialised, cold cache)")
    print(f"{'kernel#occurrence':28s} {'us':>8s} {'share':>6s} {'rd MB':>8s} {'wr MB':>8s} {'occ%':>5s}")
    for k, a in agg.items():
        n = a["n"]
        t = a["gpu__time_duration.sum"] / n
        print(f"{k:28s} {t:8.1f} {a['gpu__time_duration.sum'] / tot:6.3f} {a['dram__bytes_read.sum'] / n / 1e6:8.2f} "
              f"{a['dram__bytes_write.sum'] / n / 1e6:8.2f} {a.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0) / n:5.1f}")


if __name__ == "__main__":
    main()
