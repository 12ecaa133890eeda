"""Summarise an ncu --csv launch list (per-kernel device time and share)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (r[ii], r[ki].split("(")[0].replace("void ", ""))
        v = float(r[vi].replace(",", "")) if r[vi] not in ("", "n/a") else 0.0
        if r[mi] == "gpu__time_duration.sum":
            v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)   # -> us
        per.setdefault(key, {})[r[mi]] = v
    return per


if __name__ == "__main__":
    per = load(sys.argv[1])
    skip = ("sy_", "max_degree")
    seq = [(k[1], m) for k, m in per.items() if not k[1].startswith(skip) and "max_degree" not in k[1]]
    tot = sum(m["gpu__time_duration.sum"] for _, m in seq)
    agg = collections.OrderedDict()
    for n, m in seq:
        agg.setdefault(n, []).append(m)
    print(f"{len(seq)} launches of egonet kernels, {tot:.1f} us total (ncu: serialised, cold cache)")
    print(f"{'kernel':28s} {'n':>4s} {'mean us':>9s} {'share':>6s} {'dram MB/launch':>14s}")
    for n, ms in sorted(agg.items(), key=lambda kv: -sum(x["gpu__time_duration.sum"] for x in kv[1])):
        t = sum(x["gpu__time_duration.sum"] for x in ms)
        dr = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ms) / len(ms)
        print(f"{n:28s} {len(ms):4d} {t / len(ms):9.2f} {t / tot:6.3f} {dr / 1e6:14.2f}")
