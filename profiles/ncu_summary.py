"""Key metrics of an ncu --set full report, one line per kernel launch (for profiles/)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Executed Ipc Active", "Grid Size", "Block Size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ii, ki, mi, ui, vi = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] in KEYS:
            per.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    for n, row in enumerate(rr[2:]):
        d = dict(zip(hh, row))
        key = list(per.keys())[n] if n < len(per) else None
        if key:
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if m in d:
                    per[key][m] = d[m] + " " + rr[1][hh.index(m)]
    for (i, k), m in per.items():
        print(f"[{i}] {k}: " + "; ".join(f"{a}={b}" for a, b in m.items()))


if __name__ == "__main__":
    main(sys.argv[1])
