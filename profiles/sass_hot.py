"""Hot SASS lines / opcode mix of one kernel in an ncu --set full report (source page).

    python profiles/sass_hot.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    ia, isrc = h.index("Address"), h.index("Source")
    iex, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ith = h.index("Thread Instructions Executed")
    f = lambda r, i: float(r[i] or 0)
    tex = sum(f(r, iex) for r in data)
    tst = sum(f(r, ist) for r in data)
    tth = sum(f(r, ith) for r in data)
    print(f"warp instr {tex:.0f}, thread instr {tth:.0f} (avg {tth / max(1, tex):.1f} lanes), stall samples {tst:.0f}")
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    sc = collections.Counter()
    for r in data:
        for c in stall_cols:
            sc[c] += f(r, h.index(c))
    print("stalls:", ", ".join(f"{c[6:]} {v / max(1, sum(sc.values())):.2f}" for c, v in sc.most_common(8)))
    print("top by stall samples:")
    for r in sorted(data, key=lambda r: -f(r, ist))[:top]:
        print(f"  {f(r, ist) / tst:6.3f} ex {f(r, iex) / tex:6.3f}  {r[isrc][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
