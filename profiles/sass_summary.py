"""SASS evidence of the hot kernels (cuobjdump -sass of libegonet.so, sm_100a): per kernel the
instruction count and the counts of the memory / TMA / tensor-core opcodes, plus excerpts of
the lines that prove the claimed hardware paths (UTMALDG / UBLKCP = TMA, UTCHMMA / LDTM =
tcgen05 MMA / TMEM loads, SYNCS = mbarriers, ATOM / RED = the fused bucket counts).

    python profiles/sass_summary.py [paper_2112_15345_b200/libegonet.so] [outdir]
"""
import collections
import os
import re
import subprocess
import sys

HOT = ("k_seed", "k_count", "k_select", "k_copy", "k_tiny", "k_kscan", "k_scatter", "k_compact_count", "k_tscan",
       "k_compact_emit", "gather_tma_kernel", "gather_ldg_kernel", "sage_kernel")
KEEP = re.compile(r"^(LDG|STG|LDS|STS|ST\.|LD\.|ATOM|RED|UTMA|UBLK|UTC|LDTM|SYNCS|SHFL|VOTE|REDUX|BAR|MATCH|IMAD\.HI|IMAD\.WIDE)")
PROOF = re.compile(r"\b(UTMALDG\S*|UTMASTG\S*|UBLKCP\S*|UTCHMMA\S*|UTCBAR\S*|LDTM\S*|SYNCS\.ARRIVE\S*|RED\.E\S*|ATOM\.E\.ADD\S*)")


def main(so, outdir):
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs, cur = collections.OrderedDict(), None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1) if any(h in m.group(1) for h in HOT) else None
            if cur:
                funcs[cur] = []
            continue
        if cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            funcs[cur].append(line.rstrip())
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "sass_summary.txt"), "w") as f, \
            open(os.path.join(outdir, "sass_excerpts.txt"), "w") as g:
        f.write(f"# cuobjdump -sass {so} (sm_100a): opcode counts of the hot kernels (profiles/sass_summary.py)\n\n")
        g.write("# cuobjdump -sass excerpts: the instructions that prove the claimed hardware paths\n")
        for name, lines in funcs.items():
            ops = collections.Counter()
            proof = []
            for l in lines:
                body = l.split("*/", 1)[1].strip() if "*/" in l else l
                body = re.sub(r"^@!?U?P\w+\s+", "", body)
                op = body.split()[0] if body.split() else ""
                if KEEP.match(op):
                    ops[op] += 1
                if PROOF.search(body):
                    proof.append(l.split("/*", 2)[1].split("*/")[0] + "  " + body.split(";")[0])
            top = ", ".join(f"{k} x{v}" for k, v in ops.most_common(14))
            f.write(f"{name}\n   total instructions {len(lines)}; {top}\n")
            if proof:
                g.write(f"\n==== {name}\n")
                for p in proof[:16]:
                    g.write(p + "\n")
    print(f"{len(funcs)} kernels -> {outdir}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2112_15345_b200/libegonet.so",
         sys.argv[2] if len(sys.argv) > 2 else "profiles/r02/sass")
