"""Per-instruction summary of an ncu --import-source capture:
usage: python tools/ncu_src.py REP KERNEL_REGEX [top]
prints the instruction mix (executed warp instructions by opcode) and the SASS lines with the most
warp-stall samples."""
import collections
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for sec in secs[:1]:
    h = sec["rows"][0]
    body = [x for x in sec["rows"][1:] if len(x) == len(h)]
    iS, iW, iI = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    f = lambda v: int(v) if v.strip().isdigit() else 0
    print(sec["name"], "samples", sum(f(x[iW]) for x in body), "warp instrs", sum(f(x[iI]) for x in body))
    ops = collections.Counter()
    for x in body:
        t = x[iS].split()
        if t:
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += f(x[iI])
    print(ops.most_common(25))
    for x in sorted(body, key=lambda x: -f(x[iW]))[:top]:
        print(x[iW], x[iI], x[0][-5:], x[iS][:90])
