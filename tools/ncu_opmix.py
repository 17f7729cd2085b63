"""Instruction mix and stall hot spots per kernel in an ncu report (SASS page).

    python tools/ncu_opmix.py report.ncu-rep [max_kernels]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
limit = int(sys.argv[2]) if len(sys.argv) > 2 else 1
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(row)
for blk in blocks[:limit]:
    hdr, data = blk["rows"][0], blk["rows"][1:]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    ex, st = Counter(), Counter()
    for r in data:
        if len(r) != len(hdr):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ex[op] += int(r[i_ex] or 0)
        st[op] += int(r[i_st] or 0)
    tot = sum(ex.values())
    print(f"{blk['name'][:80]}: total warp-instr {tot}")
    for op, n in ex.most_common(22):
        print(f"  {op:10s} {n:10d} {100 * n / tot:5.1f}%   stall samples {st[op]}")
