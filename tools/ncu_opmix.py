"""Instruction mix and stall hot spots of one kernel in an ncu report (SASS page).

    python tools/ncu_opmix.py report.ncu-rep [kernel-substring]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
args = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    args += ["-k", sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_src, i_ex, i_st = hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter()
for r in data:
    toks = r[i_src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ex[op] += int(r[i_ex] or 0)
    st[op] += int(r[i_st] or 0)
tot = sum(ex.values())
print(f"total warp-instr {tot}")
for op, n in ex.most_common(25):
    print(f"{op:10s} {n:10d} {100 * n / tot:5.1f}%   stall samples {st[op]}")
