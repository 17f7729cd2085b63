"""Per-SASS-instruction shared-memory wavefront excess of one kernel in an ncu report.

    python tools/ncu_source.py report.ncu-rep [kernel-index] [top]
"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')[1:]
rows = list(csv.reader(io.StringIO('"Kernel Name"' + blocks[kidx])))
print(rows[0][1])
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
items = []
tot = totx = 0.0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ex = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
        samp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    tot += wf
    totx += ex
    items.append((ex, wf, samp, r[ix["Address"]][-5:], r[ix["Source"]][:70],
                  r[ix["Instructions Executed"]]))
print(f"shared wavefronts {tot:.4g}, excessive {totx:.4g}")
for it in sorted(items, key=lambda x: -x[0])[:top]:
    if it[0] > 0:
        print(f"  ex={it[0]:.3g} wf={it[1]:.3g} inst={it[5]} {it[3]} {it[4]}")
