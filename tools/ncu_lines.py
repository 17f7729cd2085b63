"""Dynamic instruction counts and stall samples per SOURCE LINE of one kernel in an
ncu report captured with --import-source on (the SASS rows of the source page,
summed per file:line, with the top opcodes of each line). This is the view that
located the DST engine's and the 27-point kernels' address-generation overhead
(DESIGN.md 3.1, 3.3). Instructions inlined through several source levels are
listed under each level, so the total exceeds the kernel's instruction count:
read the percentages.

    python tools/ncu_lines.py report.ncu-rep "kernel name substring" [top] [instance]
"""
import csv, io, subprocess, sys
from collections import Counter, defaultdict
path, kname, top = sys.argv[1], sys.argv[2], int(sys.argv[3]); inst = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass,cuda"],capture_output=True,text=True).stdout
blocks=[];cur=None;fp=None
for row in csv.reader(io.StringIO(out)):
    if row and row[0]=="File Path": fp=row[1].split("/")[-1]; continue
    if row and row[0]=="Function Name":
        cur={"name":row[1],"file":fp,"rows":[]};blocks.append(cur)
    elif cur is not None: cur["rows"].append(row)
seen=Counter()
per=defaultdict(Counter); tot=Counter(); stall=Counter(); src={}
for blk in blocks:
    if kname not in blk["name"]: continue
    key=(blk["name"],blk["file"])
    seen[key]+=1
    if seen[key]-1 != inst: continue

    hdr=blk["rows"][0]
    iex=hdr.index("Instructions Executed"); ist=hdr.index("Warp Stall Sampling (All Samples)")
    line=None
    for r in blk["rows"][1:]:
        if len(r)<len(hdr): continue
        if r[0]!="":
            line=(blk["file"],int(r[0])); src[line]=r[1]; continue
        op=r[3].split()
        if not op or r[iex] in ("-",""): continue
        full=op[1] if op[0].startswith("@") else op[0]
        o=full.split(".")[0]
        if full.startswith("IMAD.MOV") or full=="MOV": o="MOV*"
        n=int(r[iex]); per[line][o]+=n; tot[line]+=n; stall[line]+=int(r[ist])
T=sum(tot.values()); S=sum(stall.values())
print("total",T,"stall samples",S)
for l,n in tot.most_common(top):
    print(f"{l[0][:10]:10s}{l[1]:5d} {n/T*100:5.1f}% st {stall[l]/S*100:4.1f}%  {src[l].strip()[:60]:60s} ", dict(per[l].most_common(6)))
