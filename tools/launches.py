"""Print an ncu --csv launch list (tools for the profiles/ summaries).

    python tools/launches.py gpurun_out/launches.csv
"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
k = OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0][:44])
        try:
            val = float(d["Metric Value"].replace(",", ""))
        except ValueError:  # "n/a" for a metric this kernel does not have
            continue
        k.setdefault(key, {})[d["Metric Name"]] = val
short = {"gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "rd_GB",
         "dram__bytes_write.sum": "wr_GB"}
for (i, name), m in k.items():
    out = []
    for key, v in m.items():
        if key == "gpu__time_duration.sum":
            out.append(f"ms={v / 1e6:.3f}")
        elif key.startswith("dram__bytes"):
            out.append(f"{short[key]}={v / 1e9:.2f}")
        else:
            out.append(f"{key.split('__')[-1]}={v:.3g}")
    print(i, name, " ".join(out))
