"""Write profiles/traffic.json from an ncu launch list of one one-call solve
(dram__bytes_read.sum + dram__bytes_write.sum per launch, in launch order).

    python tools/traffic_json.py gpurun_out/launches.csv --cfg 4 [--lean]
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--lean", action="store_true")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = None
per = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"].startswith("dram__bytes"):
            i = int(d["ID"])
            per[i] = per.get(i, 0) + float(d["Metric Value"].replace(",", ""))
names = bench.STAGES_LEAN if a.lean else bench.STAGES_FAST
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "traffic.json")
tab = json.load(open(out_path)) if os.path.exists(out_path) else {}
# the LAST complete solve of the list: the steady state (the first solve after a
# coefficient upload also fills the plan's checkpoint cache, tuning key 32)
ids = sorted(per)
last = ids[len(ids) - len(ids) % len(names) - len(names):][:len(names)] if len(ids) >= len(names) else ids
tab[f"cfg{a.cfg}"] = {nm: per[i] for i, nm in zip(last, names)}
tab["source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                 "-k regex:dstE|thomas on tools/one_solve.py --reps 3 (the last solve's launches, "
                 "in order)")
json.dump(tab, open(out_path, "w"), indent=1)
print(json.dumps(tab, indent=1))
