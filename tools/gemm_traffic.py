"""profiles/gemm_traffic.json from an ncu launch list (tools/ncu_capture.sh): DRAM bytes
(read + write) of the K2 GEMM launches of the last complete step -- bench.py's
roofline.traffic.  python tools/gemm_traffic.py gpurun_out/launches.csv"""
import csv
import json
import os
import sys

path = sys.argv[1]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi, ii, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID"), hdr.index("Metric Name")
launch, order = {}, []
for r in rows[1:]:
    if len(r) <= vi or not r[vi]:
        continue
    lid = int(r[ii])
    if lid not in launch:
        launch[lid] = {"name": r[ki]}
        order.append(lid)
    launch[lid][r[mi]] = float(r[vi].replace(",", ""))
data = [launch[i] for i in order]
idx = [i for i, d in enumerate(data) if "propose_kernel" in d["name"]]
step = data[idx[-2]:idx[-1]]
g = [d for d in step if "gemm" in d["name"]]
out = {"dram_bytes_per_step": sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in g),
       "gemm_launches_per_step": len(g), "source": os.path.basename(path),
       "note": "ncu launch list, default cache control (caches flushed per launch): upper bound"}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                  "gemm_traffic.json"), "w"), indent=1)
print(out)
