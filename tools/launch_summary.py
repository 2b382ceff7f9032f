"""Summarise an ncu --csv launch list (metrics gpu__time_duration.sum and,
optionally, dram__bytes_read/write.sum): the last complete speculative step
(between the last two propose_kernel launches), per kernel name."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi, ii, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID"), hdr.index("Metric Name")
launch = {}
order = []
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
s = idx[-2] if len(idx) > 1 else idx[-1]
e = idx[-1] if len(idx) > 1 else len(data)
step = data[s:e]
T = "gpu__time_duration.sum"
tot = sum(d.get(T, 0) for d in step)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for d in step:
    name = d["name"].split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += d.get(T, 0)
    agg[name][2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
print(f"launches in one step: {len(step)}   sum of device time: {tot/1e3:.1f} us (ncu: serialised, cold-cache)")
print(f"{'kernel':60s} {'n':>4s} {'time us':>9s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>7s}")
for k, (n, v, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = b / v if v else 0.0  # bytes / ns = GB/s
    print(f"{k:60s} {n:4d} {v/1e3:9.1f} {100*v/tot:5.1f}% {b/1e6:9.1f} {gbs:7.0f}")
g = [d.get(T, 0) for d in step if "gemm" in d["name"]]
print("first layer GEMMs (us):", [round(v / 1e3, 1) for v in g[:4]], " LM/heads:", [round(v / 1e3, 1) for v in g[-3:]])
if len(sys.argv) > 2:  # write the K2 DRAM traffic per step for bench.py's roofline.traffic
    import json
    gb = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in step if "gemm" in d["name"])
    gn = sum(1 for d in step if "gemm" in d["name"])
    json.dump({"dram_bytes_per_step": gb, "gemm_launches_per_step": gn, "source": path,
               "note": "ncu launch list, default cache control (caches flushed per launch): upper bound"},
              open(sys.argv[2], "w"), indent=1)
