"""Summarise an ncu --metrics gpu__time_duration.sum launch list: the last
complete speculative step (between the last two propose_kernel launches)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
data = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi and r[vi]]
idx = [i for i, (_, k, _) in enumerate(data) if "propose_kernel" in k]
s = idx[-2] if len(idx) > 1 else idx[-1]
e = idx[-1] if len(idx) > 1 else len(data)
step = data[s:e]
tot = sum(v for _, _, v in step)
agg = defaultdict(lambda: [0, 0.0])
for _, k, v in step:
    name = k.split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v
print(f"launches in one step: {len(step)}   sum of device time: {tot/1e3:.1f} us (serialised, cold-cache)")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} {n:4d} {v/1e3:9.1f} us {100*v/tot:5.1f}%")
g = [v for _, k, v in step if "gemm" in k]
print("first layer GEMMs (us):", [round(v / 1e3, 1) for v in g[:4]], " LM/heads:", [round(v / 1e3, 1) for v in g[-3:]])
