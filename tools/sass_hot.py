"""Top stalled SASS instructions from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
k = hdr.index("Warp Stall Sampling (All Samples)")
ex = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[k]), int(r[ex]), r[0], r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total stall samples", tot)
order = sorted(range(len(data)), key=lambda i: -data[i][0])
for i in order[: int(sys.argv[1]) if len(sys.argv) > 1 else 25]:
    d = data[i]
    print(f"{d[0]:7d} {100*d[0]/max(tot,1):5.1f}%  exec {d[1]:8d}  [{i:5d}] {d[3][:100]}")
