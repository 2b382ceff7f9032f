"""Key metrics of an ncu --set full capture (one line block per captured launch).

python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep > profiles/r01_ncu_gemm.txt"""
import csv
import io
import subprocess
import sys

DETAILS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate",
           "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
           "Grid Size", "Block Size", "Cluster Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tc.sum", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rep = sys.argv[1]
det = page(rep, "details")
h = det[0]
ii, ki, ni, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
by = {}
for r in det[1:]:
    if len(r) <= vi:
        continue
    d = by.setdefault(r[ii], {"name": r[ki]})
    if r[ni] in DETAILS and r[ni] not in d:
        d[r[ni]] = f"{r[vi]} {r[ui]}".strip()
raw = page(rep, "raw")
rh = raw[0]
for j, r in enumerate(raw[2:]):
    d = by.get(r[rh.index("ID")]) if "ID" in rh else None
    if d is None:
        continue
    for m in RAW:  # some raw names carry a section prefix ("TPC.TriageCompute.<metric>")
        col = next((c for c, name in enumerate(rh) if name == m or name.endswith("." + m)), None)
        if col is not None:
            d[m] = r[col]
print(f"ncu --set full capture: {rep}")
for lid, d in by.items():
    print(f"\n[{lid}] {d['name'][:100]}")
    for k in DETAILS + RAW:
        if k in d:
            print(f"    {k:72s} {d[k]}")
