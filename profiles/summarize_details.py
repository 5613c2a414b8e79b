"""Summarise an `ncu --page details --csv` export: a few headline metrics per profiled launch."""
import csv
import json
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Ipc Active", "Grid Size")
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
ix = {h: i for i, h in enumerate(rows[hi])}
out = {}
for r in rows[hi + 1:]:
    if len(r) < 15:
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    key = f"{name} #{r[ix['ID']]}"
    m = r[ix["Metric Name"]]
    if m in KEEP:
        out.setdefault(key, {})[m] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}".strip()
print(json.dumps(out, indent=1))
