"""Summarise an ncu report: per kernel launch, key metrics from the details page.
Usage: python tools/ncu_summary.py report.ncu-rep [regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
ki, ni, mi, ui, vi, si = (hdr.index(x) for x in ["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "Section Name"])
keep = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "L1/TEX Cache Throughput", "Dynamic Shared Memory Per Block",
        "Waves Per SM"]
cur = None
for r in rows[1:]:
    name = r[ni]
    if pat and not pat.search(name):
        continue
    key = (r[ki], name)
    if key != cur:
        cur = key
        print(f"\n== [{r[ki]}] {name[:110]}")
    if r[mi] in keep:
        print(f"   {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
