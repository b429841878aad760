"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv).

Kernels are grouped by family; per-apply figures divide by the number of applies seen
(launches of the apply's first kernel, weights_kernel). Shares are of the summed device time
of one apply (ncu launches are serialised and cold-cache: compare shares, not absolutes).
Usage: python tools/ncu_launches.py launches.csv [out.json]"""
import csv, json, re, sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
I = {h: i for i, h in enumerate(hdr)}
launch = defaultdict(dict)
for r in rows[1:]:
    launch[int(r[I["ID"]])]["name"] = r[I["Kernel Name"]]
    v = r[I["Metric Value"]].replace(",", "")
    launch[int(r[I["ID"]])][r[I["Metric Name"]]] = float(v)


def family(name):
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name.split("(")[0]


applies = sum(1 for l in launch.values() if family(l["name"]) == "weights_kernel")
fam = defaultdict(lambda: {"launches": 0, "ns": 0.0, "dram_read": 0.0, "dram_write": 0.0})
first_apply = min(i for i, l in launch.items() if family(l["name"]) == "weights_kernel")
for i, l in launch.items():
    if i < first_apply:
        fam["setup:" + family(l["name"])]["launches"] += 1
        continue
    f = fam[family(l["name"])]
    f["launches"] += 1
    f["ns"] += l.get("gpu__time_duration.sum", 0.0)
    f["dram_read"] += l.get("dram__bytes_read.sum", 0.0)
    f["dram_write"] += l.get("dram__bytes_write.sum", 0.0)
tot = sum(f["ns"] for k, f in fam.items() if not k.startswith("setup:")) / max(applies, 1)
out = {"applies": applies, "apply_ms_serialised": tot * 1e-6, "kernels": {}}
for k, f in sorted(fam.items(), key=lambda kv: -kv[1]["ns"]):
    if k.startswith("setup:"):
        out["kernels"][k] = {"launches": f["launches"]}
        continue
    a = max(applies, 1)
    out["kernels"][k] = {"launches_per_apply": f["launches"] / a, "ms_per_apply": f["ns"] / a * 1e-6,
                         "share": f["ns"] / a / tot, "dram_bytes_per_apply": (f["dram_read"] + f["dram_write"]) / a}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
