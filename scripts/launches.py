"""Summarise an ncu launch list (gpurun_out/launches.csv)."""
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[hdr]
ki, vi = H.index("Kernel Name"), H.index("Metric Value")
tot = 0.0
for r in rows[hdr + 1:]:
    name = r[ki].replace("vcnn_b200::", "").replace("(anonymous namespace)::", "")
    name = name.replace("tc::<unnamed>::", "").replace("<unnamed>::", "")
    us = float(r[vi].replace(",", "")) / 1e3
    tot += us
    print(f"{us:9.2f}us  {name[:100]}")
print(f"total {tot:.1f}us")
