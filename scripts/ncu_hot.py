"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`
(one section per profiled kernel).  usage: ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
sections, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        sections.append(cur)
    elif row and row[0] == "Address":
        cur["hdr"] = row
    elif cur is not None and row:
        cur["rows"].append(row)
for sec in sections:
    h = sec["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in sec["rows"] if r[si].isdigit())
    print("=" * 100)
    print(sec["name"][:120], "samples", tot)
    rows = sorted(sec["rows"], key=lambda r: -int(r[si]) if r[si].isdigit() else 0)
    for r in rows[:top]:
        print(f"{int(r[si]):7d} {100.0*int(r[si])/max(tot,1):5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
