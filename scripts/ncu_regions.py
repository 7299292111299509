"""Warp-stall samples of one profiled kernel summed per region between
block / cluster barriers (BAR.SYNC, UCGABAR_*), with the top stall reasons of
each region.  usage: ncu_regions.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[start]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stalls = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
regions, cur = [], None


def new(label):
    return {"label": label, "samples": 0, "inst": 0, "n": 0, "st": {}}


cur = new("entry")
for r in rows[start + 1:]:
    if len(r) <= si or not r[si].strip().isdigit():
        continue
    src = r[1].strip()
    if "BAR.SYNC" in src or "UCGABAR" in src:
        regions.append(cur)
        cur = new(src.split()[0] + " @" + r[0][-5:])
    cur["samples"] += int(r[si])
    cur["inst"] += int(r[ie]) if r[ie].isdigit() else 0
    cur["n"] += 1
    for j, h in stalls:
        v = r[j].strip()
        if v.isdigit() and int(v):
            cur["st"][h] = cur["st"].get(h, 0) + int(v)
regions.append(cur)
tot = sum(g["samples"] for g in regions)
for g in regions:
    top = sorted(g["st"].items(), key=lambda kv: -kv[1])[:4]
    print(f"{g['label']:28s} {g['samples']:7d} {100.0 * g['samples'] / tot:5.1f}%  sass={g['n']:5d} "
          f"inst={g['inst']:8d}  " + " ".join(f"{k[6:]}={v}" for k, v in top))
