"""One-line-per-kernel summary of an ncu --set full report (duration, grid,
DRAM traffic, tensor-pipe / SM / issue utilisation, top stall reasons)."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us"), ("launch__grid_size", "grid"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__inst_executed.sum", "inst")]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    H, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[H.index("Kernel Name")]
        name = name.split("(")[0][-60:]
        parts = []
        for k, lab in KEYS:
            if k in H:
                i = H.index(k)
                parts.append(f"{lab}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
        st = [(float(r[i]), H[i]) for i in range(len(H))
              if "smsp__pcsamp_warps_issue_stalled" in H[i] and "not_issued" not in H[i]
              and r[i].replace(".", "", 1).isdigit()]
        tot = sum(v for v, _ in st) or 1
        st.sort(reverse=True)
        stalls = ",".join(f"{n.split('stalled_')[1]}:{100 * v / tot:.0f}%" for v, n in st[:4])
        print(f"{name} | " + " ".join(parts) + f" | stalls {stalls}")
