"""Per-kernel counts of the instructions that show which hardware path a
kernel uses (cuobjdump -sass of libvcnn_cuda.so): UTCHMMA / UTCQMMA (tcgen05
MMA), HMMA (legacy mma.sync), LDTM (tcgen05.ld), UTMALDG (tensor TMA),
UBLKCP (bulk copy), FFMA (SIMT fp32)."""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_1501_07338_b200/libvcnn_cuda.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
keys = ["UTCHMMA", "UTCQMMA", "HMMA", "LDTM", "UTMALDG", "UBLKCP", "FFMA"]
counts = collections.OrderedDict()
fn = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    if fn is None:
        continue
    for k in keys:
        if re.search(r"\b" + k + r"\b", line):
            counts[fn][k] += 1


def short(name):
    try:
        d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        d = name
    return re.sub(r"vcnn_b200::|\(anonymous namespace\)::", "", d)[:110]


print("%-110s " % "kernel" + " ".join("%8s" % k for k in keys))
seen = set()
for fn, c in counts.items():
    row = "%-110s " % short(fn) + " ".join("%8d" % c[k] for k in keys)
    if any(c[k] for k in keys[:6]) and row not in seen:  # (each cubin lists a kernel once)
        seen.add(row)
        print(row)
