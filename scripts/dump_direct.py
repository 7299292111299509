"""Dump the direct conv kernel's staged smem (debug build, `make phase`)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("VCNN_LIB_PATH", os.path.join(ROOT, "build", "libvcnn_cuda_phase.so"))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1501_07338_b200 import ops  # noqa: E402
from paper_1501_07338_b200._lib import lib  # noqa: E402

L = lib()
L.vcnn_debug_dump.argtypes = [C.c_void_p]
x = torch.arange(64, device="cuda", dtype=torch.float32).view(1, 1, 8, 8) + 1
w = torch.arange(16 * 9, device="cuda", dtype=torch.float32).view(16, 9) * 0.01 + 1
b = torch.zeros(16, device="cuda")
y = ops.conv_forward(x, w, b, 3, 3)
torch.cuda.synchronize()
buf = (C.c_float * 1024)()
L.vcnn_debug_dump(buf)
for k, nm in enumerate(["raw", "A copies", "B pack", "ep(after tmem)"]):
    print(nm, [round(buf[k * 256 + i], 3) for i in range(64)])
print("y", y[0, 0, 0].tolist())
