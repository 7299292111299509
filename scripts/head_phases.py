"""Phase timing of the fused two-layer tail kernel (debug build, `make phase`):
clock64 stamps per CTA of one CIFAR-3 training step.  Diagnostic only."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("VCNN_LIB_PATH", os.path.join(ROOT, "build", "libvcnn_cuda_phase.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_07338_b200 import spec as S  # noqa: E402
from paper_1501_07338_b200._lib import lib  # noqa: E402
from paper_1501_07338_b200.engine import Network  # noqa: E402
from paper_1501_07338_b200.spec import Precision  # noqa: E402

L = lib()
L.vcnn_debug_hphases.argtypes = [C.c_void_p]
B = 128
spec = S.cifar3()
net = Network(spec, B, Precision.tf32)
rng = np.random.default_rng(0)
x = torch.as_tensor(rng.standard_normal((B, 32 * 32 * 3), dtype=np.float32), device="cuda")
net.load_batch(x, cls=torch.as_tensor(rng.integers(0, 10, B).astype(np.int32), device="cuda"))
for _ in range(5):
    net.forward_backward(B)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 256)()
L.vcnn_debug_hphases(buf)
names = ["pdl-wait", "stage", "gemm1", "sync1", "reduce+head", "sync2", "gather", "gemm4", "sync3"]
for r in range(16):
    t = [buf[r * 16 + i] for i in range(16)]
    print(f"cta {r:2d} " + " ".join(f"{n}={t[i + 1] - t[i]}" for i, n in enumerate(names)),
          "total", t[9] - t[0])
    print("        head: reduce=%d y=%d loss=%d dWO+gH=%d push=%d" % (
        t[10] - t[4], t[11] - t[10], t[12] - t[11], t[13] - t[12], t[5] - t[13]))

# the shifted-view weight gradient of conv2 (wgrad.cu) in the same step
try:
    L.vcnn_debug_wphases.argtypes = [C.c_void_p]
    wb = (C.c_ulonglong * 32)()
    L.vcnn_debug_wphases(wb)
    wn = ["load", "build", "mma-issue", "mma-drain", "tmem->smem", "store"]
    for r in range(2):
        t = [wb[r * 8 + i] for i in range(8)]
        print(f"wgrad cta {r} " + " ".join(f"{n}={t[i + 1] - t[i]}" for i, n in enumerate(wn)),
              "total", t[6] - t[0])
except AttributeError:
    pass

# the small-Kd weight gradient of conv1 (wgrad.cu wgrad_small_kernel)
try:
    L.vcnn_debug_sphases.argtypes = [C.c_void_p]
    sb = (C.c_ulonglong * 32)()
    L.vcnn_debug_sphases(sb)
    sn = ["init", "pdl-wait", "load-issue+wait", "scatter+round", "mma", "reduce+store"]
    for r in range(4):
        t = [sb[r * 8 + i] for i in range(8)]
        print(f"wgrad_small cta {r} " + " ".join(f"{n}={t[i + 1] - t[i]}" for i, n in enumerate(sn)),
              "total", t[6] - t[0])
except AttributeError:
    pass

# the small-Kd forward of conv1 (direct.cu conv_small_fwd_kernel)
try:
    L.vcnn_debug_fphases.argtypes = [C.c_void_p]
    fb = (C.c_ulonglong * 32)()
    L.vcnn_debug_fphases(fb)
    fn = ["setup+pdl", "load-wait", "round", "mma", "epilogue", "pool-store"]
    for r in range(4):
        t = [fb[r * 8 + i] for i in range(8)]
        print(f"small_fwd cta {r} " + " ".join(f"{n}={t[i + 1] - t[i]}" for i, n in enumerate(fn)),
              "total", t[6] - t[0])
except AttributeError:
    pass
