"""Phase timing of the tcgen05 GEMM kernel (debug build, `make phase`):
clock64 stamps per CTA for setup / staging / K loop / MMA drain / epilogue,
for the CIFAR-3 conv shapes through the op-level C ABI.  Diagnostic only."""
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
L.vcnn_debug_phases.argtypes = [C.c_void_p]
L.vcnn_debug_dphases.argtypes = [C.c_void_p]


def dphases(tag, fn, reps=3):
    """direct conv kernel stamps: setup, load, build, mma, epilogue, dealloc"""
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 64)()
    L.vcnn_debug_dphases(buf)
    print(f"== {tag} (direct)")
    for b in range(2):
        t = [buf[b * 8 + i] for i in range(8)]
        names = ["init", "load-wait", "build", "mma", "epilogue", "dealloc"]
        print("   cta", b, " ".join(f"{n}={t[i + 1] - t[i]}" for i, n in enumerate(names)),
              "total", t[6] - t[0],
              f"(stacked: tmem->smem {t[7] - t[4]}, sum+epilogue {t[5] - t[7]})" if t[7] > t[4] else "")
NAMES = ["setup", "stage", "kloop(prod)", "mma-issue-end", "done-wait", "epilogue", "dealloc"]


def phases(tag, fn, reps=3):
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    fn()
    ev[1].record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 128)()
    L.vcnn_debug_phases(buf)
    print(f"== {tag}: {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (events)")
    for b in range(3):
        t = [buf[b * 16 + i] for i in range(16)]
        t0 = t[0]
        d = {"setup": t[1] - t0, "stage": t[2] - t[1], "kloop(prod)": t[3] - t[2],
             "mma-end": t[4] - t[2], "done-wait": t[5] - t[2], "epilogue": t[6] - t[5],
             "dealloc": t[7] - t[6], "total": t[7] - t0}
        d.update({"prod-emptywait": t[12], "prod-gather": t[14], "mma-fullwait": t[13],
                  "nst": t[15]})
        if t[8] > t[1]:
            d.update({"x-issue": t[8] - t[1], "w-issue": t[9] - t[8], "wait": t[10] - t[9],
                      "round": t[11] - t[10]})
        print("   cta", b, " ".join(f"{k}={v}" for k, v in d.items()))


torch.manual_seed(0)
B = 128
dev = "cuda"
for name, (C_, H, K, k) in {"conv1": (3, 32, 32, 5), "conv2": (32, 14, 32, 5)}.items():
    x = torch.rand(B, C_, H, H, device=dev)
    w = (torch.rand(K, C_ * k * k, device=dev) - 0.5) * 0.1
    b = torch.zeros(K, device=dev)
    y = ops.conv_forward(x, w, b, k, k)
    dy = torch.rand_like(y)
    dphases(f"{name} fwd", lambda: ops.conv_forward(x, w, b, k, k))
    phases(f"{name} wgrad", lambda: ops.conv_backward(x, w, y, dy, k, k, need_dx=False))
    if name == "conv2":
        dphases(f"{name} dgrad", lambda: ops.conv_backward(x, w, y, dy, k, k))

# the routed dgrad inside a CIFAR-3 training step (last direct launch of backward)
from paper_1501_07338_b200 import spec as S  # noqa: E402
from paper_1501_07338_b200.engine import Network  # noqa: E402

net = Network(S.cifar3(), 128)
xb = torch.rand(128, 3 * 32 * 32, device="cuda")
cb = torch.randint(0, 10, (128,), device="cuda", dtype=torch.int32)
net.load_batch(xb, cls=cb)
dphases("cifar3 conv2 dgrad (routed, in net)", lambda: net.forward_backward(128))
