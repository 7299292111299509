"""Direct (shifted-view) conv kernels vs torch on small shapes (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_1501_07338_b200 import ops  # noqa: E402

torch.backends.cudnn.allow_tf32 = False
torch.manual_seed(0)
for (B, C, H, K, k) in [(1, 1, 8, 16, 3), (1, 8, 8, 16, 1), (2, 3, 12, 16, 5), (2, 32, 14, 32, 5),
                        (3, 3, 32, 32, 5)]:
    x = torch.rand(B, C, H, H, device="cuda")
    w = torch.rand(K, C * k * k, device="cuda") - 0.5
    b = torch.rand(K, device="cuda")
    y = ops.conv_forward(x, w, b, k, k)
    ref = F.conv2d(x.double(), w.double().view(K, C, k, k), b.double())
    err = (y.double() - ref).abs().max().item() / ref.abs().max().item()
    dy = torch.rand_like(y)
    dw, db, dx = ops.conv_backward(x, w, y, dy, k, k)
    xr = x.double().requires_grad_()
    wr = w.double().view(K, C, k, k).requires_grad_()
    out = F.conv2d(xr, wr)
    out.backward(dy.double())
    edx = (dx.double() - xr.grad).abs().max().item() / xr.grad.abs().max().item()
    print(f"B{B} C{C} H{H} K{K} k{k}: fwd err {err:.2e}  dgrad err {edx:.2e}")
    if err > 1e-2:
        print("  y[0,0,:2]", y[0, 0, :2].tolist())
        print("  r[0,0,:2]", ref[0, 0, :2].tolist())
