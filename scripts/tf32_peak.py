"""Measured dense TF32 tensor-core peak on this B200 (cuBLAS via torch,
8192^3, best of 10, CUDA events) -> profiles/tf32_peak.json, the roofline
denominator bench.py uses for tensor-bound kernels (same method as the
driver's bf16 figure in MEASURED_PEAKS.json)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    a @ b
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) * 1e-3)
tf = 2 * n ** 3 / best / 1e12
out = {"tf32_tflops": tf, "how": "torch.matmul fp32 with allow_tf32 (cuBLAS TF32 tensor cores), "
       "8192^3, best of 10, CUDA events", "gpu": torch.cuda.get_device_name()}
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "tf32_peak.json"), "w"), indent=1)
print(json.dumps(out))
