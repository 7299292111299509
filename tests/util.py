"""Shared helpers for the parity tests."""
import numpy as np

from paper_1501_07338_b200.spec import Precision

# Tolerances (north_star): normwise max|gpu-ref| / max|ref|.
#   TF32 (tcgen05 kind::tf32, fp32 accumulate)       1e-3
#   3xTF32 (split hi/lo, fp32-faithful) and FP32 SIMT 1e-5
TOL = {Precision.tf32: 1e-3, Precision.tf32x3: 1e-5, Precision.fp32: 1e-5}
ALL_PREC = [Precision.tf32, Precision.tf32x3, Precision.fp32]


def normwise(gpu, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape or gpu.size == ref.size, (gpu.shape, ref.shape)
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    return float(np.abs(gpu.reshape(ref.shape) - ref).max(initial=0.0) / scale)


def assert_close(gpu, ref, tol, what=""):
    e = normwise(gpu, ref)
    assert e <= tol, f"{what}: normwise error {e:.3e} > {tol:.1e}"
    return e


def f32(a):
    """Round to fp32 (the GPU's input precision), returned as float64 for the oracle."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)
