"""Shared helpers for the parity tests."""
import numpy as np

from paper_1501_07338_b200.spec import Precision

# Tolerances (north_star), normwise max|gpu-ref| / max|ref| per tensor:
#   TF32   (tcgen05 kind::tf32, fp32 accumulate in TMEM)          1e-3
#   3xTF32 (hi/lo split, 3 tcgen05 MMAs, fp32 accumulate in TMEM) 1e-5
#   FP32   (SIMT FMA, the fp32-faithful path)                     1e-5
# Whole-network TF32 gradients are additionally checked "teacher-forced"
# (every layer fed the GPU's own trace), because TF32 rounding legitimately
# flips near-tied max-pool argmaxes / ReLU kinks -- the cases the reference's
# own fd_safe() (tests/helpers.hpp:148-203) excludes from its gradient checks.
TOL = {Precision.tf32: 1e-3, Precision.tf32x3: 1e-5, Precision.fp32: 1e-5}
# Weights after N free-running training steps.  A trajectory amplifies every
# near-tie decision flip (max-pool argmax, ReLU kink) over the N steps, so the
# bar is max(TOL_STEPS, 2 x the drift of the REFERENCE'S OWN float build from
# its f64 build on the same case): no fp32 implementation can be held
# tighter than the reference is to itself.  TF32 (10-bit mantissa) gets 2e-2
# normwise plus an update-direction check; its kernel numerics are gated at
# 1e-3 per layer by the teacher-forced checks.
TOL_STEPS = {Precision.tf32: 2e-2, Precision.tf32x3: 1e-5, Precision.fp32: 1e-5}


def ref_f32_drift(spec, p0, x, cls, vals, lr, mom, steps):
    """normwise(reference float trajectory, reference f64 trajectory) after
    `steps` run_batch + sgd_step on the same fp32 inputs (oracle/_ref), for
    the weights and for the update (weights - p0)."""
    import oracle_py as O
    if O.ref() is None:
        return 0.0, 0.0
    p0 = np.asarray(p0, dtype=np.float32).astype(np.float64)
    xf = np.asarray(x, dtype=np.float32)
    p64, _ = O.ref_net_train_steps(spec, p0, xf.astype(np.float64), cls, vals, lr, mom, steps)
    p32, _ = O.ref_net_train_steps_f32(spec, p0, xf, cls, vals, lr, mom, steps)
    return normwise(p32, p64), normwise(p32 - p0, p64 - p0)
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


def act_np(act, x):
    """layers.hpp:25-34 in numpy."""
    act = int(act)
    if act == 1:
        return np.where(x > 0, x, 0.0)
    if act == 2:
        return 1.0 / (1.0 + np.exp(-x))
    if act == 3:
        return np.tanh(x)
    return x


def act_grad_np(act, y):
    """layers.hpp:39-48 in numpy (derivative from the output)."""
    act = int(act)
    if act == 1:
        return (y > 0).astype(np.float64)
    if act == 2:
        return y * (1 - y)
    if act == 3:
        return 1 - y * y
    return np.ones_like(y)
