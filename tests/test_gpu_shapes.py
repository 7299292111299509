"""Parity at the BASELINE.json shapes themselves, on the kernels the benchmark
runs (the kernel choice depends on the geometry and the batch: direct /
small-Kd / K=1 / slab / implicit / explicit-dgrad paths, split-K plans):

  * denoise-16 (64x64, 16x16 first layer, 64 maps) and deconv-121 (184x184,
    121x1 / 1x121, 38 maps) at their real spatial shapes -- vs the oracle per
    layer (teacher-forced), the whole gradient and N SGD steps (3xTF32), at
    the oracle batch AND at the benchmark batch;
  * the single-conv sweep cells C in {64,128,256} x k in {3,7,11} on 32x32
    (forward, weight AND data gradient: the sweep conv is the second layer of
    a two-conv net so its dgrad runs too);
  * CIFAR-3 at the roofline batch 1024.

Tolerances: normwise max|gpu-ref|/max|ref| per tensor, TF32 1e-3
and 3xTF32 1e-5, no multipliers.  Conv layers are checked with the BLAS-f64
restatement (oracle_py.conv_*_np, pinned to the C oracle by
test_oracle_golden.py), everything else with the C oracle.  Each case also
asserts that the production path (trace off) computes bit-identically to the
trace path the per-layer checks read."""
import numpy as np
import pytest

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Network
from paper_1501_07338_b200.spec import Precision

from .test_gpu_net import _load, _targets, teacher_forced
from .util import TOL, assert_close, f32

pytestmark = pytest.mark.gpu
A = S.Activation
PRECS = [Precision.tf32, Precision.tf32x3]
pid = lambda p: p.name  # noqa: E731


def _run(spec, B, prec, seed=8):
    """trace-path forward_backward + the same pass on the production path;
    returns (net in trace mode after the pass, x, cls, vals)."""
    x, cls, vals = S.synth_bench_data(spec, B, seed)
    net = Network(spec, B, prec)
    _load(net, spec, x, cls, vals)
    net.forward_backward(B)
    g_prod, l_prod = net.get_grads(), net.loss()
    net.set_trace(True)
    net.forward_backward(B)
    assert np.array_equal(net.get_grads(), g_prod) and net.loss() == l_prod, \
        "production path differs from the trace path"
    return net, x, cls, vals


REAL = {  # name: (spec, oracle batch, benchmark batch, oracle SGD steps)
    "denoise16": (S.denoise16(), 2, 128, 10),
    "deconv121": (S.deconv121(), 1, 16, 2),
}


@pytest.mark.parametrize("prec", PRECS, ids=pid)
@pytest.mark.parametrize("name", list(REAL))
def test_real_shape_vs_oracle(name, prec):
    """Per layer (teacher-forced) at the real shape; for 3xTF32 also the
    loss, the whole gradient and the weights after N SGD steps (lr 0.01,
    momentum 0.9) against the oracle's own trajectory."""
    spec, B, _, steps = REAL[name]
    net, x, cls, vals = _run(spec, B, prec)
    tol = TOL[prec]
    teacher_forced(net, spec, x, B, tol, numpy_conv=True)
    if prec == Precision.tf32x3:
        p0 = net.get_params().astype(np.float64)
        r = O.net_run_batch(spec, p0, f32(x), **_targets(spec, cls, vals))
        assert abs(net.loss() - r["loss"]) <= tol * max(1.0, abs(r["loss"]))
        assert_close(net.get_grads(), r["grads"], tol, "whole gradient")
        net.set_trace(False)
        p, v = p0.copy(), np.zeros_like(p0)
        for _ in range(steps):
            net.train_step(B, 0.01, 0.9)
            g = O.net_run_batch(spec, p, f32(x), **_targets(spec, cls, vals))["grads"]
            O.sgd_step(p, v, g, 0.01, 0.9)
        assert_close(net.get_params(), p, tol, f"weights after {steps} steps")
        assert_close(net.get_params() - p0, p - p0, tol, f"update after {steps} steps")
    net.close()


@pytest.mark.parametrize("prec", PRECS, ids=pid)
@pytest.mark.parametrize("name", list(REAL) + ["cifar3-b1024"])
def test_benchmark_batch_teacher_forced(name, prec):
    """The benchmark batch (denoise-16 b128, deconv-121 b16, CIFAR-3 b1024):
    every layer's output, dW, db and handed-down gradient vs the f64
    restatement on the GPU's own trace."""
    if name == "cifar3-b1024":
        spec, B = S.cifar3(), 1024
    else:
        spec, _, B, _ = REAL[name]
    net, x, _, _ = _run(spec, B, prec)
    teacher_forced(net, spec, x, B, TOL[prec], numpy_conv=True)
    net.close()


SWEEP = [(c, k) for c in (64, 128, 256) for k in (3, 7, 11)]


def sweep_spec(c, k):
    """32x32xC -> 1x1 conv C (relu) -> the sweep cell's k x k conv C->C
    (relu) -> MSE: the sweep conv runs forward, weight AND data gradient."""
    return S.NetworkSpec((32, 32, c), [S.ConvSpec(c, 1, 1, 1, A.relu),
                                       S.ConvSpec(c, k, k, 1, A.relu)], S.LossKind.mse, 7)


@pytest.mark.parametrize("prec", PRECS, ids=pid)
@pytest.mark.parametrize("cell", SWEEP, ids=lambda t: f"c{t[0]}k{t[1]}")
def test_sweep_cell_teacher_forced(cell, prec):
    c, k = cell
    spec = sweep_spec(c, k)
    net, x, _, _ = _run(spec, 2, prec)
    teacher_forced(net, spec, x, 2, TOL[prec], numpy_conv=True)
    net.close()


@pytest.mark.parametrize("prec", PRECS, ids=pid)
@pytest.mark.parametrize("cell,B", [((64, 5), 128), ((256, 3), 128), ((128, 11), 64),
                                    ((32, 5), 1024)], ids=lambda v: str(v))
def test_sweep_bench_spec_at_batch(cell, B, prec):
    """The bench's own single-conv spec (S.single_conv) at sweep batches."""
    c, k = cell
    spec = S.single_conv(channels=c, k=k)
    net, x, _, _ = _run(spec, B, prec)
    teacher_forced(net, spec, x, B, TOL[prec], numpy_conv=True)
    net.close()


@pytest.mark.parametrize("cell,B", [((256, 7), 256), ((64, 11), 1024)], ids=str)
def test_sweep_cells_beyond_2e31_patch_elements(cell, B):
    """Sweep cells whose patch matrix (kd x pixels) exceeds 2^31 elements run
    on the implicit GEMMs (no patch is materialised): one training step is
    finite and the forward of an image equals the same image run alone."""
    import torch
    c, k = cell
    spec = S.single_conv(channels=c, k=k)
    x, _, v = S.synth_bench_data(spec, B, 8)
    net = Network(spec, B)
    _load(net, spec, x, None, v)
    net.forward(B)
    y_full = net.output(B)[:1]
    net.forward_backward(B)
    assert np.isfinite(net.loss()) and np.isfinite(net.get_grads()).all()
    one = Network(spec, 1)
    one.load_batch(torch.as_tensor(x[:1].reshape(1, -1), device="cuda"),
                   values=torch.as_tensor(v[:1], device="cuda"))
    one.forward(1)
    assert_close(y_full, one.output(1), 1e-4, "image 0 in the big batch vs alone")
    net.close()
    one.close()
