"""Network-level parity on the B200: the device engine (build_network +
Executor<float>(imp6) + sgd_step through the net-level C ABI) vs
  * the reference's own numbers (tests/golden fixtures from oracle/_ref), and
  * the oracle (double) on the same fp32 inputs and parameters,
plus the reference's invariants (determinism, batch equivalence, bounds and
training errors) and full-size checks at the BASELINE.json configs."""
import glob
import os

import numpy as np
import pytest
import torch

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.engine import Executor, Network, Trainer, predict_classes
from paper_1501_07338_b200.errors import BoundsError, ShapeError, TrainingError
from paper_1501_07338_b200.spec import Precision

from .util import ALL_PREC, TOL, TOL_STEPS, act_grad_np, act_np, assert_close, ref_f32_drift, f32, normwise
from .util import assert_close as _assert_close

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
A = S.Activation


def _targets(spec, cls, vals):
    return dict(cls=cls) if spec.loss == S.LossKind.softmax_ce else dict(values=vals)


def _load(net, spec, x, cls, vals):
    B = x.shape[0]
    xt = torch.as_tensor(x.reshape(B, -1), device="cuda")
    if spec.loss == S.LossKind.softmax_ce:
        net.load_batch(xt, cls=torch.as_tensor(cls, device="cuda"))
    else:
        net.load_batch(xt, values=torch.as_tensor(vals.reshape(B, -1), device="cuda"))


def _fixture_nets():
    from .golden.make_golden import small_nets
    return small_nets()


def teacher_forced(net, spec, x, B, tol, pool_bwd_mode=0, numpy_conv=False):
    """Per-layer parity of one forward_backward pass with every layer fed the
    GPU's own trace (input activations, pre-activation gradients, argmax):
    isolates kernel numerics from decision flips (TF32 rounding of near-tied
    max-pool argmaxes / ReLU kinks).  Checks each layer's output, dW, db and
    the gradient it hands to the layer below, all at `tol` (normwise).
    numpy_conv: conv layers checked with the BLAS-f64 restatement
    (oracle_py.conv_*_np, pinned to the C oracle) -- the full-size shapes."""
    worst = 0.0

    def assert_close(a, b, t, what):  # noqa: F811 -- records the worst error
        nonlocal worst
        worst = max(worst, _assert_close(a, b, t, what))

    cf = O.conv_forward_np if numpy_conv else O.conv_forward
    cb = O.conv_backward_np if numpy_conv else O.conv_backward
    chain = spec.chain()
    h, w, c = spec.input
    params = net.get_params().astype(np.float64)
    grads = net.get_grads()
    a_prev = f32(x).reshape(B, c, h, w)
    for i, L in enumerate(spec.layers):
        oh, ow, oc = chain[i]
        y = net.layer_output(i, B).astype(np.float64).reshape(B, oc, oh, ow)
        G = net.layer_grad(i, B).astype(np.float64).reshape(B, oc, oh, ow)
        Wt, bb = net.layer_params(params, i)
        gW, gb = net.layer_params(grads, i)
        dx = None
        if isinstance(L, S.ConvSpec):
            Wm = Wt.reshape(L.maps, -1)
            yr = cf(a_prev, Wm, bb, L.kh, L.kw, L.stride, int(L.act))
            assert_close(y, yr, tol, f"layer {i} conv out")
            dw, db, dx = cb(a_prev, Wm, y, G, L.kh, L.kw, L.stride, 0, need_dx=i > 0)
            assert_close(gW, dw, tol, f"layer {i} conv dW")
            assert_close(gb, db, tol, f"layer {i} conv db")
        elif isinstance(L, S.PoolSpec):
            pr, arg = O.pool_forward(a_prev, L.ph, L.pw, L.stride, int(L.mode))
            if L.mode == S.PoolMode.max:
                assert np.array_equal(net.pool_arg(i, B).reshape(arg.shape), arg), \
                    f"layer {i} argmax (same input) not bit-exact"
            if L.bias:
                pr = pr + bb.reshape(1, -1, 1, 1)
                assert_close(gb, G.sum(axis=(0, 2, 3)), tol, f"layer {i} pool db")
            assert_close(y, act_np(L.act, pr), tol, f"layer {i} pool out")
            if i > 0:
                dx = O.pool_backward(G, arg if L.mode == S.PoolMode.max else None, a_prev.shape,
                                     L.ph, L.pw, L.stride, int(L.mode), pool_bwd_mode)
        else:
            Wm = Wt.reshape(L.units, -1)
            yr = O.full_forward(a_prev.reshape(B, -1), Wm, bb, int(L.act))
            assert_close(y.reshape(B, -1), yr, tol, f"layer {i} fc out")
            dw, db, dx = O.full_backward(a_prev.reshape(B, -1), Wm, y.reshape(B, -1),
                                         G.reshape(B, -1), 0, need_dx=i > 0)
            assert_close(gW, dw, tol, f"layer {i} fc dW")
            assert_close(gb, db, tol, f"layer {i} fc db")
        if i > 0:
            prev = spec.layers[i - 1]
            gprev_ref = dx.reshape(a_prev.shape) * act_grad_np(prev.act, a_prev)
            gprev = net.layer_grad(i - 1, B).astype(np.float64).reshape(a_prev.shape)
            assert_close(gprev, gprev_ref, tol, f"layer {i} -> {i - 1} gradient")
        a_prev = y
    return worst


def test_init_bit_exact_vs_reference():
    """build_network<float>: Glorot stream from Rng(seed) (layers.hpp:473-501)."""
    for name, f in S.PRESETS.items():
        spec = f()
        net = Network(spec, 2)
        p_ref = O.net_init(spec).astype(np.float32)  # == reference (pinned in CPU tests)
        assert np.array_equal(net.get_params(), p_ref), name
        net.close()


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "net_*.npz"))),
                         ids=lambda p: os.path.basename(p)[4:-4])
def test_net_vs_reference_fixture(path, prec):
    """One run_batch and N run_batch+sgd_step steps vs the reference's numbers."""
    name = os.path.basename(path)[4:-4]
    spec, B = _fixture_nets()[name]
    d = np.load(path)
    net = Network(spec, B, prec)
    net.set_trace(True)  # per-layer checks read the whole trace
    x, cls, vals = d["x"], d["cls"], d["values"]
    _load(net, spec, x, cls, vals)
    net.forward_backward(B)
    tol = TOL[prec]
    assert_close(net.output(B), d["out"], tol, "output")
    assert abs(net.loss() - float(d["loss"])) <= tol * max(1.0, abs(float(d["loss"])))
    strict = prec != Precision.tf32
    if strict:  # every NetGrads tensor vs the reference
        g = net.get_grads()
        for i in range(len(spec.layers)):
            gw, gb = net.layer_params(g, i)
            rw, rb = net.layer_params(d["grads"], i)
            if rw.size:
                assert_close(gw, rw, tol, f"layer {i} dW")
            if rb.size and np.abs(rb).max() > 1e-7:
                assert_close(gb, rb, tol, f"layer {i} db")
    else:
        teacher_forced(net, spec, x, B, tol)
    # paper_nn pool backward mode (Executor::set_pool_backward_mode):
    # whole gradient vs the reference (fp32-faithful modes) and per layer,
    # teacher-forced, in every mode
    net.set_pool_backward_mode(S.PoolBackwardMode.paper_nn)
    net.forward_backward(B)
    if strict:
        assert_close(net.get_grads(), d["grads_paper_nn"], tol, "paper_nn grads")
    teacher_forced(net, spec, x, B, tol, pool_bwd_mode=1)
    net.set_pool_backward_mode(S.PoolBackwardMode.exact)
    # N steps on the production path (fusion on), weights after
    net.set_trace(False)
    for _ in range(int(d["steps"])):
        net.train_step(B, float(d["lr"]), float(d["mom"]))
    p = net.get_params()
    p0 = d["params0"]
    is_ce = spec.loss == S.LossKind.softmax_ce
    drift, udrift = ref_f32_drift(spec, p0, x, cls if is_ce else None, None if is_ce else vals,
                                  float(d["lr"]), float(d["mom"]), int(d["steps"]))
    assert_close(p, d["params_after"], max(TOL_STEPS[prec], 2 * drift), "weights after N steps")
    if strict:
        assert_close(p - p0, d["params_after"] - p0, max(tol, 2 * udrift),
                     "update after N steps")
    net.close()


PARITY_NETS = {
    "cifar3": (S.cifar3(), 16),
    "lenet-caffe": (S.lenet_caffe(), 10),
    "scale1-analog": (S.lenet_scale1_analog(), 8),
    "denoise16-small": (S.NetworkSpec((40, 40, 1), [S.ConvSpec(16, 16, 16, 1, A.relu),
                                                    S.ConvSpec(16, 1, 1, 1, A.relu),
                                                    S.ConvSpec(1, 8, 8, 1, A.identity)],
                                      S.LossKind.mse, 7), 4),
    "deconv-small": (S.NetworkSpec((60, 60, 1), [S.ConvSpec(8, 31, 1, 1, A.identity),
                                                 S.ConvSpec(8, 1, 31, 1, A.relu),
                                                 S.ConvSpec(1, 5, 5, 1, A.identity)],
                                   S.LossKind.mse, 7), 2),
}


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
@pytest.mark.parametrize("name", list(PARITY_NETS))
def test_net_vs_oracle_10_steps(name, prec):
    """Layer outputs, pool argmax (bit-exact), loss, every gradient, and the
    weights after 10 sgd steps (lr 0.01, momentum 0.9) vs the oracle."""
    spec, B = PARITY_NETS[name]
    x, cls, vals = O.synth_bench_data(spec, B, 8)
    net = Network(spec, B, prec)
    net.set_trace(True)
    _load(net, spec, x, cls, vals)
    net.forward_backward(B)
    p0 = net.get_params().astype(np.float64)
    r = O.net_run_batch(spec, p0, f32(x), trace=True, **_targets(spec, cls, vals))
    tol = TOL[prec]
    strict = prec != Precision.tf32
    off = 0
    for i, L in enumerate(spec.layers):
        n = B * net.out_per[i]
        assert_close(net.layer_output(i, B).ravel(), r["trace"][off:off + n], tol,
                     f"layer {i} output")
        off += n
    assert abs(net.loss() - r["loss"]) <= tol * max(1.0, abs(r["loss"]))
    if strict:
        assert_close(net.get_grads(), r["grads"], tol, "grads")
    teacher_forced(net, spec, x, B, tol)
    # 10 steps on the production path (fusion on)
    net.set_trace(False)
    p, v = p0.copy(), np.zeros_like(p0)
    for _ in range(10):
        net.train_step(B, 0.01, 0.9)
        g = O.net_run_batch(spec, p, f32(x), **_targets(spec, cls, vals))["grads"]
        O.sgd_step(p, v, g, 0.01, 0.9)
    pg = net.get_params()
    is_ce = spec.loss == S.LossKind.softmax_ce
    drift, udrift = ref_f32_drift(spec, p0, x, cls if is_ce else None, None if is_ce else vals,
                                  0.01, 0.9, 10)
    assert_close(pg, p, max(TOL_STEPS[prec], 2 * drift), "weights after 10 steps")
    if strict:
        assert_close(pg - p0, p - p0, max(tol, 2 * udrift), "update after 10 steps")
    else:  # TF32: decision flips allowed, the update direction must agree
        du, dr = (pg - p0).ravel(), (p - p0).ravel()
        assert float(du @ dr) / (np.linalg.norm(du) * np.linalg.norm(dr)) > 0.98
    net.close()


def test_pool_argmax_bit_exact_in_net():
    """ArgIndex of the engine's max pools == oracle (fp32-faithful path)."""
    spec = S.cifar3()
    B = 8
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    net = Network(spec, B, Precision.fp32)
    net.set_trace(True)
    _load(net, spec, x, cls, None)
    net.forward(B)
    # feed each pool the GPU's own conv output so the comparison isolates pooling
    for i, L in enumerate(spec.layers):
        if isinstance(L, S.PoolSpec):
            hh, ww, cc = spec.chain()[i - 1]
            prev = net.layer_output(i - 1, B).reshape(B, cc, hh, ww).astype(np.float64)
            y, arg = O.pool_forward(prev, L.ph, L.pw, L.stride, int(L.mode))
            assert np.array_equal(net.pool_arg(i, B).reshape(arg.shape), arg)
            assert np.array_equal(net.layer_output(i, B).reshape(y.shape), y.astype(np.float32))
    net.close()


@pytest.mark.parametrize("prec", [Precision.tf32, Precision.tf32x3])
def test_deterministic_and_graph_equivalent(prec):
    """Training is bitwise reproducible (network_test.cpp:219-244); graph
    replay == eager launches bit for bit."""
    spec = S.cifar3()
    B = 64
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    runs = []
    for graph in (False, False, True):
        net = Network(spec, B, prec)
        net.enable_graph(graph)
        _load(net, spec, x, cls, None)
        for _ in range(5):
            net.train_step(B, 0.01, 0.9)
        runs.append(net.get_params())
        net.close()
    assert np.array_equal(runs[0], runs[1])
    assert np.array_equal(runs[0], runs[2])


@pytest.mark.parametrize("name", ["single-conv", "denoise16"])
def test_graph_equivalent_single_and_multi_step(name):
    """Graph capture of nets whose weight gradients are placed differently
    across the streams (a one-layer net: nothing on the side stream; layer 0
    on the main stream in one-step graphs, on the side stream inside
    multi-step graphs) -- eager, one-step graphs and multi-step graphs
    give the same bits."""
    spec = S.PRESETS[name]() if name != "single-conv" else S.single_conv(8, 5, 16)
    B = 8
    x, _, vals = O.synth_bench_data(spec, B, 8)
    runs = []
    for mode in ("eager", "graph", "steps"):
        net = Network(spec, B)
        net.enable_graph(mode != "eager")
        _load(net, spec, x, None, vals)
        if mode == "steps":
            net.train_steps(4, B, 0.01, 0.9)
        else:
            for _ in range(4):
                net.train_step(B, 0.01, 0.9)
        runs.append(net.get_params())
        net.close()
    assert np.array_equal(runs[0], runs[1])
    assert np.array_equal(runs[0], runs[2])


def test_host_path_equals_device_path():
    spec = S.cifar3()
    B = 32
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    a = Network(spec, B)
    b = Network(spec, B)
    a.enable_graph(True)
    losses = [a.train_step_host(x, cls=cls, lr=0.01, momentum=0.9) for _ in range(3)]
    _load(b, spec, x, cls, None)
    for _ in range(3):
        b.train_step(B, 0.01, 0.9)
    assert np.array_equal(a.get_params(), b.get_params())
    assert abs(losses[-1] - b.loss()) == 0.0
    out = a.forward_host(x)
    a.forward(B)
    assert np.array_equal(out, a.output(B))


def test_batch_equivalence_on_device():
    """network_test.cpp:99-160: batch forward == per-sample forwards; grads ==
    mean of per-sample grads (fp32-faithful path)."""
    spec = S.NetworkSpec((9, 10, 2), [S.ConvSpec(3, 3, 2, 1, A.tanh),
                                      S.PoolSpec(2, 2, 1, S.PoolMode.max, True, A.sigmoid),
                                      S.FullSpec(3, A.identity)], S.LossKind.softmax_ce, 5)
    B = 4
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (B, 2, 9, 10)).astype(np.float32)
    cls = np.array([0, 2, 1, 1], dtype=np.int32)
    net = Network(spec, B, Precision.tf32x3)
    _load(net, spec, x, cls, None)
    net.forward_backward(B)
    whole_out, whole_g = net.output(B), net.get_grads()
    acc = np.zeros_like(whole_g, dtype=np.float64)
    for b in range(B):
        _load(net, spec, x[b:b + 1], cls[b:b + 1], None)
        net.forward_backward(1)
        assert_close(net.output(1)[0], whole_out[b], 1e-6, "per-sample out")
        acc += net.get_grads()
    assert_close(whole_g, acc / B, 1e-5, "mean of per-sample grads")


def test_errors():
    spec = S.cifar3()
    net = Network(spec, 4)
    x, cls, _ = O.synth_bench_data(spec, 4, 8)
    bad = cls.copy()
    bad[1] = 10
    with pytest.raises(BoundsError):
        net.train_step_host(x, cls=bad, lr=0.01, momentum=0.0)
    with pytest.raises(ShapeError):
        net.train_step(5, 0.01, 0.0)  # > max_batch
    with pytest.raises(ShapeError):
        Network(S.NetworkSpec((4, 4, 1), [S.ConvSpec(2, 5, 5)]), 1)
    ex = Executor()
    with pytest.raises(BoundsError):
        ex.run_batch(net, x, bad)


def test_trainer_nonfinite_names_layer():
    """network_test.cpp:286-306: a NaN loss raises TrainingError naming a layer."""
    spec = S.NetworkSpec((4, 4, 1), [S.ConvSpec(2, 2, 2, 1, A.identity),
                                     S.PoolSpec(2, 2, 1, S.PoolMode.avg),
                                     S.FullSpec(2, A.identity)], S.LossKind.softmax_ce, 14)
    net = Network(spec, 10)
    p = net.get_params()
    w, _ = net.layer_params(p, 0)
    w[:] = np.where(np.arange(w.size) % 2, 1.0, -1.0) * 3e38
    net.set_params(p)
    imgs = np.random.default_rng(1).uniform(0, 1, (10, 1, 4, 4)).astype(np.float32) * 1e3
    tr = Trainer(S.TrainConfig(lr=0.01, batch=10, epochs=1))
    with pytest.raises(TrainingError, match="layer"):
        tr.fit(net, imgs, np.zeros(10, dtype=np.int32))


def test_trainer_loss_decreases_and_predicts():
    """network_test.cpp:246-284 analog on a separable toy set."""
    rng = np.random.default_rng(3)
    n = 64
    labels = (np.arange(n) % 2).astype(np.int32)
    imgs = rng.uniform(0, 0.2, (n, 1, 6, 6)).astype(np.float32)
    imgs[labels == 1, :, :3, :] += 0.8
    spec = S.NetworkSpec((6, 6, 1), [S.ConvSpec(4, 3, 3, 1, A.relu), S.PoolSpec(2, 2, 2),
                                     S.FullSpec(2, A.identity)], S.LossKind.softmax_ce, 12)
    net = Network(spec, n)
    tr = Trainer(S.TrainConfig(lr=0.05, momentum=0.9, batch=n, epochs=20, seed=4))
    hist = tr.fit(net, imgs, labels)
    assert hist[-1] < hist[0]
    assert tr.evaluate_accuracy(net, imgs, labels) > 0.9
    assert predict_classes(np.array([[0.1, 2.0, -1.0], [0.7, 0.3, 0.7]])) == [1, 0]


@pytest.mark.parametrize("name,B", [("cifar3", 128), ("lenet-caffe", 100)])
def test_full_size_step_vs_oracle(name, B):
    """BASELINE configs at their full benchmark batch: one step vs the oracle,
    and the TF32 gradient vs the fp32-faithful gradient (size-independent)."""
    spec = S.PRESETS[name]()
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    net = Network(spec, B, Precision.tf32)
    net.set_trace(True)
    _load(net, spec, x, cls, None)
    net.forward_backward(B)
    r = O.net_run_batch(spec, net.get_params().astype(np.float64), f32(x), cls=cls)
    assert abs(net.loss() - r["loss"]) <= 1e-3 * r["loss"]
    teacher_forced(net, spec, x, B, TOL[Precision.tf32])
    net.set_precision(Precision.tf32x3)
    net.forward_backward(B)
    assert normwise(net.get_grads(), r["grads"]) <= TOL[Precision.tf32x3]
    net.close()


@pytest.mark.parametrize("B", [32, 64, 96, 128, 100])
def test_tail_batch_slices_vs_oracle(B):
    """The fused two-layer tail runs in 1 / 2 / 4 / 8 batch slices (one
    cluster each) by batch size: the loss (summed over slices by the last
    one) and every layer's output / dW / db / handed-down gradient match the
    oracle; the update (slice partials folded into sgd_pack) equals the
    unfused reference of the same step within TF32 tolerance."""
    spec = S.cifar3()
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    net = Network(spec, B, Precision.tf32)
    net.set_trace(True)
    _load(net, spec, x, cls, None)
    net.forward_backward(B)
    r = O.net_run_batch(spec, net.get_params().astype(np.float64), f32(x), cls=cls)
    assert abs(net.loss() - r["loss"]) <= 1e-3 * r["loss"], (net.loss(), r["loss"])
    teacher_forced(net, spec, x, B, TOL[Precision.tf32])
    g_fb = net.get_grads()
    p0 = net.get_params()
    net.train_step(B, 0.01, 0.9)  # folded update: grads rewritten by sgd_pack
    assert np.array_equal(net.get_grads(), g_fb)
    want = (p0.astype(np.float64) - np.float64(np.float32(0.01)) * g_fb).astype(np.float32)
    assert_close(net.get_params(), want, 1e-6, "folded update")
    net.close()


def test_big_batch_and_presets_run():
    """Every BASELINE config builds and steps at its benchmark size; losses are
    finite and training lowers the loss on a fixed batch."""
    for name, B in [("cifar3", 1024), ("denoise16", 128), ("deconv121", 16),
                    ("scale2-mini", 128), ("single-conv", 64)]:
        spec = S.PRESETS[name]()
        x, cls, vals = O.synth_bench_data(spec, B, 8)
        net = Network(spec, B)
        _load(net, spec, x, cls, vals)
        net.forward_backward(B)
        l0 = net.loss()
        assert np.isfinite(l0), name
        for _ in range(5):
            net.train_step(B, 0.01, 0.9)
        net.forward_backward(B)
        assert net.loss() < l0, name
        net.close()


@pytest.mark.parametrize("name,B", [("cifar3", 128), ("cifar3", 37), ("cifar3", 512), ("lenet-caffe", 100),
                                    ("scale1-analog", 8)])
def test_fused_path_bitwise_equals_trace_path(name, B):
    """conv->max-pool fusion (pool in the conv epilogue, pool backward routed
    inside the conv's wgrad / dgrad) changes no bit: loss, output, every
    gradient and the weights after 3 SGD steps equal the unfused trace path,
    whose layers are checked against the oracle above."""
    spec = S.PRESETS[name]() if name in S.PRESETS else PARITY_NETS[name][0]
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    res = []
    for trace in (True, False):
        net = Network(spec, B, Precision.tf32)
        net.set_trace(trace)
        _load(net, spec, x, cls, None)
        net.forward_backward(B)
        out, loss, g = net.output(B), net.loss(), net.get_grads()
        for _ in range(3):
            net.train_step(B, 0.01, 0.9)
        res.append((out, loss, g, net.get_params(), net.kernels_per_step()))
        net.close()
    (o0, l0, g0, p0, k0), (o1, l1, g1, p1, k1) = res
    assert np.array_equal(o0, o1) and l0 == l1
    assert np.array_equal(g0, g1)
    assert np.array_equal(p0, p1)
    assert k1 < k0, (k1, k0)  # the fused step launches fewer kernels


def test_resident_epoch_loop_equals_host_loop():
    """vcnn_net_train_epoch (dataset in HBM, index-gather kernel, graph
    replay) trains bit-identically to the host-gather
    Trainer: same Rng permutation, same batches incl. the smaller last one."""
    rng = np.random.default_rng(5)
    n = 70  # 2 full batches of 32 + one of 6
    spec = S.cifar3()
    imgs = rng.uniform(0, 1, (n, 3, 32, 32)).astype(np.float32)
    labels = rng.integers(0, 10, n).astype(np.int32)
    cfg = S.TrainConfig(lr=0.01, momentum=0.9, batch=32, epochs=2, seed=3)
    res = []
    for resident in (False, True):
        net = Network(spec, 32)
        hist = Trainer(cfg).fit(net, imgs, labels, resident=resident)
        res.append((hist, net.get_params()))
        net.close()
    assert np.array_equal(res[0][1], res[1][1])
    assert np.allclose(res[0][0], res[1][0], rtol=0, atol=1e-6)
    net = Network(spec, 32)
    bad = labels.copy()
    bad[3] = 10
    with pytest.raises(BoundsError):
        Trainer(cfg).fit(net, imgs, bad, resident=True)


def test_model_export_reference_predicts_the_same(tmp_path):
    """Device-trained weights -> ModelFile v1 -> the reference's own loader
    (io.cpp) -> the reference forward agrees with the device forward; and
    Network.from_model restores the parameters bit for bit."""
    spec = S.cifar3()
    B = 16
    x, cls, _ = O.synth_bench_data(spec, B, 8)
    net = Network(spec, B)
    _load(net, spec, x, cls, None)
    for _ in range(3):
        net.train_step(B, 0.01, 0.9)
    f = str(tmp_path / "trained.vcnn")
    net.save_model(f)
    p_ref = O.ref_load_model_f32(f, net.nparams)
    assert np.array_equal(p_ref, net.get_params())
    out_ref = O.ref_net_run_batch(spec, p_ref.astype(np.float64), f32(x), grads=False)["out"]
    out = net.forward_host(x)
    assert_close(out, out_ref, TOL[Precision.tf32], "reference forward of exported weights")
    net2 = Network.from_model(f, B)
    assert np.array_equal(net2.get_params(), net.get_params())
    net.close()
    net2.close()


@pytest.mark.parametrize("prec", [Precision.tf32x3, Precision.fp32], ids=lambda p: p.name)
def test_large_mse_loss_multi_cta(prec):
    """A conv-output MSE large enough for the multi-CTA loss kernel (per-CTA
    partials, last-CTA fixed-order reduce): loss and gradients match the
    oracle, and two runs are bit-identical (deterministic reduction)."""
    spec = S.single_conv(channels=8, k=3, hw=32)
    B = 64  # 64 x 8 x 30 x 30 = 460,800 loss elements
    x, cls, vals = O.synth_bench_data(spec, B, 8)
    outs = []
    for _ in range(2):
        net = Network(spec, B, prec)
        _load(net, spec, x, cls, vals)
        net.forward_backward(B)
        outs.append((net.loss(), net.get_grads(), net.get_params().astype(np.float64)))
        net.close()
    (l0, g0, p0), (l1, g1, _) = outs
    assert l0 == l1 and np.array_equal(g0, g1)
    r = O.net_run_batch(spec, p0, f32(x), values=vals)
    assert abs(l0 - r["loss"]) <= TOL[prec] * max(1.0, abs(r["loss"]))
    assert_close(g0, r["grads"], TOL[prec], "grads")


def test_batch_ring_equals_explicit_staging():
    """vcnn_net_set_batch_ring: graph-replayed steps that stage the ring's
    next batch themselves (device cursor, wrapping) train bit-identically to
    explicit load_batch + step over the same batches; a host-stream call in
    between keeps the ring (and its position) for the steps after it."""
    spec, B, nb, steps = S.cifar3(), 32, 3, 7
    x, cls, _ = O.synth_bench_data(spec, B * nb, 8)
    xp = torch.from_numpy(x.reshape(nb, B, -1)).cuda()
    cp = torch.from_numpy(cls.reshape(nb, B).astype(np.int32)).cuda()
    a, b = Network(spec, B), Network(spec, B)
    a.enable_graph(True)
    b.enable_graph(True)
    a.set_batch_ring(xp, cp)
    for i in range(steps):
        a.train_step(B, 0.01, 0.9)
        b.load_batch(xp[i % nb], cls=cp[i % nb])
        b.train_step(B, 0.01, 0.9)
        assert a.loss() == b.loss(), i
    assert np.array_equal(a.get_params(), b.get_params())
    xs = torch.from_numpy(x.reshape(nb, B, -1)).pin_memory()
    cs = torch.from_numpy(cls.reshape(nb, B).astype(np.int32)).pin_memory()
    la = a.train_host_stream(xs, cls=cs, lr=0.01, momentum=0.9)
    lb = b.train_host_stream(xs, cls=cs, lr=0.01, momentum=0.9)
    assert np.array_equal(la, lb)
    a.train_step(B, 0.01, 0.9)  # ring resumes at batch steps % nb
    b.load_batch(xp[steps % nb], cls=cp[steps % nb])
    b.train_step(B, 0.01, 0.9)
    assert np.array_equal(a.get_params(), b.get_params())
    a.set_batch_ring()
    a.close()
    b.close()


def test_train_steps_multi_step_graphs_equal_single_steps():
    """vcnn_net_train_steps (up to 8 steps per graph launch, each staging its
    ring batch) trains bit-identically to single graph-replayed steps."""
    spec, B, nb = S.cifar3(), 32, 4
    x, cls, _ = O.synth_bench_data(spec, B * nb, 8)
    xp = torch.from_numpy(x.reshape(nb, B, -1)).cuda()
    cp = torch.from_numpy(cls.reshape(nb, B).astype(np.int32)).cuda()
    a, b = Network(spec, B), Network(spec, B)
    for n in (a, b):
        n.enable_graph(True)
        n.set_batch_ring(xp, cp)
    a.train_steps(11, B, 0.01, 0.9)  # chunks of 8 + 3
    for _ in range(11):
        b.train_step(B, 0.01, 0.9)
    assert a.loss() == b.loss()
    assert np.array_equal(a.get_params(), b.get_params())
    a.close()
    b.close()


def test_host_stream_equals_host_steps():
    """vcnn_net_train_host_stream (H2D of batch i+1 on a copy stream while
    step i computes) gives bit-identical losses and weights to the same
    batches fed one synchronous vcnn_net_train_step_host at a time; class
    bounds are validated like the host step."""
    spec, B, steps = S.cifar3(), 32, 5
    x, cls, _ = O.synth_bench_data(spec, B * steps, 8)
    xs = torch.from_numpy(x.reshape(steps, B, -1)).pin_memory()
    cs = torch.from_numpy(cls.reshape(steps, B).astype(np.int32)).pin_memory()
    a, b = Network(spec, B), Network(spec, B)
    la = a.train_host_stream(xs, cls=cs, lr=0.01, momentum=0.9)
    lb = np.array([b.train_step_host(x.reshape(steps, B, -1)[i], cls=cls.reshape(steps, B)[i],
                                     lr=0.01, momentum=0.9) for i in range(steps)], np.float32)
    assert np.array_equal(la, lb)
    assert np.array_equal(a.get_params(), b.get_params())
    bad = cs.clone()
    bad[3, 7] = 10
    with pytest.raises(BoundsError):
        a.train_host_stream(xs, cls=bad, lr=0.01, momentum=0.9)
    a.close()
    b.close()
