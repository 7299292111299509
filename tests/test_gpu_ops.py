"""Op-level parity on the B200: every kernel through the C ABI vs the oracle
(double precision on the same fp32 inputs).  Index maps and argmax are
compared bit-exactly; floating-point results normwise with the tolerance of
the precision mode (tests/util.py: TF32 1e-3, 3xTF32 / FP32 1e-5)."""
import os

import numpy as np
import pytest
import torch

import oracle_py as O
from paper_1501_07338_b200 import ops
from paper_1501_07338_b200.errors import BoundsError, GeometryError, ShapeError
from paper_1501_07338_b200.spec import Activation as A, LossKind, PoolMode, Precision

from .util import ALL_PREC, TOL, assert_close, f32

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
dev = torch.device("cuda")


def T(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)


def H(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


CONV_GEOMS = [  # (B, C, H, W, K, kh, kw, s)
    (4, 3, 32, 32, 32, 5, 5, 1),    # CIFAR3 conv1
    (4, 32, 14, 14, 32, 5, 5, 1),   # CIFAR3 conv2
    (4, 32, 5, 5, 64, 5, 5, 1),     # CIFAR3 conv3 (1x1 output)
    (3, 1, 28, 28, 20, 5, 5, 1),    # LeNet conv1
    (3, 20, 12, 12, 50, 5, 5, 1),   # LeNet conv2
    (2, 1, 40, 40, 16, 16, 16, 1),  # denoise-style 16x16 kernel
    (2, 1, 64, 30, 6, 121 // 4, 1, 1),  # long 1-D vertical kernel
    (2, 6, 20, 64, 5, 1, 33, 1),    # long 1-D horizontal kernel
    (2, 3, 9, 11, 4, 3, 2, 2),      # stride 2, rectangular
    (3, 2, 7, 7, 3, 1, 1, 1),       # 1x1
    (1, 5, 6, 6, 300, 3, 3, 1),     # N > 256: two N tiles
]


@pytest.mark.parametrize("g", CONV_GEOMS, ids=lambda g: "x".join(map(str, g)))
def test_im2col_col2im_and_map(g):
    B, Cc, Hh, W, K, kh, kw, s = g
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (B, Cc, Hh, W)).astype(np.float32)
    P = H(ops.im2col(T(x), kh, kw, s))
    assert np.array_equal(P, O.im2col(x.astype(np.float64), kh, kw, s).astype(np.float32))
    geom = ops.conv_geometry(Hh, W, Cc, B, kh, kw, s)
    if P.size <= 4_000_000:
        src, tgt = ops.build_col2im_map(geom)
        osrc, otgt = O.col2im_map(B, Cc, Hh, W, kh, kw, s)
        assert np.array_equal(H(src), osrc) and np.array_equal(H(tgt), otgt)  # bit-exact
    dP = rng.uniform(-1, 1, P.shape).astype(np.float32)
    dX = H(ops.col2im(T(dP), geom))
    assert_close(dX, O.col2im(f32(dP), B, Cc, Hh, W, kh, kw, s), 1e-6, "col2im")


def test_ops_vs_reference_fixture():
    """Maps / pooling vs numbers produced by the reference itself (oracle/_ref)."""
    d = np.load(os.path.join(GOLD, "ops.npz"))
    gi = 0
    while f"conv{gi}_geom" in d:
        B, Cc, Hh, W, kh, kw, s = d[f"conv{gi}_geom"].tolist()
        geom = ops.conv_geometry(Hh, W, Cc, B, kh, kw, s)
        src, tgt = ops.build_col2im_map(geom)
        assert np.array_equal(H(src), d[f"conv{gi}_src"])
        assert np.array_equal(H(tgt), d[f"conv{gi}_tgt"])
        P = H(ops.im2col(T(d[f"conv{gi}_x"]), kh, kw, s))
        assert np.array_equal(P, d[f"conv{gi}_P"].astype(np.float32))
        gi += 1
    gi = 0
    while f"pool{gi}_geom" in d:
        B, Cc, Hh, W, ph, pw, s, mode = d[f"pool{gi}_geom"].tolist()
        y, arg = ops.pool_forward(T(d[f"pool{gi}_x"]), ph, pw, s, PoolMode(mode))
        assert np.array_equal(H(y), d[f"pool{gi}_y"].astype(np.float32))
        if mode == 0:
            assert np.array_equal(H(arg), d[f"pool{gi}_arg"])  # ties -> lowest index
        geom = ops.pool_geometry(Hh, W, Cc, B, ph, pw, s, PoolMode(mode))
        src, tgt = ops.build_pool_map(geom)
        assert np.array_equal(H(src), d[f"pool{gi}_src"])
        assert np.array_equal(H(tgt), d[f"pool{gi}_tgt"])
        for bm, key in ((0, "exact"), (1, "paper_nn")):
            dx = ops.pool_backward(T(d[f"pool{gi}_dy"]), geom,
                                   T(d[f"pool{gi}_arg"], torch.int64) if mode == 0 else None, bm)
            assert_close(H(dx), d[f"pool{gi}_dx_{key}"], 1e-6, f"pool_backward {key}")
        gi += 1


POOL_GEOMS = [(4, 32, 28, 28, 2, 2, 2), (3, 20, 24, 24, 2, 2, 2), (2, 3, 9, 9, 3, 3, 1),
              (2, 2, 7, 8, 2, 3, 2), (1, 4, 5, 5, 5, 5, 1), (2, 3, 6, 6, 1, 1, 1)]


@pytest.mark.parametrize("mode", [PoolMode.max, PoolMode.avg])
@pytest.mark.parametrize("g", POOL_GEOMS, ids=lambda g: "x".join(map(str, g)))
def test_pool(g, mode):
    B, Cc, Hh, W, ph, pw, s = g
    rng = np.random.default_rng(2)
    x = rng.integers(-3, 4, (B, Cc, Hh, W)).astype(np.float32)  # many ties
    y, arg = ops.pool_forward(T(x), ph, pw, s, mode)
    oy, oarg = O.pool_forward(x.astype(np.float64), ph, pw, s, int(mode))
    if mode == PoolMode.max:
        assert np.array_equal(H(y), oy.astype(np.float32))
        assert np.array_equal(H(arg), oarg)  # bit-exact int64 ArgIndex
    else:
        assert_close(H(y), oy, 1e-6, "avg pool")
    geom = ops.pool_geometry(Hh, W, Cc, B, ph, pw, s, mode)
    dy = rng.uniform(-1, 1, oy.shape).astype(np.float32)
    for bm in (0, 1):
        dx = ops.pool_backward(T(dy), geom, arg, bm)
        ref = O.pool_backward(f32(dy), oarg if mode == PoolMode.max else None, (B, Cc, Hh, W), ph,
                              pw, s, int(mode), bm)
        assert_close(H(dx), ref, 1e-6, f"pool_backward mode={bm}")


def test_pool_nan_and_ties():
    x = np.array([[[[7, 7], [7, 7]]]], dtype=np.float32)
    y, arg = ops.pool_forward(T(x), 2, 2, 1)
    assert H(arg).ravel()[0] == 0 and H(y).ravel()[0] == 7
    x = np.array([[[[np.nan, 5], [1, 2]]]], dtype=np.float32)  # NaN first: kept
    y, arg = ops.pool_forward(T(x), 2, 2, 1)
    assert np.isnan(H(y).ravel()[0]) and H(arg).ravel()[0] == 0
    x = np.array([[[[1, np.nan], [5, 2]]]], dtype=np.float32)  # NaN later: skipped
    y, arg = ops.pool_forward(T(x), 2, 2, 1)
    assert H(y).ravel()[0] == 5 and H(arg).ravel()[0] == 2


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
@pytest.mark.parametrize("g", CONV_GEOMS, ids=lambda g: "x".join(map(str, g)))
def test_conv_forward_backward(g, prec):
    B, Cc, Hh, W, K, kh, kw, s = g
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (B, Cc, Hh, W)).astype(np.float32)
    a = np.sqrt(6.0 / (Cc * kh * kw + K * kh * kw))
    w = rng.uniform(-a, a, (K, Cc * kh * kw)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, K).astype(np.float32)
    for act in (A.relu, A.tanh):
        y = ops.conv_forward(T(x), T(w), T(b), kh, kw, s, act, prec)
        yr = O.conv_forward(f32(x), f32(w), f32(b), kh, kw, s, int(act))
        assert_close(H(y), yr, TOL[prec], f"conv fwd {prec.name} {act.name}")
        # backward from the GPU's own forward output (the trace the engine keeps)
        yh = H(y)
        dy = rng.uniform(-1, 1, yr.shape).astype(np.float32)
        dw, db, dx = ops.conv_backward(T(x), T(w), y, T(dy), kh, kw, s, act, prec)
        rdw, rdb, rdx = O.conv_backward(f32(x), f32(w), f32(yh), f32(dy), kh, kw, s, int(act))
        assert_close(H(dw), rdw, TOL[prec], f"conv dW {prec.name}")
        assert_close(H(db), rdb, TOL[prec], f"conv db {prec.name}")
        assert_close(H(dx), rdx, TOL[prec], f"conv dX {prec.name}")


FC_SHAPES = [(128, 64, 10), (100, 800, 500), (100, 500, 100), (3, 7, 5), (128, 1600, 300),
             (1, 300, 1)]


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
@pytest.mark.parametrize("shp", FC_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_full_forward_backward(shp, prec):
    B, n_in, n_out = shp
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (B, n_in)).astype(np.float32)
    a = np.sqrt(6.0 / (n_in + n_out))
    w = rng.uniform(-a, a, (n_out, n_in)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, n_out).astype(np.float32)
    for act in (A.relu, A.sigmoid, A.identity):
        y = ops.full_forward(T(x), T(w), T(b), act, prec)
        yr = O.full_forward(f32(x), f32(w), f32(b), int(act))
        assert_close(H(y), yr, TOL[prec], f"fc fwd {prec.name}")
        dy = rng.uniform(-1, 1, yr.shape).astype(np.float32)
        dw, db, dx = ops.full_backward(T(x), T(w), y, T(dy), act, prec)
        rdw, rdb, rdx = O.full_backward(f32(x), f32(w), f32(H(y)), f32(dy), int(act))
        assert_close(H(dw), rdw, TOL[prec], "fc dW")
        assert_close(H(db), rdb, TOL[prec], "fc db")
        assert_close(H(dx), rdx, TOL[prec], "fc dX")


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
def test_matmul(prec):
    c = H(ops.matmul(T([[1.0, 2.0], [3.0, 4.0]]), T([[5.0], [6.0]]), prec))
    assert c.ravel().tolist() == [17, 39]  # tensor_test.cpp:37-42 (exact in tf32 too)
    rng = np.random.default_rng(5)
    for (m, k, n) in [(37, 129, 61), (300, 64, 257), (5, 1000, 3)]:
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        assert_close(H(ops.matmul(T(a), T(b), prec)), O.matmul(f32(a), f32(b)), TOL[prec], "mm")
        bt = np.ascontiguousarray(b.T)
        assert_close(H(ops.matmul_transB(T(a), T(bt), prec)), O.matmul_transB(f32(a), f32(bt)),
                     TOL[prec], "mm_tB")


def test_loss():
    rng = np.random.default_rng(6)
    for B, units in [(128, 10), (100, 10), (7, 1000), (1, 3)]:
        l = rng.uniform(-3, 3, (B, units)).astype(np.float32)
        cls = rng.integers(0, units, B).astype(np.int32)
        lf = float(H(ops.loss_forward(LossKind.softmax_ce, T(l), cls)))
        assert abs(lf - O.loss_forward(0, f32(l), cls=cls)) <= 1e-5 * max(1, abs(lf))
        g = H(ops.loss_backward(LossKind.softmax_ce, T(l), cls))
        assert_close(g, O.loss_backward(0, f32(l), cls=cls), 1e-5, "ce grad")
        v = rng.uniform(0, 1, (B, units)).astype(np.float32)
        lm = float(H(ops.loss_forward(LossKind.mse, T(l), v)))
        assert abs(lm - O.loss_forward(1, f32(l), values=f32(v))) <= 1e-5 * abs(lm)
        gm = H(ops.loss_backward(LossKind.mse, T(l), v))
        assert_close(gm, O.loss_backward(1, f32(l), values=f32(v)), 1e-6, "mse grad")
    assert abs(float(H(ops.loss_forward(LossKind.softmax_ce, T(np.zeros((1, 10))), [3]))) -
               np.log(10)) < 1e-6  # layers_test.cpp:217-222
    with pytest.raises(BoundsError):
        ops.loss_forward(LossKind.softmax_ce, T(np.zeros((2, 10))), [1, 10])


def test_sgd():
    w, v, g = T([1.0]), T([0.0]), T([2.0])
    ops.sgd_step(w, v, g, 0.1, 0.0)
    assert abs(H(w)[0] - 0.8) < 1e-7  # network_test.cpp:162-177
    w, v, g = T([0.0]), T([0.0]), T([1.0])
    ops.sgd_step(w, v, g, 0.1, 0.5)
    ops.sgd_step(w, v, g, 0.1, 0.5)
    assert abs(H(w)[0] + 0.25) < 1e-7  # network_test.cpp:178-196
    rng = np.random.default_rng(7)
    n = 1_000_003
    w0, v0, g0 = (rng.uniform(-1, 1, n).astype(np.float32) for _ in range(3))
    w, v, g = T(w0), T(v0), T(g0)
    ops.sgd_step(w, v, g, 0.01, 0.9)
    vr = 0.9 * f32(v0) + f32(g0)
    assert_close(H(v), vr, 1e-6, "v")
    assert_close(H(w), f32(w0) - 0.01 * vr, 1e-6, "w")


def test_accumulate_by_index_and_max_arg():
    rng = np.random.default_rng(8)
    vals = rng.integers(-3, 4, 50).astype(np.float32)
    src = rng.integers(0, 50, 200)
    tgt = rng.integers(0, 17, 200)
    for red in ("sum", "mean", "max"):
        out = H(ops.accumulate_by_index(T(vals), T(src, torch.int64), T(tgt, torch.int64), 20, red))
        ref = np.zeros(20)
        for t in range(20):
            sel = vals[src[tgt == t]].astype(np.float64)
            if sel.size:
                ref[t] = sel.sum() if red == "sum" else sel.mean() if red == "mean" else sel.max()
        assert_close(out, ref, 1e-6, red)
    out, arg = ops.accumulate_max_arg(T(vals), T(src, torch.int64), T(tgt, torch.int64), 20)
    out, arg = H(out), H(arg)
    for t in range(20):
        s_t = src[tgt == t]
        if s_t.size == 0:
            assert arg[t] == -1 and out[t] == 0
        else:
            best = vals[s_t].max()
            assert out[t] == best and arg[t] == s_t[vals[s_t] == best].min()


def test_geometry_errors():
    with pytest.raises(GeometryError):
        ops.conv_geometry(4, 4, 1, 1, 5, 5, 1)
    with pytest.raises(GeometryError):
        ops.conv_geometry(4, 4, 1, 1, 2, 2, 0)
    with pytest.raises(GeometryError):
        ops.pool_geometry(2, 2, 1, 1, 3, 3, 1)
    with pytest.raises(ShapeError):
        ops.conv_forward(T(np.zeros((1, 3, 3, 3))), T(np.zeros((1, 4))), T(np.zeros(1)), 2, 2)


@pytest.mark.parametrize("prec", ALL_PREC, ids=lambda p: p.name)
def test_gemm_transposes_bias_act(prec):
    """vcnn_gemm: every trans_a / trans_b combination, bias + act
    epilogue, vs the oracle's matmul / matmul_transB on explicit transposes."""
    rng = np.random.default_rng(9)
    m, k, n = 37, 300, 45
    for ta in (False, True):
        for tb in (False, True):
            # pre-activations O(1) (a saturated tanh hides nothing but turns the
            # normwise error of the output into an absolute one)
            a = (rng.uniform(-1, 1, (k, m) if ta else (m, k)) * 3 / np.sqrt(k)).astype(np.float32)
            b = rng.uniform(-1, 1, (n, k) if tb else (k, n)).astype(np.float32)
            bias = rng.uniform(-1, 1, n).astype(np.float32)
            am = f32(a).T if ta else f32(a)
            bm = f32(b).T if tb else f32(b)
            ref = O.matmul(np.ascontiguousarray(am), np.ascontiguousarray(bm))
            for act in (A.identity, A.relu, A.tanh):
                c = ops.gemm(T(a), T(b), ta, tb, T(bias), act, prec)
                want = O.activate(act, ref + f32(bias))
                assert_close(H(c), want, TOL[prec], f"gemm ta={ta} tb={tb} {act.name}")
    c = ops.gemm(T([[1.0, 2.0], [3.0, 4.0]]), T([[5.0], [6.0]]), precision=prec)
    assert H(c).ravel().tolist() == [17, 39]
