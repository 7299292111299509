"""Pin the oracle (CPU, no GPU): the C restatement must reproduce
  (1) the known-answer vectors of the reference's own doctest suites, and
  (2) the reference itself -- via the committed fixtures made from oracle/_ref
      (tests/golden/make_golden.py) and, when oracle/_ref is built here, live.
"""
import glob
import math
import os

import numpy as np
import pytest

import oracle_py as O
from paper_1501_07338_b200 import spec as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
A = S.Activation


def rel_err(a, b):  # helpers.hpp:21-25
    scale = max(abs(a), abs(b))
    return 0.0 if scale < 1e-14 else abs(a - b) / scale


# ---------------------------------------------------------------- (1) known answers
def test_im2col_golden_matrix():  # vectorize_test.cpp:9-17
    f = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    P = O.im2col(f, 2, 2, 1)
    want = np.array([[1, 2, 4, 5], [2, 3, 5, 6], [4, 5, 7, 8], [5, 6, 8, 9]], dtype=np.float64)
    assert np.array_equal(P.T, want)


def test_im2col_degenerate():  # vectorize_test.cpp:19-38
    f = np.random.default_rng(3).uniform(-1, 1, (1, 1, 4, 5))
    assert np.array_equal(O.im2col(f, 1, 1, 1).ravel(), f.ravel())
    assert np.array_equal(O.im2col(f, 4, 5, 1).ravel(), f.ravel())
    with pytest.raises(O.OrcError) as e:
        O.im2col(f, 5, 5, 1)
    assert e.value.status == 2  # GeometryError
    with pytest.raises(O.OrcError):
        O.im2col(f, 2, 2, 0)


def test_col2im_membership_counts():  # vectorize_test.cpp:40-46
    dX = O.col2im(np.ones((4, 4)), 1, 1, 3, 3, 2, 2, 1)
    assert list(dX.ravel()) == [1, 2, 1, 2, 4, 2, 1, 2, 1]


def test_col2im_identity_and_zero():  # vectorize_test.cpp:48-60
    f = np.random.default_rng(4).uniform(-1, 1, (2, 2, 3, 4))
    P = O.im2col(f, 1, 1, 1)
    assert np.array_equal(O.col2im(P, 2, 2, 3, 4, 1, 1, 1), f)
    assert not O.col2im(np.zeros((8, 9)), 1, 2, 4, 4, 2, 2, 1).any()


def test_adjoint_identity_120_geometries():  # vectorize_test.cpp:70-91
    rng = S.Rng(42)
    for _ in range(120):
        h, w = 2 + rng.uniform_int(7), 2 + rng.uniform_int(7)
        c, b = 1 + rng.uniform_int(3), 1 + rng.uniform_int(3)
        kh, kw = 1 + rng.uniform_int(h), 1 + rng.uniform_int(w)
        s = 1 + rng.uniform_int(2)
        f = np.array([rng.uniform(-1, 1) for _ in range(h * w * c * b)]).reshape(b, c, h, w)
        P = O.im2col(f, kh, kw, s)
        g = np.array([rng.uniform(-1, 1) for _ in range(P.size)]).reshape(P.shape)
        lhs = float((P * g).sum())
        rhs = float((f * O.col2im(g, b, c, h, w, kh, kw, s)).sum())
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def test_pool_golden():  # vectorize_test.cpp:149-172
    f = np.arange(1, 17, dtype=np.float64).reshape(1, 1, 4, 4)
    y, arg = O.pool_forward(f, 2, 2, 2, 0)
    assert list(y.ravel()) == [6, 8, 14, 16]
    assert list(arg.ravel()) == [5, 7, 13, 15]
    y, _ = O.pool_forward(f, 2, 2, 2, 1)
    assert list(y.ravel()) == [3.5, 5.5, 11.5, 13.5]
    y, _ = O.pool_forward(f, 1, 1, 1, 0)
    assert np.array_equal(y, f)


def test_pool_ties_lowest_index():  # vectorize_test.cpp:192-198, tensor_test.cpp:203-209
    y, arg = O.pool_forward(np.full((1, 1, 2, 2), 7.0), 2, 2, 1, 0)
    assert y.ravel()[0] == 7 and arg.ravel()[0] == 0


def test_pool_backward_examples():  # vectorize_test.cpp:200-225
    assert list(O.pool_backward(np.array([[[[4.0]]]]), None, (1, 1, 2, 2), 2, 2, 1, 1).ravel()) \
        == [1, 1, 1, 1]
    assert list(O.pool_backward(np.array([[[[1.0]]]]), np.array([[[[3]]]]), (1, 1, 2, 2), 2, 2, 1,
                                0).ravel()) == [0, 0, 0, 1]
    assert list(O.pool_backward(np.array([[[[3.25]]]]), None, (1, 1, 2, 2), 2, 2, 1, 1,
                                bwd_mode=1).ravel()) == [3.25] * 4


def test_pool_map_geometry():  # vectorize_test.cpp:117-147, :227-239
    src, tgt = O.pool_map(1, 1, 4, 4, 2, 2, 2)
    assert len(src) == 16 and np.bincount(tgt).tolist() == [4, 4, 4, 4]
    src, tgt = O.pool_map(1, 1, 3, 3, 2, 2, 1)
    assert len(src) == 16 and int((src == 4).sum()) == 4
    assert len(set(zip(src.tolist(), tgt.tolist()))) == len(src)


def test_pool_vs_brute_force_60():  # vectorize_test.cpp:174-190
    rng = S.Rng(44)
    for _ in range(60):
        h, w = 2 + rng.uniform_int(7), 2 + rng.uniform_int(7)
        c, b = 1 + rng.uniform_int(3), 1 + rng.uniform_int(3)
        ph, pw = min(1 + rng.uniform_int(3), h), min(1 + rng.uniform_int(3), w)
        s = 1 + rng.uniform_int(2)
        mode = 0 if rng.uniform_int(2) else 1
        f = np.array([rng.uniform(-1, 1) for _ in range(h * w * c * b)]).reshape(b, c, h, w)
        y, _ = O.pool_forward(f, ph, pw, s, 1 - mode if False else (0 if mode == 0 else 1))
        oh, ow = (h - ph) // s + 1, (w - pw) // s + 1
        ref = np.empty((b, c, oh, ow))
        for yy in range(oh):
            for xx in range(ow):
                win = f[:, :, yy * s:yy * s + ph, xx * s:xx * s + pw]
                ref[:, :, yy, xx] = win.max(axis=(2, 3)) if mode == 0 else win.mean(axis=(2, 3))
        assert np.abs(y - ref).max() < 1e-12


def test_matmul_hand_values():  # tensor_test.cpp:37-42
    c = O.matmul(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0], [6.0]]))
    assert list(c.ravel()) == [17, 39]
    ct = O.matmul_transB(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0]]))
    assert list(ct.ravel()) == [17, 39]


def test_conv_hand_examples():  # layers_test.cpp:48-63
    f = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    y = O.conv_forward(f, np.array([[1.0, 0, 0, 0]]), np.array([0.0]), 2, 2, 1, 0)
    assert list(y.ravel()) == [1, 2, 4, 5]
    y = O.conv_forward(np.array([[[[1.0, 2], [3, 4]]]]), np.array([[0.25] * 4]), np.zeros(1), 2,
                       2, 1, 0)
    assert list(y.ravel()) == [2.5]


def test_conv_backward_1x1():  # layers_test.cpp:95-105
    f = np.array([[[[1.0, 2], [3, 4]]]])
    w = np.array([[2.0]])
    y = O.conv_forward(f, w, np.zeros(1), 1, 1, 1, 0)
    go = np.array([[[[0.5, 1.0], [-1.0, 2.0]]]])
    dw, db, dx = O.conv_backward(f, w, y, go, 1, 1, 1, 0)
    assert math.isclose(dw.ravel()[0], 0.5 * 1 + 1.0 * 2 - 1.0 * 3 + 2.0 * 4)
    assert math.isclose(db[0], 0.5 + 1.0 - 1.0 + 2.0)
    assert list(dx.ravel()) == [1.0, 2.0, -2.0, 4.0]


def test_conv_vs_brute_25():  # layers_test.cpp:71-81 (brute_conv, helpers.hpp:43-63)
    rng = np.random.default_rng(21)
    for _ in range(25):
        B = 1 + int(rng.integers(3))
        x = rng.uniform(-1, 1, (B, 3, 6, 6))
        w = rng.uniform(-0.5, 0.5, (3, 27))
        b = rng.uniform(-0.1, 0.1, 3)
        y = O.conv_forward(x, w, b, 3, 3, 1, 1)
        ref = np.zeros((B, 3, 4, 4))
        wr = w.reshape(3, 3, 3, 3)
        for yy in range(4):
            for xx in range(4):
                ref[:, :, yy, xx] = np.einsum("bcij,kcij->bk", x[:, :, yy:yy + 3, xx:xx + 3], wr) + b
        assert np.abs(y - np.maximum(ref, 0)).max() < 1e-10


def test_loss_ln10_and_mse_zero():  # layers_test.cpp:216-230
    assert abs(O.loss_forward(0, np.zeros((1, 10)), cls=[3]) - math.log(10)) < 1e-12
    v = np.random.default_rng(1).uniform(size=(2, 5))
    assert O.loss_forward(1, v, values=v) == 0.0
    with pytest.raises(O.OrcError) as e:
        O.loss_forward(0, np.zeros((1, 10)), cls=[10])
    assert e.value.status == 3  # BoundsError


def test_loss_shift_invariance_and_fd():  # layers_test.cpp:231-272
    rng = np.random.default_rng(2)
    l = rng.uniform(-2, 2, (3, 7))
    cls = [1, 6, 0]
    a = O.loss_forward(0, l, cls=cls)
    assert abs(a - O.loss_forward(0, l + 5.0, cls=cls)) < 1e-12
    g = O.loss_backward(0, l, cls=cls)
    h = 1e-6
    for i in range(3):
        for u in range(7):
            lp, lm = l.copy(), l.copy()
            lp[i, u] += h
            lm[i, u] -= h
            num = (O.loss_forward(0, lp, cls=cls) - O.loss_forward(0, lm, cls=cls)) / (2 * h)
            assert rel_err(num, g[i, u]) < 1e-6 or abs(num - g[i, u]) < 1e-9


def test_sgd_examples():  # network_test.cpp:162-196
    w, v, g = np.array([1.0]), np.zeros(1), np.array([2.0])
    O.sgd_step(w, v, g, 0.1, 0.0)
    assert math.isclose(w[0], 0.8)
    w, v, g = np.array([0.0]), np.zeros(1), np.array([1.0])
    O.sgd_step(w, v, g, 0.1, 0.5)
    O.sgd_step(w, v, g, 0.1, 0.5)
    assert math.isclose(w[0], -0.25)


def test_whole_net_finite_differences():  # network_test.cpp:207-217 (fd_check, helpers.hpp:109-142)
    spec = S.NetworkSpec((4, 4, 1), [S.ConvSpec(2, 2, 2, 1, A.tanh),
                                     S.PoolSpec(2, 2, 1, S.PoolMode.avg),
                                     S.FullSpec(2, A.identity)], S.LossKind.softmax_ce, 3)
    p = O.net_init(spec)
    x = np.random.default_rng(59).uniform(0.05, 0.95, (2, 1, 4, 4))
    cls = [0, 1]
    r = O.net_run_batch(spec, p, x, cls=cls)
    h, worst = 1e-5, 0.0
    for k in range(p.size):
        pp, pm = p.copy(), p.copy()
        pp[k] += h
        pm[k] -= h
        lp = O.net_run_batch(spec, pp, x, cls=cls)["loss"]
        lm = O.net_run_batch(spec, pm, x, cls=cls)["loss"]
        num = (lp - lm) / (2 * h)
        worst = max(worst, abs(num - r["grads"][k]) / max(abs(num), abs(r["grads"][k]), 1e-6))
    assert worst < 1e-4


def test_batch_equivalence():  # network_test.cpp:99-160
    spec = S.NetworkSpec((9, 10, 2), [S.ConvSpec(3, 3, 2, 1, A.tanh),
                                      S.PoolSpec(2, 2, 1, S.PoolMode.max, True, A.sigmoid),
                                      S.FullSpec(3, A.identity)], S.LossKind.softmax_ce, 5)
    p = O.net_init(spec)
    x = np.random.default_rng(7).uniform(-1, 1, (4, 2, 9, 10))
    cls = [0, 2, 1, 1]
    whole = O.net_run_batch(spec, p, x, cls=cls)
    acc = np.zeros_like(whole["grads"])
    loss = 0.0
    for b in range(4):
        r = O.net_run_batch(spec, p, x[b:b + 1], cls=cls[b:b + 1])
        assert np.abs(r["out"][0] - whole["out"][b]).max() < 1e-10
        acc += r["grads"]
        loss += r["loss"]
    assert abs(whole["loss"] - loss / 4) < 1e-10
    assert np.abs(whole["grads"] - acc / 4).max() < 1e-10


def test_rng_matches_reference_stream():  # common.hpp:58-66 via fixture from oracle/_ref
    d = np.load(os.path.join(GOLD, "ops.npz"))
    r = O.OrcRng(8)
    assert np.array_equal(r.fill(64), d["rng8_uniform"])
    r = O.OrcRng(9)
    assert [r.uniform_int(10) for _ in range(64)] == d["rng9_uniform_int10"].tolist()
    pr = S.Rng(8)
    assert [pr.uniform() for _ in range(64)] == d["rng8_uniform"].tolist()


# ---------------------------------------------------------------- (2) vs the reference itself
def test_ops_vs_reference_fixtures():
    d = np.load(os.path.join(GOLD, "ops.npz"))
    gi = 0
    while f"conv{gi}_geom" in d:
        B, Cc, H, W, kh, kw, s = d[f"conv{gi}_geom"].tolist()
        assert np.array_equal(O.im2col(d[f"conv{gi}_x"], kh, kw, s), d[f"conv{gi}_P"])
        src, tgt = O.col2im_map(B, Cc, H, W, kh, kw, s)
        assert np.array_equal(src, d[f"conv{gi}_src"]) and np.array_equal(tgt, d[f"conv{gi}_tgt"])
        assert np.array_equal(O.col2im(d[f"conv{gi}_dP"], B, Cc, H, W, kh, kw, s),
                              d[f"conv{gi}_dX"])
        gi += 1
    gi = 0
    while f"pool{gi}_geom" in d:
        B, Cc, H, W, ph, pw, s, mode = d[f"pool{gi}_geom"].tolist()
        y, arg = O.pool_forward(d[f"pool{gi}_x"], ph, pw, s, mode)
        assert np.array_equal(y, d[f"pool{gi}_y"])
        if mode == 0:
            assert np.array_equal(arg, d[f"pool{gi}_arg"])
        for bm, key in ((0, "exact"), (1, "paper_nn")):
            dx = O.pool_backward(d[f"pool{gi}_dy"], d[f"pool{gi}_arg"] if mode == 0 else None,
                                 (B, Cc, H, W), ph, pw, s, mode, bwd_mode=bm)
            assert np.allclose(dx, d[f"pool{gi}_dx_{key}"], rtol=0, atol=1e-15)
        src, tgt = O.pool_map(B, Cc, H, W, ph, pw, s)
        assert np.array_equal(src, d[f"pool{gi}_src"]) and np.array_equal(tgt, d[f"pool{gi}_tgt"])
        gi += 1


def _fixture_nets():
    from golden.make_golden import small_nets  # noqa
    return small_nets()


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "net_*.npz"))),
                         ids=lambda p: os.path.basename(p)[4:-4])
def test_net_vs_reference_fixture(path):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    name = os.path.basename(path)[4:-4]
    spec, B = _fixture_nets()[name]
    d = np.load(path)
    p0 = O.net_init(spec)
    assert np.array_equal(p0, d["params0"])  # build_network bit-exact (Glorot stream)
    kw = dict(cls=d["cls"]) if spec.loss == S.LossKind.softmax_ce else dict(values=d["values"])
    x = d["x"].astype(np.float64)
    r = O.net_run_batch(spec, p0, x, **kw)
    tol = 1e-12
    assert np.abs(r["out"] - d["out"]).max() <= tol * max(1, np.abs(d["out"]).max())
    assert abs(r["loss"] - float(d["loss"])) <= tol
    assert np.abs(r["grads"] - d["grads"]).max() <= tol * max(1, np.abs(d["grads"]).max())
    rn = O.net_run_batch(spec, p0, x, pool_bwd_mode=1, **kw)
    assert np.abs(rn["grads"] - d["grads_paper_nn"]).max() <= tol * max(
        1, np.abs(d["grads_paper_nn"]).max())
    # N steps of run_batch + sgd_step
    p, v = p0.copy(), np.zeros_like(p0)
    for _ in range(int(d["steps"])):
        g = O.net_run_batch(spec, p, x, **kw)["grads"]
        O.sgd_step(p, v, g, float(d["lr"]), float(d["mom"]))
    assert np.abs(p - d["params_after"]).max() <= 1e-11


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (reference sources absent)")
def test_oracle_vs_live_reference_random_nets():
    """helpers.hpp random_net_spec family: 20 random nets, oracle vs reference."""
    rng = S.Rng(2024)
    for _ in range(20):
        h, w, c = 6 + rng.uniform_int(5), 6 + rng.uniform_int(5), 1 + rng.uniform_int(3)
        layers = []
        ch, cw = h, w
        acts = list(A)
        for _i in range(1 + rng.uniform_int(2)):
            if ch < 3 or cw < 3:
                break
            cs = S.ConvSpec(1 + rng.uniform_int(4), min(2 + rng.uniform_int(2), ch),
                            min(2 + rng.uniform_int(2), cw), 1 + rng.uniform_int(2),
                            acts[rng.uniform_int(4)])
            layers.append(cs)
            ch, cw = (ch - cs.kh) // cs.stride + 1, (cw - cs.kw) // cs.stride + 1
            if ch >= 2 and cw >= 2 and rng.uniform_int(2):
                ps = S.PoolSpec(2, 2, 1 + rng.uniform_int(2),
                                S.PoolMode.max if rng.uniform_int(2) else S.PoolMode.avg,
                                rng.uniform_int(3) == 0,
                                acts[rng.uniform_int(4)] if rng.uniform_int(3) == 0 else A.identity)
                layers.append(ps)
                ch, cw = (ch - 2) // ps.stride + 1, (cw - 2) // ps.stride + 1
        layers.append(S.FullSpec(2 + rng.uniform_int(5), acts[rng.uniform_int(4)]))
        loss = S.LossKind.mse if rng.uniform_int(4) == 0 else S.LossKind.softmax_ce
        if loss == S.LossKind.mse:
            layers[-1].act = A.identity
        spec = S.NetworkSpec((h, w, c), layers, loss, rng.next_u64() & 0xFFFF)
        B = 1 + rng.uniform_int(4)
        p = O.net_init(spec)
        assert np.array_equal(p, O.ref_net_init(spec))
        x = np.array([rng.uniform(-1, 1) for _ in range(B * h * w * c)]).reshape(B, c, h, w)
        units = spec.output_units()
        if loss == S.LossKind.softmax_ce:
            kw = dict(cls=[rng.uniform_int(units) for _ in range(B)])
        else:
            kw = dict(values=np.array([rng.uniform(-1, 1) for _ in range(B * units)]))
        for pm in (0, 1):
            a = O.net_run_batch(spec, p, x, pool_bwd_mode=pm, **kw)
            b = O.ref_net_run_batch(spec, p, x, pool_bwd_mode=pm, **kw)
            assert np.abs(a["out"] - b["out"]).max() <= 1e-12
            assert abs(a["loss"] - b["loss"]) <= 1e-12
            assert np.abs(a["grads"] - b["grads"]).max() <= 1e-12 * max(1, np.abs(b["grads"]).max())


def test_numpy_conv_restatement_equals_c_oracle():
    """oracle_py.conv_*_np (BLAS f64, used for the full-size GPU parity
    checks) == the C restatement on 30 random geometries (incl. stride)."""
    rng = np.random.default_rng(11)
    for _ in range(30):
        B, Cc = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        kh, kw, s = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 3))
        Hh, W = kh + int(rng.integers(0, 7)), kw + int(rng.integers(0, 7))
        K, act = int(rng.integers(1, 6)), int(rng.integers(0, 4))
        x = rng.uniform(-1, 1, (B, Cc, Hh, W))
        w = rng.uniform(-1, 1, (K, Cc * kh * kw))
        b = rng.uniform(-1, 1, K)
        y = O.conv_forward(x, w, b, kh, kw, s, act)
        assert np.abs(O.conv_forward_np(x, w, b, kh, kw, s, act) - y).max() <= 1e-12
        dy = rng.uniform(-1, 1, y.shape)
        ref = O.conv_backward(x, w, y, dy, kh, kw, s, act)
        got = O.conv_backward_np(x, w, y, dy, kh, kw, s, act)
        for a, r in zip(got, ref):
            assert np.abs(a - r).max() <= 1e-12 * max(1.0, np.abs(r).max())


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (reference sources absent)")
def test_ref_fit_equals_restated_loop():
    """The reference's Trainer<double>::fit (ref_fit, training.hpp:60-88) ==
    the restated loop: Rng(seed) shuffle carried across epochs, smaller last
    batch, run_batch + sgd_step per batch, mean epoch loss."""
    spec = S.NetworkSpec((8, 8, 1), [S.ConvSpec(3, 3, 3, 1, A.relu), S.PoolSpec(2, 2, 2),
                                     S.FullSpec(4, A.identity)], S.LossKind.softmax_ce, 3)
    n, batch, epochs, seed = 11, 4, 3, 9
    rng = np.random.default_rng(2)
    x = rng.uniform(0, 1, (n, 1, 8, 8))
    cls = rng.integers(0, 4, n).astype(np.int32)
    p0 = O.net_init(spec)
    pr, el, acc = O.ref_fit(spec, p0, x, cls, None, 0.05, 0.9, batch, epochs, seed)
    p, v = p0.copy(), np.zeros_like(p0)
    r, order, losses = S.Rng(seed), list(range(n)), []
    for _ in range(epochs):
        r.shuffle(order)
        tot, nb = 0.0, 0
        for st in range(0, n, batch):
            ids = order[st:st + batch]
            res = O.net_run_batch(spec, p, x[ids], cls=cls[ids])
            O.sgd_step(p, v, res["grads"], 0.05, 0.9)
            tot += res["loss"]
            nb += 1
        losses.append(tot / nb)
    assert np.abs(pr - p).max() <= 1e-12 and np.abs(el - losses).max() <= 1e-12
    out = O.net_run_batch(spec, p, x, grads=False)["out"]
    assert acc == np.mean(np.argmax(out, axis=1) == cls)
