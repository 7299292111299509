"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs the reference compiled from its own sources (oracle/_ref, built by
oracle/Makefile from /root/reference/proj) -- never the restatement -- on
small seeded cases and stores inputs + outputs as .npz.  The fixtures travel
with the repo, so parity tests on the GPU box (where /root/reference does not
exist) still compare against the reference's own numbers.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ctypes as C  # noqa: E402

import oracle_py as O  # noqa: E402
from paper_1501_07338_b200 import spec as S  # noqa: E402

A = S.Activation


def small_nets():
    """Small networks covering every layer kind, activation, pool mode, pool
    bias, overlap, stride and both losses (the helpers.hpp random_net_spec
    families, fixed here)."""
    return {
        "cifar3_b4": (S.cifar3(), 4),
        "lenet_mini_b3": (S.NetworkSpec((28, 28, 1), [S.ConvSpec(4, 5, 5, 1, A.relu),
                                                     S.PoolSpec(2, 2, 2),
                                                     S.ConvSpec(6, 5, 5, 1, A.relu),
                                                     S.PoolSpec(2, 2, 2),
                                                     S.FullSpec(20, A.relu),
                                                     S.FullSpec(10, A.identity)],
                                        S.LossKind.softmax_ce, 10), 3),
        "denoise_small_b2": (S.NetworkSpec((20, 20, 1), [S.ConvSpec(8, 6, 6, 1, A.relu),
                                                        S.ConvSpec(8, 1, 1, 1, A.relu),
                                                        S.ConvSpec(1, 3, 3, 1, A.identity)],
                                           S.LossKind.mse, 11), 2),
        "deconv_small_b2": (S.NetworkSpec((30, 30, 1), [S.ConvSpec(6, 11, 1, 1, A.identity),
                                                       S.ConvSpec(6, 1, 11, 1, A.relu),
                                                       S.ConvSpec(1, 3, 3, 1, A.identity)],
                                          S.LossKind.mse, 12), 2),
        "mixed_b3": (S.NetworkSpec((9, 10, 2), [S.ConvSpec(3, 3, 2, 1, A.tanh),
                                              S.PoolSpec(2, 2, 1, S.PoolMode.max, True, A.sigmoid),
                                              S.ConvSpec(4, 2, 3, 2, A.sigmoid),
                                              S.PoolSpec(2, 2, 1, S.PoolMode.avg, True, A.tanh),
                                              S.FullSpec(5, A.tanh), S.FullSpec(3, A.identity)],
                                 S.LossKind.softmax_ce, 13), 3),
        "avgpool_mse_b2": (S.NetworkSpec((8, 8, 1), [S.ConvSpec(2, 3, 3, 1, A.relu),
                                                    S.PoolSpec(2, 2, 2, S.PoolMode.avg),
                                                    S.FullSpec(4, A.identity)],
                                       S.LossKind.mse, 14), 2),
        "single_conv_b2": (S.single_conv(8, 3, 10, 15), 2),
    }


def make_net_fixture(name, spec, B, steps=3, lr=0.01, mom=0.9):
    x, cls, vals = O.synth_bench_data(spec, B, 8)          # bench.cpp:29-45 stream
    p0 = O.ref_net_init(spec)                              # build_network<double>
    kw = dict(cls=cls) if spec.loss == S.LossKind.softmax_ce else dict(values=vals)
    r = O.ref_net_run_batch(spec, p0, x.astype(np.float64), **kw)
    rnn = O.ref_net_run_batch(spec, p0, x.astype(np.float64), pool_bwd_mode=1, **kw)
    pN, losses = O.ref_net_train_steps(spec, p0, x.astype(np.float64), kw.get("cls"),
                                       kw.get("values"), lr, mom, steps)
    np.savez_compressed(os.path.join(HERE, f"net_{name}.npz"), x=x, cls=cls, values=vals,
                        params0=p0, out=r["out"], loss=r["loss"], grads=r["grads"],
                        grads_paper_nn=rnn["grads"], params_after=pN, losses=losses,
                        steps=steps, lr=lr, mom=mom, batch=B)


def make_op_fixtures():
    R = O.ref()
    rng = np.random.default_rng(5)
    geoms = [(2, 3, 7, 6, 3, 2, 1), (1, 2, 9, 9, 3, 3, 2), (3, 1, 5, 8, 5, 1, 1),
             (2, 2, 6, 6, 1, 1, 1)]
    out = {}
    for gi, (B, Cc, H, W, kh, kw, s) in enumerate(geoms):
        x = rng.uniform(-1, 1, (B, Cc, H, W))
        OH, OW = (H - kh) // s + 1, (W - kw) // s + 1
        P = np.empty((Cc * kh * kw, B * OH * OW))
        R.ref_im2col(B, Cc, H, W, kh, kw, s, x.ctypes.data_as(C.c_void_p),
                     P.ctypes.data_as(C.c_void_p))
        n = P.size
        src = np.empty(n, np.int64)
        tgt = np.empty(n, np.int64)
        R.ref_col2im_map(B, Cc, H, W, kh, kw, s, src.ctypes.data_as(C.c_void_p),
                         tgt.ctypes.data_as(C.c_void_p))
        dP = rng.uniform(-1, 1, P.shape)
        dX = np.empty(x.shape)
        R.ref_col2im(B, Cc, H, W, kh, kw, s, dP.ctypes.data_as(C.c_void_p),
                     dX.ctypes.data_as(C.c_void_p))
        out.update({f"conv{gi}_geom": np.array([B, Cc, H, W, kh, kw, s]), f"conv{gi}_x": x,
                    f"conv{gi}_P": P, f"conv{gi}_src": src, f"conv{gi}_tgt": tgt,
                    f"conv{gi}_dP": dP, f"conv{gi}_dX": dX})
    pgeoms = [(2, 3, 6, 6, 2, 2, 2, 0), (1, 2, 5, 7, 2, 3, 1, 0), (2, 1, 6, 5, 3, 2, 1, 1),
              (1, 2, 4, 4, 2, 2, 2, 1)]
    for gi, (B, Cc, H, W, ph, pw, s, mode) in enumerate(pgeoms):
        # integer-valued inputs with many ties exercise the lowest-index rule
        x = rng.integers(0, 4, (B, Cc, H, W)).astype(np.float64)
        OH, OW = (H - ph) // s + 1, (W - pw) // s + 1
        y = np.empty((B, Cc, OH, OW))
        arg = np.empty((B, Cc, OH, OW), np.int64)
        R.ref_pool_forward(B, Cc, H, W, ph, pw, s, mode, x.ctypes.data_as(C.c_void_p),
                           y.ctypes.data_as(C.c_void_p), arg.ctypes.data_as(C.c_void_p))
        dy = rng.uniform(-1, 1, y.shape)
        dxs = {}
        for bm in (0, 1):
            dx = np.empty(x.shape)
            R.ref_pool_backward(B, Cc, H, W, ph, pw, s, mode, bm, dy.ctypes.data_as(C.c_void_p),
                                arg.ctypes.data_as(C.c_void_p), dx.ctypes.data_as(C.c_void_p))
            dxs[bm] = dx
        n = B * Cc * OH * OW * ph * pw
        src = np.empty(n, np.int64)
        tgt = np.empty(n, np.int64)
        R.ref_pool_map(B, Cc, H, W, ph, pw, s, src.ctypes.data_as(C.c_void_p),
                       tgt.ctypes.data_as(C.c_void_p))
        out.update({f"pool{gi}_geom": np.array([B, Cc, H, W, ph, pw, s, mode]),
                    f"pool{gi}_x": x, f"pool{gi}_y": y, f"pool{gi}_arg": arg,
                    f"pool{gi}_dy": dy, f"pool{gi}_dx_exact": dxs[0],
                    f"pool{gi}_dx_paper_nn": dxs[1], f"pool{gi}_src": src,
                    f"pool{gi}_tgt": tgt})
    # the Rng stream (common.hpp:58-66)
    u = np.empty(64)
    R.ref_rng_fill_uniform(8, u.ctypes.data_as(C.c_void_p), 64, 0.0, 1.0)
    ui = np.empty(64, np.int32)
    R.ref_rng_fill_uniform_int(9, ui.ctypes.data_as(C.c_void_p), 64, 10)
    out.update({"rng8_uniform": u, "rng9_uniform_int10": ui})
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)


def main():
    if O.ref() is None:
        raise SystemExit("oracle/_ref not built: run `make -C oracle` with /root/reference present")
    make_op_fixtures()
    for name, (spec, B) in small_nets().items():
        make_net_fixture(name, spec, B)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
