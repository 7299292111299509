"""Per-layer / per-op error report of the device engine vs the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py as O  # noqa
from paper_1501_07338_b200 import ops, spec as S  # noqa
from paper_1501_07338_b200.engine import Network  # noqa


def nw(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def T(a, dt=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def H(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


rng = np.random.default_rng(3)
for (B, Cc, Hh, W, K, kh, kw, s) in [(4, 3, 32, 32, 32, 5, 5, 1), (4, 32, 14, 14, 32, 5, 5, 1),
                                      (2, 2, 6, 6, 16, 3, 3, 1), (1, 1, 8, 8, 16, 3, 3, 1)]:
    x = rng.uniform(0, 1, (B, Cc, Hh, W)).astype(np.float32)
    w = rng.uniform(-0.2, 0.2, (K, Cc * kh * kw)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, K).astype(np.float32)
    for prec in S.Precision:
        y = ops.conv_forward(T(x), T(w), T(b), kh, kw, s, S.Activation.identity, prec)
        yr = O.conv_forward(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64), kh,
                            kw, s, 0)
        dy = rng.uniform(-1, 1, yr.shape).astype(np.float32)
        dw, db, dx = ops.conv_backward(T(x), T(w), y, T(dy), kh, kw, s, S.Activation.identity,
                                       prec)
        rdw, rdb, rdx = O.conv_backward(x.astype(np.float64), w.astype(np.float64), yr,
                                        dy.astype(np.float64), kh, kw, s, 0)
        print(f"conv {B}x{Cc}x{Hh}x{W} K{K} k{kh}x{kw} {prec.name:7s}: fwd {nw(H(y), yr):.2e} "
              f"dW {nw(H(dw), rdw):.2e} db {nw(H(db), rdb):.2e} dX {nw(H(dx), rdx):.2e}")
        if prec == S.Precision.tf32 and nw(H(dw), rdw) > 1e-2:
            e = np.abs(H(dw) - rdw)
            print("   dW err by row(n):", np.round(e.max(axis=1), 4)[:8])
            print("   dW err by col(k):", np.round(e.max(axis=0), 4)[:12])
            print("   gpu", H(dw)[0, :6], "\n   ref", rdw[0, :6])

spec = S.cifar3()
B = 4
x, cls, _ = O.synth_bench_data(spec, B, 8)
for prec in S.Precision:
    net = Network(spec, B, prec)
    net.load_batch(T(x.reshape(B, -1)), cls=T(cls, torch.int32))
    net.forward_backward(B)
    p0 = net.get_params().astype(np.float64)
    r = O.net_run_batch(spec, p0, x.astype(np.float64), cls=cls, trace=True)
    g = net.get_grads()
    msg = [f"loss {net.loss():.6f}/{r['loss']:.6f}"]
    for i in range(len(spec.layers)):
        gw, gb = net.layer_params(g, i)
        rw, rb = net.layer_params(r["grads"], i)
        if rw.size:
            msg.append(f"L{i} dW {nw(gw, rw):.1e} db {nw(gb, rb):.1e}")
    print(prec.name, " | ".join(msg))
    net.close()
