"""ctypes wrapper over the parity checker -- TEST INFRASTRUCTURE ONLY.

Loads oracle/liboracle.so (the C restatement, vcnn_oracle.c) and, when built,
oracle/_ref/libvcnn_ref_*.so (the reference compiled from its own sources).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product package never does.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")


class OrcLayer(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("kind", "units", "kh", "kw", "stride", "pool_mode", "pool_bias", "act")]


class OrcNet(C.Structure):
    _fields_ = [("in_h", C.c_int), ("in_w", C.c_int), ("in_c", C.c_int), ("nlayers", C.c_int),
                ("layers", C.POINTER(OrcLayer)), ("loss", C.c_int), ("seed", C.c_uint64)]


def make_net(spec):
    """OrcNet from a NetworkSpec-like object (duck-typed: .input, .layers, .loss,
    .seed; layers are converted with paper_1501_07338_b200.spec.layer_fields
    semantics)."""
    arr = (OrcLayer * max(1, len(spec.layers)))()
    for i, L in enumerate(spec.layers):
        arr[i] = OrcLayer(*_layer_fields(L))
    n = OrcNet(spec.input[0], spec.input[1], spec.input[2], len(spec.layers),
               C.cast(arr, C.POINTER(OrcLayer)), int(spec.loss), int(spec.seed))
    n._keep = arr
    return n


def _layer_fields(L):
    name = type(L).__name__
    if name == "ConvSpec":
        return (0, L.maps, L.kh, L.kw, L.stride, 0, 0, int(L.act))
    if name == "PoolSpec":
        return (1, 0, L.ph, L.pw, L.stride, int(L.mode), int(bool(L.bias)), int(L.act))
    return (2, L.units, 0, 0, 1, 0, 0, int(L.act))


def _dp(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


_orc = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.check_call(["make", "-s", "-C", HERE, os.path.join(HERE, "liboracle.so")])
        L = C.CDLL(ORACLE_SO)
        for name in dir(L):
            pass
        L.orc_net_num_params.restype = C.c_int64
        L.orc_net_trace_size.restype = C.c_int64
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_uniform_range.restype = C.c_double
        L.orc_rng_next_u64.restype = C.c_uint64
        L.orc_activate.restype = C.c_double
        L.orc_activate.argtypes = [C.c_int, C.c_double]
        L.orc_activation_grad_from_output.restype = C.c_double
        L.orc_activation_grad_from_output.argtypes = [C.c_int, C.c_double]
        L.orc_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.orc_rng_fill_uniform.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                           C.c_double]
        L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_sgd_step.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                   C.c_double]
        L.orc_matmul.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p]
        L.orc_matmul_transB.argtypes = L.orc_matmul.argtypes
        L.orc_synth_bench_data.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        _orc = L
    return _orc


class OrcError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def _chk(st, what):
    if st:
        raise OrcError(st, what)


# ---------------------------------------------------------------- rng
class OrcRng:
    def __init__(self, seed):
        self._buf = C.create_string_buffer(312 * 8 + 64)
        orc().orc_rng_seed(self._buf, seed)

    def uniform(self, lo=0.0, hi=1.0):
        return orc().orc_rng_uniform_range(self._buf, lo, hi)

    def uniform_int(self, n):
        return orc().orc_rng_uniform_int(self._buf, n)

    def fill(self, n, lo=0.0, hi=1.0):
        out = np.empty(n, dtype=np.float64)
        orc().orc_rng_fill_uniform(self._buf, _dp(out), n, lo, hi)
        return out


# ---------------------------------------------------------------- ops (double)
def conv_out(n, k, s):
    return (n - k) // s + 1 if s > 0 and k <= n else 1


def im2col(x, kh, kw, s):
    B, Cc, H, W = x.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    OH, OW = conv_out(H, kh, s), conv_out(W, kw, s)
    P = np.empty((Cc * kh * kw, B * OH * OW))
    _chk(orc().orc_im2col(B, Cc, H, W, kh, kw, s, _dp(x), _dp(P)), "im2col")
    return P


def col2im_map(B, Cc, H, W, kh, kw, s):
    OH, OW = conv_out(H, kh, s), conv_out(W, kw, s)
    n = Cc * kh * kw * B * OH * OW
    src = np.empty(n, dtype=np.int64)
    tgt = np.empty(n, dtype=np.int64)
    _chk(orc().orc_col2im_map(B, Cc, H, W, kh, kw, s, _dp(src), _dp(tgt)), "col2im_map")
    return src, tgt


def col2im(dP, B, Cc, H, W, kh, kw, s):
    dP = np.ascontiguousarray(dP, dtype=np.float64)
    dX = np.empty((B, Cc, H, W))
    _chk(orc().orc_col2im(B, Cc, H, W, kh, kw, s, _dp(dP), _dp(dX)), "col2im")
    return dX


def pool_map(B, Cc, H, W, ph, pw, s):
    OH, OW = conv_out(H, ph, s), conv_out(W, pw, s)
    n = B * Cc * OH * OW * ph * pw
    src = np.empty(n, dtype=np.int64)
    tgt = np.empty(n, dtype=np.int64)
    _chk(orc().orc_pool_map(B, Cc, H, W, ph, pw, s, _dp(src), _dp(tgt)), "pool_map")
    return src, tgt


def pool_forward(x, ph, pw, s, mode):
    B, Cc, H, W = x.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    OH, OW = conv_out(H, ph, s), conv_out(W, pw, s)
    y = np.empty((B, Cc, OH, OW))
    arg = np.empty((B, Cc, OH, OW), dtype=np.int64)
    _chk(orc().orc_pool_forward(B, Cc, H, W, ph, pw, s, int(mode), _dp(x), _dp(y), _dp(arg)),
         "pool_forward")
    return y, arg


def pool_backward(dy, arg, in_shape, ph, pw, s, mode, bwd_mode=0):
    B, Cc, H, W = in_shape
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    arg = np.ascontiguousarray(arg if arg is not None else np.full(dy.shape, -1), dtype=np.int64)
    dx = np.empty((B, Cc, H, W))
    _chk(orc().orc_pool_backward(B, Cc, H, W, ph, pw, s, int(mode), int(bwd_mode), _dp(dy),
                                 _dp(arg), _dp(dx)), "pool_backward")
    return dx


def matmul(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]))
    orc().orc_matmul(a.shape[0], a.shape[1], b.shape[1], _dp(a), _dp(b), _dp(c))
    return c


def matmul_transB(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[0]))
    orc().orc_matmul_transB(a.shape[0], a.shape[1], b.shape[0], _dp(a), _dp(b), _dp(c))
    return c


def conv_forward(x, w, b, kh, kw, s, act):
    B, Cc, H, W = x.shape
    K = w.shape[0]
    x, w, b = (np.ascontiguousarray(t, dtype=np.float64) for t in (x, w, b))
    y = np.empty((B, K, conv_out(H, kh, s), conv_out(W, kw, s)))
    _chk(orc().orc_conv_forward(B, Cc, H, W, K, kh, kw, s, int(act), _dp(x), _dp(w), _dp(b),
                                _dp(y)), "conv_forward")
    return y


def conv_backward(x, w, y, dy, kh, kw, s, act, need_dx=True):
    B, Cc, H, W = x.shape
    K = w.shape[0]
    x, w, y, dy = (np.ascontiguousarray(t, dtype=np.float64) for t in (x, w, y, dy))
    dw = np.empty(w.shape)
    db = np.empty(K)
    dx = np.empty(x.shape) if need_dx else None
    _chk(orc().orc_conv_backward(B, Cc, H, W, K, kh, kw, s, int(act), _dp(x), _dp(w), _dp(y),
                                 _dp(dy), _dp(dw), _dp(db), _dp(dx)), "conv_backward")
    return dw, db, dx


def full_forward(x, w, b, act):
    B = x.shape[0]
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(B, -1)
    w, b = (np.ascontiguousarray(t, dtype=np.float64) for t in (w, b))
    y = np.empty((B, w.shape[0]))
    _chk(orc().orc_full_forward(B, x.shape[1], w.shape[0], int(act), _dp(x), _dp(w), _dp(b),
                                _dp(y)), "full_forward")
    return y


def full_backward(x, w, y, dy, act, need_dx=True):
    B = x.shape[0]
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(B, -1)
    w, y, dy = (np.ascontiguousarray(t, dtype=np.float64) for t in (w, y, dy))
    dw = np.empty(w.shape)
    db = np.empty(w.shape[0])
    dx = np.empty(x.shape) if need_dx else None
    _chk(orc().orc_full_backward(B, x.shape[1], w.shape[0], int(act), _dp(x), _dp(w), _dp(y),
                                 _dp(dy), _dp(dw), _dp(db), _dp(dx)), "full_backward")
    return dw, db, dx


def loss_forward(kind, pred, cls=None, values=None):
    B = pred.shape[0]
    pred = np.ascontiguousarray(pred, dtype=np.float64).reshape(B, -1)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(B, -1) if values is not None else None
    out = C.c_double()
    _chk(orc().orc_loss_forward(int(kind), B, pred.shape[1], _dp(pred), _dp(c), _dp(v),
                                C.byref(out)), "loss_forward")
    return out.value


def loss_backward(kind, pred, cls=None, values=None):
    B = pred.shape[0]
    pred = np.ascontiguousarray(pred, dtype=np.float64).reshape(B, -1)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(B, -1) if values is not None else None
    g = np.empty(pred.shape)
    _chk(orc().orc_loss_backward(int(kind), B, pred.shape[1], _dp(pred), _dp(c), _dp(v), _dp(g)),
         "loss_backward")
    return g


def activate(act, x):
    f = np.vectorize(lambda v: orc().orc_activate(int(act), float(v)))
    return f(np.asarray(x, dtype=np.float64))


# ------------------------------------------- numpy (BLAS f64) restatement
# The same conv_forward / conv_backward (layers.hpp:139-195) through numpy's
# f64 GEMM, for the full-size parity checks (BASELINE shapes: 16x16 / 121-tap
# kernels, 256-channel sweep cells) where the scalar C restatement would take
# minutes.  Pinned against the C restatement in tests/test_oracle_golden.py.
def _act_np(act, x):
    act = int(act)
    if act == 1:
        return np.where(x > 0, x, 0.0)
    if act == 2:
        return 1.0 / (1.0 + np.exp(-x))
    if act == 3:
        return np.tanh(x)
    return x


def _act_grad_np(act, y):
    act = int(act)
    if act == 1:
        return (y > 0).astype(np.float64)
    if act == 2:
        return y * (1 - y)
    if act == 3:
        return 1 - y * y
    return np.ones_like(y)


def _patches_np(x, kh, kw, s):
    """im2col (vectorize.hpp:54-79) as rows: [B*OH*OW][C*kh*kw], (c,ky,kx) order."""
    from numpy.lib.stride_tricks import sliding_window_view
    v = sliding_window_view(x, (kh, kw), axis=(2, 3))[:, :, ::s, ::s]  # B,C,OH,OW,kh,kw
    B, Cc, OH, OW = v.shape[:4]
    return v.transpose(0, 2, 3, 1, 4, 5).reshape(B * OH * OW, Cc * kh * kw), OH, OW


def _chunk(x, kh, kw):
    """images per chunk so one chunk's patch matrix stays under ~256 MB."""
    B, Cc, H, W = x.shape
    per = 8 * Cc * kh * kw * H * W
    return max(1, min(B, (256 << 20) // max(per, 1)))


def conv_forward_np(x, w, b, kh, kw, s, act):
    x = np.asarray(x, dtype=np.float64)
    B = x.shape[0]
    K = w.shape[0]
    wt = np.asarray(w, np.float64).reshape(K, -1).T
    b = np.asarray(b, np.float64)
    outs = []
    cb = _chunk(x, kh, kw)
    for i in range(0, B, cb):
        xi = x[i:i + cb]
        P, OH, OW = _patches_np(xi, kh, kw, s)
        Z = P @ wt + b
        outs.append(Z.reshape(xi.shape[0], OH, OW, K).transpose(0, 3, 1, 2))
    return _act_np(act, np.concatenate(outs))


def conv_backward_np(x, w, y, dy, kh, kw, s, act, need_dx=True):
    """(dW [K][C*kh*kw], db [K], dX or None); dy is the gradient of the
    post-activation output y (act' taken from y, layers.hpp:39-48)."""
    x = np.asarray(x, dtype=np.float64)
    B, Cc, H, W = x.shape
    K = w.shape[0]
    w = np.asarray(w, np.float64).reshape(K, -1)
    G = np.asarray(dy, np.float64) * _act_grad_np(act, np.asarray(y, np.float64))
    OH, OW = G.shape[2], G.shape[3]
    dw = np.zeros((K, Cc * kh * kw))
    db = np.zeros(K)
    dx = np.zeros_like(x) if need_dx else None
    cb = _chunk(x, kh, kw)
    for i in range(0, B, cb):
        n = min(cb, B - i)
        Gm = G[i:i + n].transpose(0, 2, 3, 1).reshape(-1, K)
        P, _, _ = _patches_np(x[i:i + n], kh, kw, s)
        dw += Gm.T @ P
        db += Gm.sum(axis=0)
        if need_dx:
            dP = (Gm @ w).reshape(n, OH, OW, Cc, kh, kw)
            for ky in range(kh):
                for kx in range(kw):
                    dx[i:i + n, :, ky:ky + s * (OH - 1) + 1:s, kx:kx + s * (OW - 1) + 1:s] += \
                        dP[:, :, :, :, ky, kx].transpose(0, 3, 1, 2)
    return dw, db, dx


# ---------------------------------------------------------------- network
def net_num_params(spec):
    return orc().orc_net_num_params(C.byref(make_net(spec)))


def net_init(spec):
    n = make_net(spec)
    p = np.empty(orc().orc_net_num_params(C.byref(n)))
    _chk(orc().orc_net_init(C.byref(n), _dp(p)), "net_init")
    return p


def net_run_batch(spec, params, x, cls=None, values=None, pool_bwd_mode=0, grads=True,
                  trace=False):
    """Executor<double>(imp6).run_batch restated.  Returns dict(out, loss, grads,
    trace, args)."""
    n = make_net(spec)
    B = x.shape[0]
    x = np.ascontiguousarray(x, dtype=np.float64)
    params = np.ascontiguousarray(params, dtype=np.float64)
    units = spec.output_units()
    out = np.empty((B, units))
    g = np.empty(params.size) if grads else None
    loss = C.c_double(0)
    tr = np.empty(orc().orc_net_trace_size(C.byref(n), B)) if trace else None
    npool = sum(1 for L in spec.layers if type(L).__name__ == "PoolSpec")
    args = None
    if trace and npool:
        chain = spec.chain()
        sz = sum(B * h * w * c for (h, w, c), L in zip(chain, spec.layers)
                 if type(L).__name__ == "PoolSpec")
        args = np.empty(sz, dtype=np.int64)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64) if values is not None else None
    _chk(orc().orc_net_run_batch(C.byref(n), B, _dp(params), _dp(x), _dp(c), _dp(v),
                                 int(pool_bwd_mode), int(bool(grads)), _dp(out), C.byref(loss),
                                 _dp(g), _dp(tr), _dp(args)), "net_run_batch")
    return {"out": out, "loss": loss.value, "grads": g, "trace": tr, "args": args}


def sgd_step(w, v, g, lr, mom):
    orc().orc_sgd_step(w.size, _dp(w), _dp(v), _dp(g), lr, mom)


def synth_bench_data(spec, B, seed):
    n = make_net(spec)
    x = np.empty((B,) + (spec.input[2], spec.input[0], spec.input[1]), dtype=np.float32)
    units = spec.output_units()
    cls = np.zeros(B, dtype=np.int32)
    vals = np.zeros((B, units), dtype=np.float32)
    _chk(orc().orc_synth_bench_data(C.byref(n), B, seed, _dp(x), _dp(cls), _dp(vals)),
         "synth_bench_data")
    return x, cls, vals


# ---------------------------------------------------------------- reference itself
def _cpu_has_avx512():
    try:
        with open("/proc/cpuinfo") as f:
            return "avx512f" in f.read()
    except OSError:
        return False


def ref_path():
    """Path of the reference library compiled from /root/reference (or None)."""
    for v in (("v4", "v3") if _cpu_has_avx512() else ("v3",)):
        p = os.path.join(REF_DIR, f"libvcnn_ref_{v}.so")
        if os.path.exists(p):
            return p
    return None


_ref = None


def ref():
    """The reference's own code (oracle/_ref), or None when not built."""
    global _ref
    if _ref is None:
        p = ref_path()
        if p is None:
            return None
        L = C.CDLL(p)
        L.ref_bench_create.restype = C.c_void_p
        L.ref_bench_create.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_double]
        L.ref_bench_set_variant.argtypes = [C.c_void_p, C.c_int]
        L.ref_bench_step.restype = C.c_float
        L.ref_bench_step.argtypes = [C.c_void_p, C.c_int]
        L.ref_bench_get_params.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_bench_destroy.argtypes = [C.c_void_p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_fill_uniform.argtypes = [C.c_uint64, C.c_void_p, C.c_int64, C.c_double,
                                           C.c_double]
        L.ref_rng_fill_uniform_int.argtypes = [C.c_uint64, C.c_void_p, C.c_int64, C.c_int]
        L.ref_net_train_steps.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                          C.c_int, C.c_void_p]
        L.ref_save_model.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p]
        L.ref_load_model_f32.argtypes = [C.c_char_p, C.c_void_p, C.c_int64]
        L.ref_net_train_steps_f32.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                              C.c_int, C.c_void_p]
        L.ref_synth_bench_data.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        L.ref_fit.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                              C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
        _ref = L
    return _ref


def ref_net_init(spec):
    n = make_net(spec)
    p = np.empty(orc().orc_net_num_params(C.byref(n)))
    _chk(ref().ref_net_init(C.byref(n), _dp(p)), "ref_net_init")
    return p


def ref_net_run_batch(spec, params, x, cls=None, values=None, pool_bwd_mode=0, variant=6,
                      grads=True):
    n = make_net(spec)
    B = x.shape[0]
    x = np.ascontiguousarray(x, dtype=np.float64)
    params = np.ascontiguousarray(params, dtype=np.float64)
    out = np.empty((B, spec.output_units()))
    g = np.empty(params.size)
    loss = C.c_double(0)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64) if values is not None else None
    _chk(ref().ref_net_run_batch(C.byref(n), variant, B, _dp(params), _dp(x), _dp(c), _dp(v),
                                 int(pool_bwd_mode), int(bool(grads)), _dp(out), C.byref(loss),
                                 _dp(g)), "ref_net_run_batch")
    return {"out": out, "loss": loss.value, "grads": g if grads else None}


def ref_net_train_steps(spec, params, x, cls, values, lr, mom, steps):
    n = make_net(spec)
    B = x.shape[0]
    p = np.ascontiguousarray(params, dtype=np.float64).copy()
    x = np.ascontiguousarray(x, dtype=np.float64)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64) if values is not None else None
    losses = np.empty(steps)
    _chk(ref().ref_net_train_steps(C.byref(n), B, _dp(p), _dp(x), _dp(c), _dp(v), lr, mom, steps,
                                   _dp(losses)), "ref_net_train_steps")
    return p, losses


def ref_net_train_steps_f32(spec, params, x, cls, values, lr, mom, steps):
    """The reference's own float Executor<float>(imp6) + sgd_step trajectory."""
    n = make_net(spec)
    B = x.shape[0]
    p = np.ascontiguousarray(params, dtype=np.float32).copy()
    x = np.ascontiguousarray(x, dtype=np.float32)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float32) if values is not None else None
    losses = np.empty(steps)
    _chk(ref().ref_net_train_steps_f32(C.byref(n), B, p.ctypes.data, x.ctypes.data,
                                       _dp(c), None if v is None else v.ctypes.data, lr, mom,
                                       steps, _dp(losses)), "ref_net_train_steps_f32")
    return p, losses


def ref_fit(spec, params, x, cls, values, lr, mom, batch, epochs, seed, f32=False):
    """The reference's Trainer<T>(cfg).fit + evaluate_accuracy
    (training.hpp:50-107): (final params, epoch losses, accuracy or None)."""
    n = make_net(spec)
    count = x.shape[0]
    p = np.ascontiguousarray(params, dtype=np.float64).copy()
    x = np.ascontiguousarray(x, dtype=np.float64)
    c = np.ascontiguousarray(cls, dtype=np.int32) if cls is not None else None
    v = np.ascontiguousarray(values, dtype=np.float64) if values is not None else None
    el = np.empty(epochs)
    acc = C.c_double(-1.0)
    _chk(ref().ref_fit(C.byref(n), count, _dp(p), _dp(x), _dp(c), _dp(v), lr, mom, batch,
                       epochs, seed, int(bool(f32)), _dp(el), C.byref(acc)), "ref_fit")
    return p, el, (acc.value if cls is not None else None)


def ref_save_model(spec, params, path, f32=True):
    """The reference's save_model(model_from_network(net)) (io.cpp:265-307)."""
    n = make_net(spec)
    p = np.ascontiguousarray(params, dtype=np.float64)
    _chk(ref().ref_save_model(C.byref(n), _dp(p), int(bool(f32)), path.encode()),
         "ref_save_model")


def ref_load_model_f32(path, count):
    """The reference's load_model + network_from_model<float> (io.cpp:309-404)."""
    out = np.empty(count, dtype=np.float32)
    _chk(ref().ref_load_model_f32(path.encode(), out.ctypes.data, count), "ref_load_model")
    return out
