"""Op-level API: the reference's free functions (proj/include/vcnn/
{tensor,vectorize,layers,network}.hpp) on CUDA tensors, each one C-ABI call
into libvcnn_cuda.so.  torch is used only to own device memory and to pick the
current stream; every arithmetic op runs in the library's sm_100a kernels.

Layouts follow the reference: feature maps NCHW ``[B][C][H][W]``
(tensor.hpp:80-82); conv weights ``[maps][C*kh*kw]`` with (c,ky,kx) flattening
(layers.hpp:68); FC weights ``[out][in]`` (layers.hpp:202); patch matrices
``[C*kh*kw][B*OH*OW]`` (vectorize.hpp:44-52).
"""
import ctypes as C

import torch

from ._lib import ConvGeometryC, PoolGeometryC, check, lib
from .errors import ShapeError
from .spec import Activation, LossKind, PoolBackwardMode, PoolMode, Precision

_REDUCERS = {"sum": 0, "max": 1, "mean": 2}


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _cuda(t, dtype=torch.float32, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ShapeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def _empty(*shape, dtype=torch.float32, device=None):
    return torch.empty(*shape, dtype=dtype, device=device or torch.device("cuda"))


# ---------------------------------------------------------------- geometry
def conv_geometry(in_h, in_w, channels, batch, kh, kw, stride) -> ConvGeometryC:
    """ConvGeometry(Shape, kh, kw, stride) (vectorize.hpp:19-29)."""
    g = ConvGeometryC()
    check(lib().vcnn_conv_geometry_init(C.byref(g), in_h, in_w, channels, batch, kh, kw, stride))
    return g


def pool_geometry(in_h, in_w, channels, batch, ph, pw, stride, mode=PoolMode.max) -> PoolGeometryC:
    """PoolGeometry(Shape, ph, pw, stride, mode) (vectorize.hpp:141-151)."""
    g = PoolGeometryC()
    check(lib().vcnn_pool_geometry_init(C.byref(g), in_h, in_w, channels, batch, ph, pw, stride,
                                        int(mode)))
    return g


def _geom_of(x, kh, kw, stride):
    if x.dim() != 4:
        raise ShapeError("feature map must be [B][C][H][W]")
    B, Cc, H, W = x.shape
    return conv_geometry(H, W, Cc, B, kh, kw, stride)


# ---------------------------------------------------------------- tensor.hpp
def matmul(a, b, precision=Precision.tf32):
    """matmul (tensor.hpp:131-150)."""
    a, b = _cuda(a, name="a"), _cuda(b, name="b")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul shape mismatch: {a.shape[0]}x{a.shape[1]} * "
                         f"{b.shape[0]}x{b.shape[1]}")
    c = _empty(a.shape[0], b.shape[1], device=a.device)
    check(lib().vcnn_matmul(a.shape[0], a.shape[1], b.shape[1], _p(a), _p(b), _p(c),
                            int(precision), _stream()))
    return c


def matmul_transB(a, b, precision=Precision.tf32):
    """matmul_transB (tensor.hpp:154-174)."""
    a, b = _cuda(a, name="a"), _cuda(b, name="b")
    if a.shape[1] != b.shape[1]:
        raise ShapeError(f"matmul_transB shape mismatch: {a.shape[0]}x{a.shape[1]} * "
                         f"{b.shape[0]}x{b.shape[1]}^T")
    c = _empty(a.shape[0], b.shape[0], device=a.device)
    check(lib().vcnn_matmul_transB(a.shape[0], a.shape[1], b.shape[0], _p(a), _p(b), _p(c),
                                   int(precision), _stream()))
    return c


def gemm(a, b, trans_a=False, trans_b=False, bias=None, act=Activation.identity,
         precision=Precision.tf32):
    """vcnn_gemm: act(op(a) @ op(b) + bias) (op = transpose when trans_*)."""
    a = _cuda(a, name="a")
    b = _cuda(b, name="b")
    m, k = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    kb, n = (b.shape[1], b.shape[0]) if trans_b else (b.shape[0], b.shape[1])
    if kb != k:
        raise ShapeError(f"gemm: inner extents {k} and {kb} differ")
    if bias is not None:
        bias = _cuda(bias, name="bias")
        if bias.numel() != n:
            raise ShapeError("gemm: bias must have n entries")
    c = _empty(m, n)
    check(lib().vcnn_gemm(int(trans_a), int(trans_b), m, n, k, _p(a), a.shape[1], _p(b),
                          b.shape[1], _p(c), n, _p(bias) if bias is not None else None,
                          int(act), int(precision), _stream()))
    return c


def accumulate_by_index(values, source, target, target_len, reducer="sum"):
    """accumulate_by_index (tensor.hpp:228-266)."""
    values = _cuda(values, name="values")
    source = _cuda(source, torch.int64, "source")
    target = _cuda(target, torch.int64, "target")
    out = _empty(int(target_len), device=values.device)
    check(lib().vcnn_accumulate_by_index(_p(values), values.numel(), _p(source), _p(target),
                                         source.numel(), int(target_len), _REDUCERS[reducer],
                                         _p(out), _stream()))
    return out


def accumulate_max_arg(values, source, target, target_len):
    """accumulate_max_arg (tensor.hpp:271-289)."""
    values = _cuda(values, name="values")
    source = _cuda(source, torch.int64, "source")
    target = _cuda(target, torch.int64, "target")
    out = _empty(int(target_len), device=values.device)
    arg = _empty(int(target_len), dtype=torch.int64, device=values.device)
    check(lib().vcnn_accumulate_max_arg(_p(values), values.numel(), _p(source), _p(target),
                                        source.numel(), int(target_len), _p(out), _p(arg),
                                        _stream()))
    return out, arg


# ------------------------------------------------------------- vectorize.hpp
def im2col(x, kh, kw, stride=1):
    """im2col (vectorize.hpp:54-79) -> patch matrix [C*kh*kw][B*OH*OW]."""
    x = _cuda(x, name="x")
    g = _geom_of(x, kh, kw, stride)
    P = _empty(g.channels * kh * kw, g.batch * g.out_h * g.out_w, device=x.device)
    check(lib().vcnn_im2col(C.byref(g), _p(x), _p(P), _stream()))
    return P


def col2im(dP, geom: ConvGeometryC):
    """col2im (vectorize.hpp:111-120): exact adjoint of im2col."""
    dP = _cuda(dP, name="grad")
    rows, cols = geom.channels * geom.kh * geom.kw, geom.batch * geom.out_h * geom.out_w
    from .errors import GeometryError
    if dP.dim() != 2 or dP.shape[0] != rows or dP.shape[1] != cols:
        raise GeometryError(f"col2im: gradient {tuple(dP.shape)} does not match geometry "
                            f"{rows}x{cols}")
    dX = _empty(geom.batch, geom.channels, geom.in_h, geom.in_w, device=dP.device)
    check(lib().vcnn_col2im(C.byref(geom), _p(dP), _p(dX), _stream()))
    return dX


def build_col2im_map(geom: ConvGeometryC, device="cuda"):
    """build_col2im_map (vectorize.hpp:84-106) -> (source, target) int64."""
    n = geom.channels * geom.kh * geom.kw * geom.batch * geom.out_h * geom.out_w
    src = _empty(n, dtype=torch.int64, device=device)
    tgt = _empty(n, dtype=torch.int64, device=device)
    check(lib().vcnn_col2im_map(C.byref(geom), _p(src), _p(tgt), _stream()))
    return src, tgt


def build_pool_map(geom: PoolGeometryC, device="cuda"):
    """build_pool_map (vectorize.hpp:167-191) -> (source, target) int64."""
    n = geom.channels * geom.batch * geom.out_h * geom.out_w * geom.ph * geom.pw
    src = _empty(n, dtype=torch.int64, device=device)
    tgt = _empty(n, dtype=torch.int64, device=device)
    check(lib().vcnn_pool_map(C.byref(geom), _p(src), _p(tgt), _stream()))
    return src, tgt


def pool_forward(x, ph, pw, stride, mode=PoolMode.max):
    """pool_forward (vectorize.hpp:197-215) -> (y, arg int64 | None)."""
    x = _cuda(x, name="x")
    B, Cc, H, W = x.shape
    g = pool_geometry(H, W, Cc, B, ph, pw, stride, mode)
    y = _empty(B, Cc, g.out_h, g.out_w, device=x.device)
    arg = _empty(B, Cc, g.out_h, g.out_w, dtype=torch.int64, device=x.device) \
        if mode == PoolMode.max else None
    check(lib().vcnn_pool_forward(C.byref(g), _p(x), _p(y), _p(arg), _stream()))
    return y, arg


def pool_backward(dy, geom: PoolGeometryC, arg, mode=PoolBackwardMode.exact):
    """pool_backward (vectorize.hpp:224-249)."""
    dy = _cuda(dy, name="grad")
    from .errors import GeometryError
    if tuple(dy.shape) != (geom.batch, geom.channels, geom.out_h, geom.out_w):
        raise GeometryError(f"pool_backward: gradient {tuple(dy.shape)} does not match pooled "
                            f"extents")
    arg = _cuda(arg, torch.int64, "arg") if arg is not None else None
    dx = _empty(geom.batch, geom.channels, geom.in_h, geom.in_w, device=dy.device)
    check(lib().vcnn_pool_backward(C.byref(geom), int(mode), _p(dy), _p(arg), _p(dx), _stream()))
    return dx


# ---------------------------------------------------------------- layers.hpp
def activation_forward(x, act):
    """apply_activation (layers.hpp:50-54)."""
    x = _cuda(x, name="x")
    y = torch.empty_like(x)
    check(lib().vcnn_activation_forward(x.numel(), int(act), _p(x), _p(y), _stream()))
    return y


def activation_backward(y, grad, act):
    """apply_activation_grad (layers.hpp:57-61): returns grad * act'(y)."""
    y, g = _cuda(y, name="y"), _cuda(grad, name="grad").clone()
    check(lib().vcnn_activation_backward(y.numel(), int(act), _p(y), _p(g), _stream()))
    return g


def conv_forward(x, w, b, kh, kw, stride=1, act=Activation.identity, precision=Precision.tf32):
    """conv_forward (layers.hpp:139-149): y = act(W * col(x) + b)."""
    x, w, b = _cuda(x, name="x"), _cuda(w, name="weights"), _cuda(b, name="bias")
    g = _geom_of(x, kh, kw, stride)
    maps = w.shape[0]
    if w.dim() != 2 or w.shape[1] != g.channels * kh * kw:
        raise ShapeError(f"conv layer: weight row length {w.shape[-1]} != kernel size "
                         f"{g.channels * kh * kw}")
    if b.numel() != maps:
        raise ShapeError("conv layer: bias length does not match kernel count")
    y = _empty(g.batch, maps, g.out_h, g.out_w, device=x.device)
    check(lib().vcnn_conv_forward(C.byref(g), maps, _p(x), _p(w), _p(b), int(act),
                                  int(precision), _p(y), _stream()))
    return y


def conv_backward(x, w, y, dy, kh, kw, stride=1, act=Activation.identity,
                  precision=Precision.tf32, need_dx=True):
    """conv_backward (layers.hpp:183-195) -> (dW, db, dX | None)."""
    x, w = _cuda(x, name="x"), _cuda(w, name="weights")
    y, dy = _cuda(y, name="y"), _cuda(dy, name="grad")
    g = _geom_of(x, kh, kw, stride)
    maps = w.shape[0]
    if tuple(dy.shape) != (g.batch, maps, g.out_h, g.out_w):
        raise ShapeError(f"conv_backward: gradient {tuple(dy.shape)} does not match forward "
                         f"output")
    dw = torch.empty_like(w)
    db = _empty(maps, device=x.device)
    dx = torch.empty_like(x) if need_dx else None
    check(lib().vcnn_conv_backward(C.byref(g), maps, _p(x), _p(w), _p(y), _p(dy), int(act),
                                   int(precision), _p(dw), _p(db), _p(dx), _stream()))
    return dw, db, dx


def full_forward(x, w, b, act=Activation.identity, precision=Precision.tf32):
    """full_forward (layers.hpp:230-247); x [B][...] flattens per sample."""
    x, w, b = _cuda(x, name="x"), _cuda(w, name="weights"), _cuda(b, name="bias")
    B = x.shape[0]
    per = x.numel() // B
    if per != w.shape[1]:
        raise ShapeError(f"full layer expects {w.shape[1]} inputs, got {per}")
    y = _empty(B, w.shape[0], device=x.device)
    check(lib().vcnn_full_forward(B, per, w.shape[0], _p(x), _p(w), _p(b), int(act),
                                  int(precision), _p(y), _stream()))
    return y


def full_backward(x, w, y, dy, act=Activation.identity, precision=Precision.tf32, need_dx=True):
    """full_backward (layers.hpp:269-278) -> (dW, db, dX | None)."""
    x, w = _cuda(x, name="x"), _cuda(w, name="weights")
    y, dy = _cuda(y, name="y"), _cuda(dy, name="grad")
    B = x.shape[0]
    per = x.numel() // B
    dw = torch.empty_like(w)
    db = _empty(w.shape[0], device=x.device)
    dx = torch.empty_like(x) if need_dx else None
    check(lib().vcnn_full_backward(B, per, w.shape[0], _p(x), _p(w), _p(y), _p(dy), int(act),
                                   int(precision), _p(dw), _p(db), _p(dx), _stream()))
    return dw, db, dx


def pool_layer_forward(x, ph, pw, stride, mode=PoolMode.max, bias=None, act=Activation.identity):
    """pool_layer_forward (layers.hpp:305-321) -> (y, arg | None)."""
    x = _cuda(x, name="x")
    bias = _cuda(bias, name="bias")
    B, Cc, H, W = x.shape
    g = pool_geometry(H, W, Cc, B, ph, pw, stride, mode)
    if bias is not None and bias.numel() != Cc:
        raise ShapeError(f"pool layer: bias length {bias.numel()} != channel count {Cc}")
    y = _empty(B, Cc, g.out_h, g.out_w, device=x.device)
    arg = _empty(B, Cc, g.out_h, g.out_w, dtype=torch.int64, device=x.device) \
        if mode == PoolMode.max else None
    check(lib().vcnn_pool_layer_forward(C.byref(g), _p(x), _p(bias), int(act), _p(y), _p(arg),
                                        _stream()))
    return y, arg


def pool_layer_backward(geom: PoolGeometryC, y, dy, arg, act=Activation.identity, has_bias=False,
                        mode=PoolBackwardMode.exact):
    """pool_layer_backward (layers.hpp:356-363) -> (dX, dbias | None)."""
    y, dy = _cuda(y, name="y"), _cuda(dy, name="grad")
    arg = _cuda(arg, torch.int64, "arg") if arg is not None else None
    dx = _empty(geom.batch, geom.channels, geom.in_h, geom.in_w, device=dy.device)
    dbias = _empty(geom.channels, device=dy.device) if has_bias else None
    check(lib().vcnn_pool_layer_backward(C.byref(geom), int(mode), _p(y), int(act), _p(dy),
                                         _p(arg), _p(dx), _p(dbias), _stream()))
    return dx, dbias


def _targets(kind, targets, device):
    if kind == LossKind.softmax_ce:
        cls = torch.as_tensor(targets, dtype=torch.int32, device=device).contiguous()
        return cls, None
    return None, _cuda(torch.as_tensor(targets, device=device).float(), name="values")


def loss_forward(kind, pred, targets):
    """loss_forward (layers.hpp:402-434) -> 0-d CUDA tensor."""
    pred = _cuda(pred, name="pred")
    B = pred.shape[0]
    cls, vals = _targets(kind, targets, pred.device)
    loss = _empty(1, device=pred.device)
    check(lib().vcnn_loss_forward(int(kind), B, pred.numel() // B, _p(pred), _p(cls), _p(vals),
                                  _p(loss), _stream()))
    return loss[0]


def loss_backward(kind, pred, targets):
    """loss_backward (layers.hpp:436-468)."""
    pred = _cuda(pred, name="pred")
    B = pred.shape[0]
    cls, vals = _targets(kind, targets, pred.device)
    grad = torch.empty_like(pred)
    check(lib().vcnn_loss_backward(int(kind), B, pred.numel() // B, _p(pred), _p(cls), _p(vals),
                                   _p(grad), _stream()))
    return grad


def sgd_step(w, v, g, lr, momentum, grad_scale=1.0):
    """sgd_step (network.hpp:242-273) on flat buffers, in place."""
    w, v, g = _cuda(w, name="w"), _cuda(v, name="v"), _cuda(g, name="g")
    check(lib().vcnn_sgd_step(w.numel(), _p(w), _p(v), _p(g), float(lr), float(momentum),
                              float(grad_scale), _stream()))
