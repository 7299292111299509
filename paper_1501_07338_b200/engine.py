"""Network-level API: a device-resident drop-in for the reference's
build_network + Executor<float>(Variant::imp6) + sgd_step + Trainer
(proj/include/vcnn/network.hpp:102-130, :242-273; variants.hpp:333-359;
training.hpp:50-124), driving one `vcnn_net` handle of libvcnn_cuda.so.

Parameters, gradients, momentum and the forward trace stay in HBM; host
copies happen only when asked for (get_params, output, ...).
"""
import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from ._lib import check, lib
from .errors import BoundsError, ShapeError, TrainingError
from .spec import LossKind, NetworkSpec, PoolBackwardMode, Precision, Rng, TrainConfig

COMPONENTS = ("conv_f", "conv_b", "pool_f", "pool_b", "full_f", "full_b", "other_f", "other_b")


class _DevBuf:
    """__cuda_array_interface__ view over a library-owned device buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Network:
    """build_network(spec) on the device; owns one vcnn_net handle."""

    def __init__(self, spec: NetworkSpec, max_batch: int, precision=Precision.tf32, stream=None):
        spec.chain()  # ShapeError before touching the device
        self.spec = spec
        self.max_batch = int(max_batch)
        self.precision = Precision(precision)
        self._c_spec = spec.to_c()
        h = C.c_void_p()
        check(lib().vcnn_net_create(C.byref(self._c_spec), self.max_batch, int(precision),
                                    C.byref(h)))
        self._h = h
        self.set_stream(stream)
        self.nparams = lib().vcnn_net_num_params(self._h)
        n = len(spec.layers)
        self.w_off = (C.c_int64 * n)()
        self.w_len = (C.c_int64 * n)()
        self.b_off = (C.c_int64 * n)()
        self.b_len = (C.c_int64 * n)()
        check(lib().vcnn_net_param_layout(self._h, self.w_off, self.w_len, self.b_off,
                                          self.b_len))
        self.out_per = []
        for i in range(n):
            v = C.c_int64()
            check(lib().vcnn_net_layer_out_size(self._h, i, C.byref(v)))
            self.out_per.append(v.value)
        self.in_per = spec.input_size()
        self.units = self.out_per[-1]

    # ---- lifetime ----
    def close(self):
        if getattr(self, "_h", None):
            for d in getattr(self, "_dps", []):  # data-parallel groups attached to it
                d.close()
            lib().vcnn_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- configuration ----
    def set_stream(self, stream=None):
        self._stream = stream
        check(lib().vcnn_net_set_stream(self._h, _stream_ptr(stream)))

    def set_precision(self, precision):
        self.precision = Precision(precision)
        check(lib().vcnn_net_set_precision(self._h, int(precision)))

    # ---- ModelFile v1 (io.cpp:265-404), SURVEY 8f row 4 ----
    def save_model(self, path, dtype="f32"):
        """Write the device parameters in the reference's model format."""
        from .modelfile import save_model
        save_model(path, self.spec, self.get_params(), dtype)

    @classmethod
    def from_model(cls, path, max_batch, precision=Precision.tf32, stream=None):
        """A device network initialised from a reference model file."""
        from .modelfile import load_model
        spec, params, _ = load_model(path)
        net = cls(spec, max_batch, precision, stream)
        net.set_params(params.astype(np.float32))
        return net

    def set_fusion(self, on=True):
        """TF32 slab kernels + conv->max-pool fusion (default on)."""
        check(lib().vcnn_net_set_fusion(self._h, int(bool(on))))

    def set_trace(self, keep=True):
        """Materialise every layer output / pre-activation gradient (the
        reference's LayerTrace, variants.hpp:305-323); disables fusion."""
        check(lib().vcnn_net_set_trace(self._h, int(bool(keep))))

    def set_pool_backward_mode(self, mode):
        """Executor::set_pool_backward_mode (variants.hpp:342)."""
        check(lib().vcnn_net_set_pool_backward_mode(self._h, int(mode)))

    def enable_graph(self, on=True):
        check(lib().vcnn_net_enable_graph(self._h, int(bool(on))))

    # ---- parameters (flat NetGrads order: per layer weights, then bias) ----
    def _get(self, fn):
        out = np.empty(self.nparams, dtype=np.float32)
        check(fn(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def get_params(self):
        return self._get(lib().vcnn_net_get_params)

    def set_params(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        if flat.size != self.nparams:
            raise ShapeError(f"expected {self.nparams} parameters, got {flat.size}")
        check(lib().vcnn_net_set_params(self._h, flat.ctypes.data_as(C.c_void_p)))

    def get_grads(self):
        return self._get(lib().vcnn_net_get_grads)

    def get_velocity(self):
        return self._get(lib().vcnn_net_get_velocity)

    def set_velocity(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        check(lib().vcnn_net_set_velocity(self._h, flat.ctypes.data_as(C.c_void_p)))

    def layer_params(self, flat, i):
        """(weights, bias) slices of layer i from a flat buffer."""
        w = flat[self.w_off[i]:self.w_off[i] + self.w_len[i]]
        b = flat[self.b_off[i]:self.b_off[i] + self.b_len[i]]
        return w, b

    def device_tensors(self):
        """(params, grads, velocity) as torch CUDA views (no copy) -- e.g. to
        all-reduce the gradient buffer in place.  `params` is read-only unless
        params_updated() is called after writing it (the conv kernels read
        tf32 weight images derived from it)."""
        p, g, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().vcnn_net_device_buffers(self._h, C.byref(p), C.byref(g), C.byref(v)))
        mk = lambda q: torch.as_tensor(_DevBuf(q.value, (self.nparams,), "<f4"), device="cuda")
        return mk(p), mk(g), mk(v)

    def params_updated(self):
        """Re-derive the conv weight images after params were written through
        device_tensors()[0] (stream-ordered)."""
        check(lib().vcnn_net_params_updated(self._h))

    def set_nonfinite_guard(self, on=True):
        """Trainer::fit's non-finite stop on the device: while on, a step with
        a non-finite loss skips its update (and all later ones until re-armed)."""
        check(lib().vcnn_net_set_nonfinite_guard(self._h, int(bool(on))))

    def grads_tensor(self):
        """The flat gradient buffer (NetGrads order) as a torch CUDA view:
        the one buffer a data-parallel step all-reduces (dp.DataParallel)."""
        return self.device_tensors()[1]

    def input_tensors(self):
        """(x [max_batch, in], cls [max_batch], values [max_batch, units]) views."""
        x, c, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().vcnn_net_input_buffers(self._h, C.byref(x), C.byref(c), C.byref(v)))
        X = torch.as_tensor(_DevBuf(x.value, (self.max_batch, self.in_per), "<f4"), device="cuda")
        Cl = torch.as_tensor(_DevBuf(c.value, (self.max_batch,), "<i4"), device="cuda")
        V = torch.as_tensor(_DevBuf(v.value, (self.max_batch, self.units), "<f4"), device="cuda")
        return X, Cl, V

    # ---- data ----
    def load_batch(self, x, cls=None, values=None):
        """Stage a device batch (torch CUDA tensors) into the input slots."""
        B = x.shape[0]
        x = x.contiguous().float()
        c = None if cls is None else cls.to(torch.int32).contiguous()
        v = None if values is None else values.contiguous().float()
        check(lib().vcnn_net_set_batch_device(self._h, B, C.c_void_p(x.data_ptr()),
                                              None if c is None else C.c_void_p(c.data_ptr()),
                                              None if v is None else C.c_void_p(v.data_ptr())))
        return B

    def set_batch_ring(self, x_pool=None, t_pool=None):
        """Device batch ring (vcnn_net_set_batch_ring): x_pool [nbatch, B, in]
        and t_pool [nbatch, B] class ids (int32) or [nbatch, B, units] targets,
        resident on the device; every following train step stages the ring's
        next batch itself (inside its graph).  No arguments detach the ring."""
        if x_pool is None:
            self._ring = None
            check(lib().vcnn_net_set_batch_ring(self._h, 0, 0, None, 0, None, 0))
            return
        x = x_pool.contiguous().float()
        t = t_pool.contiguous()
        t = t.to(torch.int32) if not t.is_floating_point() else t.float()
        nb, B = x.shape[0], x.shape[1]
        self._ring = (x, t)  # keep the buffers alive while attached
        check(lib().vcnn_net_set_batch_ring(self._h, int(nb), int(B), C.c_void_p(x.data_ptr()),
                                            int(x[0].numel()), C.c_void_p(t.data_ptr()),
                                            int(t[0].numel())))

    # ---- execution (stream-ordered) ----
    def forward_backward(self, batch):
        check(lib().vcnn_net_forward_backward(self._h, int(batch)))

    def forward(self, batch):
        check(lib().vcnn_net_forward(self._h, int(batch)))

    def sgd_step(self, lr, momentum, grad_scale=1.0):
        check(lib().vcnn_net_sgd_step(self._h, float(lr), float(momentum), float(grad_scale)))

    def train_step(self, batch, lr, momentum):
        check(lib().vcnn_net_train_step(self._h, int(batch), float(lr), float(momentum)))

    def train_steps(self, nsteps, batch, lr, momentum):
        """nsteps train steps, up to 8 per graph launch (vcnn_net_train_steps)."""
        check(lib().vcnn_net_train_steps(self._h, int(nsteps), int(batch), float(lr),
                                         float(momentum)))

    def train_step_host(self, x, cls=None, values=None, lr=0.01, momentum=0.0):
        """End to end: host batch in -> H2D -> step -> D2H loss (synchronous)."""
        x = np.ascontiguousarray(x, dtype=np.float32) if not isinstance(x, torch.Tensor) else x
        B = x.shape[0]
        keep = []

        def ptr(a, dt):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                a = a.contiguous()
                keep.append(a)
                return C.c_void_p(a.data_ptr())
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(C.c_void_p)

        loss = C.c_float()
        check(lib().vcnn_net_train_step_host(self._h, B, ptr(x, np.float32), ptr(cls, np.int32),
                                             ptr(values, np.float32), float(lr), float(momentum),
                                             C.byref(loss)))
        return loss.value

    def train_host_stream(self, x, cls=None, values=None, lr=0.01, momentum=0.0, steps=None):
        """End to end over a stream of host batches (vcnn_net_train_host_stream):
        x is [steps][B][...] (or one batch [B][...] reused for `steps` steps);
        the H2D copy of each batch overlaps the previous step.  Returns the
        per-step losses.  Pass pinned torch tensors for overlapped copies."""
        keep = []

        def prep(a, dt, tdt):
            if a is None:
                return None, None
            if isinstance(a, torch.Tensor):
                a = a.contiguous() if a.dtype == tdt else a.to(tdt).contiguous()
                keep.append(a)
                return a, C.c_void_p(a.data_ptr())
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a, a.ctypes.data_as(C.c_void_p)

        xa, xp = prep(x, np.float32, torch.float32)
        ca, cp = prep(cls, np.int32, torch.int32)
        va, vp = prep(values, np.float32, torch.float32)
        ta = ca if ca is not None else va
        per_x = self.in_per
        if steps is None:  # [steps][B][...]
            steps, B = xa.shape[0], xa.shape[1]
            xs, ts = B * per_x, ta[0].numel() if isinstance(ta, torch.Tensor) else ta[0].size
        else:  # one batch, reused
            B, xs, ts = xa.shape[0], 0, 0
        losses = np.empty(steps, dtype=np.float32)
        check(lib().vcnn_net_train_host_stream(self._h, int(steps), int(B), xp, int(xs), cp, vp,
                                               int(ts), float(lr), float(momentum),
                                               losses.ctypes.data_as(C.c_void_p)))
        return losses

    def forward_host(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        B = x.shape[0]
        out = np.empty((B, self.units), dtype=np.float32)
        check(lib().vcnn_net_forward_host(self._h, B, x.ctypes.data_as(C.c_void_p),
                                          out.ctypes.data_as(C.c_void_p)))
        return out

    # ---- results ----
    def loss(self):
        v = C.c_float()
        check(lib().vcnn_net_get_loss(self._h, C.byref(v)))
        return v.value

    def output(self, batch=None):
        out = np.empty((self.max_batch, self.units), dtype=np.float32)
        check(lib().vcnn_net_get_output(self._h, out.ctypes.data_as(C.c_void_p)))
        return out[: (batch or self.max_batch)]

    def layer_output(self, i, batch=None):
        out = np.empty((self.max_batch, self.out_per[i]), dtype=np.float32)
        check(lib().vcnn_net_get_layer_output(self._h, i, out.ctypes.data_as(C.c_void_p)))
        return out[: (batch or self.max_batch)]

    def layer_grad(self, i, batch=None):
        """Gradient w.r.t. layer i's pre-activation from the last backward pass."""
        out = np.empty((self.max_batch, self.out_per[i]), dtype=np.float32)
        check(lib().vcnn_net_get_layer_grad(self._h, i, out.ctypes.data_as(C.c_void_p)))
        return out[: (batch or self.max_batch)]

    def pool_arg(self, i, batch=None):
        out = np.empty((self.max_batch, self.out_per[i]), dtype=np.int64)
        check(lib().vcnn_net_get_pool_arg(self._h, i, out.ctypes.data_as(C.c_void_p)))
        return out[: (batch or self.max_batch)]

    def kernels_per_step(self):
        v = C.c_int()
        check(lib().vcnn_net_kernels_per_step(self._h, C.byref(v)))
        return v.value

    def enable_breakdown(self, on=True):
        check(lib().vcnn_net_enable_breakdown(self._h, int(bool(on))))

    def read_op_timing(self):
        """{(layer, op): (seconds, launches)} with op in fwd/wgrad/dgrad/loss/sgd
        (layer -1 for whole-net ops), from CUDA events in breakdown mode."""
        n = (len(self.spec.layers) + 1) * 5
        s = (C.c_double * n)()
        c = (C.c_int64 * n)()
        check(lib().vcnn_net_read_op_timing(self._h, s, c))
        names = ("fwd", "wgrad", "dgrad", "loss", "sgd")
        out = {}
        for i in range(n):
            if c[i]:
                out[(i // 5 - 1, names[i % 5])] = (s[i], c[i])
        return out

    def read_breakdown(self):
        s = (C.c_double * 8)()
        check(lib().vcnn_net_read_breakdown(self._h, s))
        return dict(zip(COMPONENTS, list(s)))


# ---------------------------------------------------------------------------
# Executor / RunResult / Trainer mirrors
# ---------------------------------------------------------------------------
@dataclass
class RunResult:  # variants.hpp:325-331
    output: np.ndarray
    loss: float = 0.0
    grads: Optional[np.ndarray] = None
    has_grads: bool = False


class Executor:
    """Executor<float>(Variant::imp6) (variants.hpp:333-359) over a device Network."""

    def __init__(self, precision=Precision.tf32):
        self.precision = Precision(precision)
        self._pool_mode = PoolBackwardMode.exact

    def set_pool_backward_mode(self, m):
        self._pool_mode = PoolBackwardMode(m)

    def pool_backward_mode(self):
        return self._pool_mode

    def run_batch(self, net: Network, batch, targets=None) -> RunResult:
        """batch: host array [B][C][H][W]; targets: class list (softmax_ce) or
        value array (mse); None -> forward only."""
        x = np.ascontiguousarray(batch, dtype=np.float32)
        B = x.shape[0]
        net.set_precision(self.precision)
        net.set_pool_backward_mode(self._pool_mode)
        dev = torch.device("cuda")
        xt = torch.from_numpy(x.reshape(B, -1)).to(dev)
        if targets is None:
            net.load_batch(xt)
            net.forward(B)
            return RunResult(output=net.output(B).copy())
        if net.spec.loss == LossKind.softmax_ce:
            cls = np.asarray(targets, dtype=np.int64)
            if cls.size != B:
                raise ShapeError(f"loss: {cls.size} class targets for {B} samples")
            if (cls < 0).any() or (cls >= net.units).any():
                bad = int(cls[(cls < 0) | (cls >= net.units)][0])
                raise BoundsError(f"loss: class index {bad} out of range [0,{net.units})")
            net.load_batch(xt, cls=torch.from_numpy(cls.astype(np.int32)).to(dev))
        else:
            vals = np.ascontiguousarray(targets, dtype=np.float32).reshape(B, -1)
            if vals.shape[1] != net.units:
                raise ShapeError("loss: prediction vs target shape mismatch")
            net.load_batch(xt, values=torch.from_numpy(vals).to(dev))
        net.forward_backward(B)
        return RunResult(output=net.output(B).copy(), loss=net.loss(), grads=net.get_grads(),
                         has_grads=True)

    def forward(self, net: Network, batch):
        return self.run_batch(net, batch, None).output


def predict_classes(out) -> List[int]:
    """network.hpp:179-192 (ties -> lowest index)."""
    return [int(i) for i in np.argmax(np.asarray(out).reshape(len(out), -1), axis=1)]


class Trainer:
    """Trainer<float>::fit / evaluate_accuracy (training.hpp:50-124) with the
    whole step device-resident: per batch one H2D of the gathered samples,
    one graph-replayed step, one D2H of the loss."""

    def __init__(self, cfg: TrainConfig, precision=Precision.tf32, use_graph=True):
        cfg.validate()
        self.cfg = cfg
        self.precision = Precision(precision)
        self.use_graph = use_graph

    def fit(self, net: Network, images, targets, resident=False, dp=None):
        """resident=True: the dataset is uploaded once and every epoch runs on
        the device (vcnn_net_train_epoch: permutation from the reference Rng,
        index-gather kernel, graph-replayed steps, one D2H of the epoch's
        losses).  A non-finite batch loss trips a device guard that skips
        that batch's update and every later one, so the weights (and the
        located layer) are those the offending batch ran on, as in the
        reference (training.hpp:77-80); the error is raised after the epoch."""
        images = np.ascontiguousarray(images, dtype=np.float32)
        count = images.shape[0]
        if count < 1:
            raise TrainingError("fit: empty dataset")
        if dp is not None and dp.world > 1:
            return self._fit_dp(net, images, targets, dp)
        if resident:
            return self._fit_resident(net, images, targets)
        net.set_precision(self.precision)
        net.enable_graph(self.use_graph)
        rng = Rng(self.cfg.seed)
        order = list(range(count))
        epoch_loss = []
        is_ce = net.spec.loss == LossKind.softmax_ce
        tg = np.asarray(targets)
        # a non-finite batch loss must stop training BEFORE that batch's
        # sgd_step (training.hpp:77-80); the step runs fwd+bwd+update in one
        # call, so the device guard skips the update
        net.set_nonfinite_guard(True)
        try:
            return self._fit_host(net, images, tg, count, rng, order, epoch_loss, is_ce)
        finally:
            net.set_nonfinite_guard(False)

    def _fit_host(self, net, images, tg, count, rng, order, epoch_loss, is_ce):
        for epoch in range(self.cfg.epochs):
            rng.shuffle(order)
            loss_sum, batches = 0.0, 0
            for start in range(0, count, self.cfg.batch):
                ids = order[start:start + self.cfg.batch]
                xb = images[ids]  # gather_batch (network.hpp:165-176)
                if is_ce:
                    loss = net.train_step_host(xb, cls=tg[ids].astype(np.int32),
                                               lr=self.cfg.lr, momentum=self.cfg.momentum)
                else:
                    loss = net.train_step_host(xb, values=tg[ids].reshape(len(ids), -1),
                                               lr=self.cfg.lr, momentum=self.cfg.momentum)
                if not np.isfinite(loss):
                    raise TrainingError(
                        f"non-finite loss at epoch {epoch}, batch {batches}; first non-finite "
                        f"output at {self._locate_nonfinite(net, len(ids))}")
                loss_sum += loss
                batches += 1
            epoch_loss.append(loss_sum / batches)
        return epoch_loss

    def _fit_dp(self, net: Network, images, targets, dp):
        """Data-parallel fit: every rank draws the same seeded
        permutation and trains on its contiguous slice of each global batch
        (dp.epoch_shards); the net's update is the group exchange weighted by
        the shard sizes, so the replicas follow the single-GPU trajectory.
        The epoch loss is the mean of the global-batch losses
        (sum_p B_p/B * loss_p, gathered over torch.distributed)."""
        import torch.distributed as dist

        from .dp import epoch_shards
        net.set_precision(self.precision)
        net.enable_graph(self.use_graph)
        count = images.shape[0]
        is_ce = net.spec.loss == LossKind.softmax_ce
        tg = np.asarray(targets)
        rng = Rng(self.cfg.seed)
        order = list(range(count))
        epoch_loss = []
        for epoch in range(self.cfg.epochs):
            rng.shuffle(order)
            total, batches = 0.0, 0
            for ids, sizes in epoch_shards(order, self.cfg.batch, dp.rank, dp.world):
                dp.set_shards(sizes)
                kw = (dict(cls=tg[ids].astype(np.int32)) if is_ce
                      else dict(values=tg[ids].reshape(len(ids), -1)))
                loss = net.train_step_host(images[ids], lr=self.cfg.lr,
                                           momentum=self.cfg.momentum, **kw)
                t = torch.tensor([loss * len(ids) / sum(sizes)], dtype=torch.float64,
                                 device="cuda" if dist.get_backend() == "nccl" else "cpu")
                dist.all_reduce(t)
                g = float(t.item())
                if not np.isfinite(g):
                    raise TrainingError(f"non-finite loss at epoch {epoch}, batch {batches}")
                total += g
                batches += 1
            epoch_loss.append(total / batches)
        return epoch_loss

    def _fit_resident(self, net: Network, images, targets):
        count = images.shape[0]
        is_ce = net.spec.loss == LossKind.softmax_ce
        net.set_precision(self.precision)
        net.enable_graph(self.use_graph)
        dev = torch.device("cuda")
        X = torch.from_numpy(images.reshape(count, -1)).to(dev)
        tg = np.asarray(targets)
        Ct = Vt = None
        if is_ce:
            cls = tg.astype(np.int32).reshape(count)
            bad = (cls < 0) | (cls >= net.units)
            if bad.any():  # layers.hpp:413-415, checked once at upload
                raise BoundsError(f"loss: class index {int(cls[bad][0])} out of range "
                                  f"[0,{net.units})")
            Ct = torch.from_numpy(cls).to(dev)
        else:
            Vt = torch.from_numpy(tg.reshape(count, -1).astype(np.float32)).to(dev)
        nb = -(-count // self.cfg.batch)
        losses = torch.empty(nb, device=dev)
        order_t = torch.empty(count, dtype=torch.int32, device=dev)
        rng = Rng(self.cfg.seed)
        order = list(range(count))
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        epoch_loss = []
        for epoch in range(self.cfg.epochs):
            rng.shuffle(order)  # Rng::shuffle (common.hpp:84-90), not reset between epochs
            order_t.copy_(torch.tensor(order, dtype=torch.int32))
            check(lib().vcnn_net_train_epoch(net._h, ptr(X), ptr(Ct), ptr(Vt), count,
                                             ptr(order_t), self.cfg.batch, self.cfg.lr,
                                             self.cfg.momentum, ptr(losses)))
            ls = losses.cpu().numpy().astype(np.float64)
            if not np.isfinite(ls).all():
                k = int(np.argmin(np.isfinite(ls)))
                ids = order[k * self.cfg.batch:(k + 1) * self.cfg.batch]
                net.forward_host(images[ids])
                raise TrainingError(
                    f"non-finite loss at epoch {epoch}, batch {k}; first non-finite output at "
                    f"{self._locate_nonfinite(net, len(ids))}")
            epoch_loss.append(float(ls.mean()))
        return epoch_loss

    @staticmethod
    def _locate_nonfinite(net: Network, B):
        """locate_nonfinite (training.hpp:28-45): first layer whose output is
        not finite -- the staged batch is re-run with the full trace kept
        (fused layers do not materialise their conv outputs)."""
        net.set_trace(True)
        try:
            net.forward(B)
            for i, L in enumerate(net.spec.layers):
                if not np.isfinite(net.layer_output(i, B)).all():
                    kind = type(L).__name__.replace("Spec", "").lower()
                    kind = {"conv": "conv", "pool": "pool", "full": "full"}.get(kind, kind)
                    return f"layer {i} ({kind})"
            return "loss head"
        finally:
            net.set_trace(False)

    def evaluate_accuracy(self, net: Network, images, labels):
        images = np.ascontiguousarray(images, dtype=np.float32)
        count = images.shape[0]
        if count == 0:
            return 0.0
        correct = 0
        for start in range(0, count, self.cfg.batch):
            xb = images[start:start + self.cfg.batch]
            pred = predict_classes(net.forward_host(xb))
            correct += sum(int(p == l) for p, l in zip(pred, labels[start:start + len(xb)]))
        return correct / count
