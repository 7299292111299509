"""Host-side mirror of the reference's declarative types.

Mirrors proj/include/vcnn/network.hpp:12-89 (ConvSpec, PoolSpec, FullSpec,
NetworkSpec, TrainConfig), layers.hpp:13 / :375 (Activation, LossKind),
vectorize.hpp:127 / :217 (PoolMode, PoolBackwardMode) and common.hpp:51-96
(Rng), with the same field names and defaults, plus the benchmark
configurations of BASELINE.json.
"""
import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Sequence, Tuple, Union

from .errors import ConfigError, ShapeError


class Activation(IntEnum):  # layers.hpp:13
    identity = 0
    relu = 1
    sigmoid = 2
    tanh = 3


class PoolMode(IntEnum):  # vectorize.hpp:127
    max = 0
    avg = 1


class PoolBackwardMode(IntEnum):  # vectorize.hpp:217
    exact = 0
    paper_nn = 1


class LossKind(IntEnum):  # layers.hpp:375
    softmax_ce = 0
    mse = 1


class Precision(IntEnum):
    """Arithmetic of the GEMM-shaped kernels (include/vcnn_cuda.h)."""
    tf32 = 0      # tcgen05 kind::tf32, fp32 accumulate
    tf32x3 = 1    # split hi/lo, 3 MMAs: fp32-faithful
    fp32 = 2      # SIMT FMA


KIND_CONV, KIND_POOL, KIND_FULL = 0, 1, 2


@dataclass
class ConvSpec:  # network.hpp:12-17
    maps: int = 1
    kh: int = 3
    kw: int = 3
    stride: int = 1
    act: Activation = Activation.relu


@dataclass
class PoolSpec:  # network.hpp:19-25
    ph: int = 2
    pw: int = 2
    stride: int = 2
    mode: PoolMode = PoolMode.max
    bias: bool = False
    act: Activation = Activation.identity


@dataclass
class FullSpec:  # network.hpp:27-30
    units: int = 1
    act: Activation = Activation.relu


LayerSpec = Union[ConvSpec, PoolSpec, FullSpec]


def _conv_out(n, k, s):
    return (n - k) // s + 1


@dataclass
class NetworkSpec:  # network.hpp:37-73
    input: Tuple[int, int, int] = (1, 1, 1)  # h, w, c of one sample
    layers: List[LayerSpec] = field(default_factory=list)
    loss: LossKind = LossKind.softmax_ce
    seed: int = 0

    def chain(self) -> List[Tuple[int, int, int]]:
        """Per-layer single-sample output shapes (h, w, c); ShapeError on a broken
        chain, prefixed 'layer i: ' like network.hpp:61-63."""
        h, w, c = self.input
        if min(h, w, c) < 1:
            raise ShapeError("shape extent must be >= 1")
        out = []
        for i, L in enumerate(self.layers):
            try:
                if isinstance(L, ConvSpec):
                    if L.kh < 1 or L.kw < 1 or L.stride < 1 or L.kh > h or L.kw > w:
                        raise ShapeError(f"kernel {L.kh}x{L.kw} exceeds input {h}x{w}"
                                         if L.kh > h or L.kw > w else "invalid kernel/stride")
                    if L.maps < 1:
                        raise ShapeError("shape extent must be >= 1")
                    h, w, c = _conv_out(h, L.kh, L.stride), _conv_out(w, L.kw, L.stride), L.maps
                elif isinstance(L, PoolSpec):
                    if L.ph < 1 or L.pw < 1 or L.stride < 1 or L.ph > h or L.pw > w:
                        raise ShapeError(f"pooling window {L.ph}x{L.pw} exceeds input {h}x{w}"
                                         if L.ph > h or L.pw > w else "invalid window/stride")
                    h, w = _conv_out(h, L.ph, L.stride), _conv_out(w, L.pw, L.stride)
                elif isinstance(L, FullSpec):
                    if L.units < 1:
                        raise ShapeError("full layer needs units >= 1")
                    h, w, c = 1, 1, L.units
                else:
                    raise ConfigError(f"unknown layer spec {L!r}")
            except ShapeError as e:
                raise ShapeError(f"layer {i}: {e}") from None
            out.append((h, w, c))
        return out

    def output_shape(self):
        ch = self.chain()
        return ch[-1] if ch else self.input

    def output_units(self) -> int:
        h, w, c = self.output_shape()
        return h * w * c

    def input_size(self) -> int:
        h, w, c = self.input
        return h * w * c

    # ---- C struct (vcnn_net_spec; identical layout to the oracle's orc_net) ----
    def to_c(self):
        from ._lib import LayerSpecC, NetSpecC
        arr = (LayerSpecC * max(1, len(self.layers)))()
        for i, L in enumerate(self.layers):
            arr[i] = LayerSpecC(*layer_fields(L))
        spec = NetSpecC(self.input[0], self.input[1], self.input[2], len(self.layers),
                        C.cast(arr, C.POINTER(LayerSpecC)), int(self.loss), self.seed)
        spec._keep = arr  # keep the array alive with the struct
        return spec


def layer_fields(L: LayerSpec):
    """(kind, units, kh, kw, stride, pool_mode, pool_bias, act) of one layer."""
    if isinstance(L, ConvSpec):
        return (KIND_CONV, L.maps, L.kh, L.kw, L.stride, 0, 0, int(L.act))
    if isinstance(L, PoolSpec):
        return (KIND_POOL, 0, L.ph, L.pw, L.stride, int(L.mode), int(bool(L.bias)), int(L.act))
    return (KIND_FULL, L.units, 0, 0, 1, 0, 0, int(L.act))


@dataclass
class TrainConfig:  # network.hpp:75-89
    lr: float = 0.01
    momentum: float = 0.0
    batch: int = 1
    epochs: int = 1
    seed: int = 0

    def validate(self):
        if not self.lr > 0:
            raise ConfigError("learning rate must be positive")
        if self.momentum < 0 or self.momentum >= 1:
            raise ConfigError("momentum must be in [0,1)")
        if self.batch < 1:
            raise ConfigError("batch size must be >= 1")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")


class Rng:
    """common.hpp:51-96: std::mt19937_64 with portable value extraction."""

    _N, _M = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self._N
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self._mt, self._idx = mt, self._N

    def next_u64(self) -> int:
        if self._idx >= self._N:
            mt = self._mt
            for i in range(self._N):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % self._N] & 0x7FFFFFFF)
                y = x >> 1
                if x & 1:
                    y ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + self._M) % self._N] ^ y
            self._idx = 0
        x = self._mt[self._idx]
        self._idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x &= 0xFFFFFFFFFFFFFFFF
        x ^= x >> 43
        return x

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        return u if (lo == 0.0 and hi == 1.0) else lo + (hi - lo) * u

    def uniform_int(self, n: int) -> int:
        v = int(self.uniform() * n)
        return v if v < n else n - 1

    def shuffle(self, seq: list):
        """Fisher-Yates exactly as common.hpp:84-90."""
        for i in range(len(seq) - 1, 0, -1):
            j = self.uniform_int(i + 1)
            seq[i], seq[j] = seq[j], seq[i]


# ---------------------------------------------------------------------------
# Benchmark configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------
A = Activation


def lenet_scale1_analog(seed=7) -> NetworkSpec:
    """bench_preset("scale1-analog") (bench.cpp:158-167)."""
    return NetworkSpec((28, 28, 1), [ConvSpec(20, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     ConvSpec(50, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     FullSpec(500, A.relu), FullSpec(100, A.relu),
                                     FullSpec(10, A.identity)], LossKind.softmax_ce, seed)


def lenet_caffe(seed=7) -> NetworkSpec:
    """BASELINE.json configs[0]: conv20-pool-conv50-pool-fc500-softmax(10)."""
    return NetworkSpec((28, 28, 1), [ConvSpec(20, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     ConvSpec(50, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     FullSpec(500, A.relu), FullSpec(10, A.identity)],
                       LossKind.softmax_ce, seed)


def cifar3(seed=7) -> NetworkSpec:
    """BASELINE.json configs[1]: 32x32x3, conv5x5 32/32/64 + pooling + fc10."""
    return NetworkSpec((32, 32, 3), [ConvSpec(32, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     ConvSpec(32, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     ConvSpec(64, 5, 5, 1, A.relu), FullSpec(10, A.identity)],
                       LossKind.softmax_ce, seed)


def scale2_mini(seed=7, out_units=1000) -> NetworkSpec:
    """bench_preset("scale2-mini") (bench.cpp:169-177)."""
    return NetworkSpec((32, 32, 3), [ConvSpec(32, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     ConvSpec(64, 5, 5, 1, A.relu), PoolSpec(2, 2, 2),
                                     FullSpec(2000, A.relu), FullSpec(out_units, A.identity)],
                       LossKind.softmax_ce, seed)


def denoise16(seed=7) -> NetworkSpec:
    """BASELINE.json configs[2]: 64x64 patches, 16x16 first-layer kernels, MSE."""
    return NetworkSpec((64, 64, 1), [ConvSpec(64, 16, 16, 1, A.relu), ConvSpec(64, 1, 1, 1, A.relu),
                                     ConvSpec(1, 8, 8, 1, A.identity)], LossKind.mse, seed)


def deconv121(seed=7) -> NetworkSpec:
    """BASELINE.json configs[3]: 121x1 / 1x121 separable kernels on 184x184."""
    return NetworkSpec((184, 184, 1), [ConvSpec(38, 121, 1, 1, A.identity),
                                       ConvSpec(38, 1, 121, 1, A.relu),
                                       ConvSpec(1, 5, 5, 1, A.identity)], LossKind.mse, seed)


def single_conv(channels=64, k=5, hw=32, seed=7) -> NetworkSpec:
    """BASELINE.json configs[4]: one conv layer C->C, kxk, relu, MSE."""
    return NetworkSpec((hw, hw, channels), [ConvSpec(channels, k, k, 1, A.relu)], LossKind.mse,
                       seed)


PRESETS = {
    "lenet-caffe": lenet_caffe,
    "scale1-analog": lenet_scale1_analog,
    "cifar3": cifar3,
    "scale2-mini": scale2_mini,
    "denoise16": denoise16,
    "deconv121": deconv121,
    "single-conv": single_conv,
}
