"""VCNN model file v1: export device-trained parameters in
the reference's on-disk format so its CPU `predict` / oracle can load them,
and import reference-trained models into the device engine.

Format (proj/src/io.cpp:265-307 save_model, :309-404 load_model), all
integers little-endian:
    "VCNN" | u32 version=1 | u8 dtype (0 f32, 1 f64) | u32 h, w, c | u8 loss
    (0 softmax_ce, 1 mse) | u64 seed | u32 nlayers | per layer: u8 kind
    (0 conv: u32 maps,kh,kw,stride, u8 act | 1 pool: u32 ph,pw,stride, u8 mode,
    u8 bias, u8 act | 2 full: u32 units, u8 act) | u32 nblobs | per blob: u8
    dtype, u32 ndims, u32 dims..., u64 nbytes, payload | u64 FNV-1a of all
    preceding bytes.
Blobs are the parameters in NetGrads order (model_from_network, io.hpp:193-
216): conv weights [K][C*kh*kw] + bias [K], pool bias [C] when present, full
weights [out][in] + bias [out] -- the engine's flat layout, so a flat
parameter vector maps onto blobs with no reordering.  Written atomically
(temp file + rename, io.cpp:406-416).
"""
import os
import struct
from typing import List, Tuple

import numpy as np

from .errors import ConfigError, ParseError
from .spec import (Activation, ConvSpec, FullSpec, LossKind, NetworkSpec, PoolMode, PoolSpec)

VERSION = 1


def fnv1a(data: bytes) -> int:
    """64-bit FNV-1a over the file body (io.cpp:82-89)."""
    h = 0xCBF29CE484222325
    prime = 0x100000001B3
    mask = 0xFFFFFFFFFFFFFFFF
    for b in memoryview(data):
        h = ((h ^ b) * prime) & mask
    return h


def _blob_shapes(spec: NetworkSpec) -> List[Tuple[int, ...]]:
    shapes, (h, w, c) = [], spec.input
    for L, (oh, ow, oc) in zip(spec.layers, spec.chain()):
        if isinstance(L, ConvSpec):
            shapes += [(L.maps, c * L.kh * L.kw), (L.maps,)]
        elif isinstance(L, PoolSpec):
            if L.bias:
                shapes.append((c,))
        else:
            shapes += [(L.units, h * w * c), (L.units,)]
        h, w, c = oh, ow, oc
    return shapes


def save_model(path: str, spec: NetworkSpec, params, dtype: str = "f32") -> None:
    """save_model(model_from_network(net)) for a flat parameter vector."""
    spec.chain()
    flat = np.asarray(params, dtype=np.float32 if dtype == "f32" else np.float64).ravel()
    shapes = _blob_shapes(spec)
    if sum(int(np.prod(s)) for s in shapes) != flat.size:
        raise ConfigError("save_model: parameter count does not match the spec")
    out = bytearray(b"VCNN")
    out += struct.pack("<IB", VERSION, 0 if dtype == "f32" else 1)
    out += struct.pack("<IIIBQI", spec.input[0], spec.input[1], spec.input[2],
                       0 if spec.loss == LossKind.softmax_ce else 1, spec.seed, len(spec.layers))
    for L in spec.layers:
        if isinstance(L, ConvSpec):
            out += struct.pack("<BIIIIB", 0, L.maps, L.kh, L.kw, L.stride, int(L.act))
        elif isinstance(L, PoolSpec):
            out += struct.pack("<BIIIBBB", 1, L.ph, L.pw, L.stride,
                               0 if L.mode == PoolMode.max else 1, 1 if L.bias else 0, int(L.act))
        else:
            out += struct.pack("<BIB", 2, L.units, int(L.act))
    out += struct.pack("<I", len(shapes))
    off = 0
    for s in shapes:
        n = int(np.prod(s))
        payload = flat[off:off + n].tobytes()
        off += n
        out += struct.pack("<BI", 0 if dtype == "f32" else 1, len(s))
        out += struct.pack("<" + "I" * len(s), *s)
        out += struct.pack("<Q", len(payload)) + payload
    out += struct.pack("<Q", fnv1a(bytes(out)))
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(out)
        f.flush()
        os.fsync(f.fileno())
    os.replace(tmp, path)


def _act(v: int, path: str) -> Activation:
    """activation_from_u8 (io.cpp): unknown codes are a ParseError."""
    try:
        return Activation(v)
    except ValueError:
        raise ParseError(f"model '{path}': unknown activation code {v}") from None


def load_model(path: str) -> Tuple[NetworkSpec, np.ndarray, str]:
    """load_model + network_from_model: (spec, flat parameters, dtype), with
    the reference reader's checks (io.cpp:309-404): magic, version, checksum,
    plausible input shape / layer and blob counts, layer fields >= 1, known
    enum codes, ndims <= 4, byte counts matching dims, no truncation, no
    trailing bytes -- every failure a ParseError."""
    with open(path, "rb") as f:
        b = f.read()
    if b[:4] != b"VCNN":
        raise ParseError(f"model '{path}': bad magic at offset 0 (expected VCNN)")
    if len(b) < 8:
        raise ParseError(f"model '{path}': truncated version")
    (version,) = struct.unpack_from("<I", b, 4)
    if version != VERSION:
        raise ParseError(f"model '{path}': unsupported version {version}")
    if len(b) < 16:
        raise ParseError(f"model '{path}': too short for checksum")
    body = len(b) - 8
    (stored,) = struct.unpack_from("<Q", b, body)
    if fnv1a(b[:body]) != stored:
        raise ParseError(f"model '{path}': checksum mismatch")
    off = 8

    def take(fmt, what):
        nonlocal off
        n = struct.calcsize("<" + fmt)
        if off + n > body:
            raise ParseError(f"model '{path}': truncated {what} at offset {off}")
        v = struct.unpack_from("<" + fmt, b, off)
        off += n
        return v

    (dt,) = take("B", "dtype")
    dtype = "f32" if dt == 0 else "f64"
    h, w, c = take("III", "input shape")
    if min(h, w, c) < 1 or max(h, w, c) > (1 << 20):
        raise ParseError(f"model '{path}': implausible input shape")
    loss, seed, nl = take("BQI", "header")
    if nl > 4096:
        raise ParseError(f"model '{path}': implausible layer count")
    layers = []
    for i in range(nl):
        (kind,) = take("B", "layer kind")
        if kind == 0:
            maps, kh, kw, st = take("IIII", "conv spec")
            act = _act(take("B", "conv act")[0], path)
            if min(maps, kh, kw, st) < 1:
                raise ParseError(f"model '{path}': invalid conv spec in layer {i}")
            layers.append(ConvSpec(maps, kh, kw, st, act))
        elif kind == 1:
            ph, pw, st, mode, bias = take("IIIBB", "pool spec")
            if mode > 1:
                raise ParseError(f"model '{path}': unknown pool mode")
            act = _act(take("B", "pool act")[0], path)
            if min(ph, pw, st) < 1:
                raise ParseError(f"model '{path}': invalid pool spec in layer {i}")
            layers.append(PoolSpec(ph, pw, st, PoolMode(mode), bool(bias), act))
        elif kind == 2:
            (units,) = take("I", "full units")
            act = _act(take("B", "full act")[0], path)
            if units < 1:
                raise ParseError(f"model '{path}': invalid full spec in layer {i}")
            layers.append(FullSpec(units, act))
        else:
            raise ParseError(f"model '{path}': unknown layer kind {kind} at offset {off - 1}")
    spec = NetworkSpec((h, w, c), layers, LossKind.softmax_ce if loss == 0 else LossKind.mse,
                       seed)
    (nb,) = take("I", "blob count")
    if nb > 8192:
        raise ParseError(f"model '{path}': implausible blob count")
    blobs = []
    for _ in range(nb):
        bdt, nd = take("BI", "blob header")
        if nd > 4:
            raise ParseError(f"model '{path}': blob with {nd} dims")
        dims = take("I" * nd, "blob dims")
        numel = int(np.prod(dims, dtype=np.uint64)) if nd else 1
        if numel > (1 << 36):
            raise ParseError(f"model '{path}': blob dimension overflow")
        (nbytes,) = take("Q", "blob size")
        width = 4 if bdt == 0 else 8
        if nbytes != numel * width:
            raise ParseError(f"model '{path}': blob byte count {nbytes} does not match dims "
                             f"at offset {off - 8}")
        if off + nbytes > body:
            raise ParseError(f"model '{path}': truncated blob payload at offset {off}")
        blobs.append((tuple(dims), np.frombuffer(b, np.float32 if bdt == 0 else np.float64,
                                                 numel, off)))
        off += nbytes
    if off != body:
        raise ParseError(f"model '{path}': {body - off} unexpected trailing bytes at offset {off}")
    try:
        want = _blob_shapes(spec)
    except Exception as e:  # chain validation (network_from_model -> build_network)
        raise ParseError(f"model '{path}': {e}") from None
    if len(blobs) != len(want):
        raise ParseError(f"model '{path}': {len(blobs)} parameter blobs, the spec needs "
                         f"{len(want)}")
    for (dims, _), s in zip(blobs, want):
        if dims != tuple(s):
            raise ParseError(f"model '{path}': blob shape {dims} does not match the spec {s}")
    flat = np.concatenate([a for _, a in blobs]) if blobs else np.zeros(0, np.float32)
    return spec, flat, dtype


# ---- exact-resume checkpoints ----------------------------
# The reference keeps Velocity outside the model file (network.hpp:237-240;
# Trainer restarts it at zero).  A checkpoint is the reference-readable model
# file plus a sibling "<path>.vel" in the same v1 format whose blobs are the
# velocity in NetGrads order, so momentum SGD resumes bit-exactly and the
# model file itself stays loadable by the reference.
def save_checkpoint(path: str, spec: NetworkSpec, params, velocity) -> None:
    save_model(path, spec, params)
    save_model(path + ".vel", spec, velocity)


def load_checkpoint(path: str) -> Tuple[NetworkSpec, np.ndarray, np.ndarray]:
    """(spec, params, velocity); velocity is zero (the reference's lazy
    Velocity, network.hpp:247-252) when the model has no .vel sibling."""
    spec, params, _ = load_model(path)
    vpath = path + ".vel"
    if not os.path.exists(vpath):
        return spec, params, np.zeros_like(params)
    vspec, vel, _ = load_model(vpath)
    if _blob_shapes(vspec) != _blob_shapes(spec):
        raise ParseError(f"checkpoint '{path}': velocity file does not match the model")
    return spec, params, vel
