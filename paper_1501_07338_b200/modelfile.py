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


def load_model(path: str) -> Tuple[NetworkSpec, np.ndarray, str]:
    """load_model + network_from_model: (spec, flat parameters, dtype)."""
    with open(path, "rb") as f:
        b = f.read()
    if b[:4] != b"VCNN":
        raise ParseError(f"model '{path}': bad magic at offset 0 (expected VCNN)")
    if len(b) < 17:
        raise ParseError(f"model '{path}': too short")
    (version,) = struct.unpack_from("<I", b, 4)
    if version != VERSION:
        raise ParseError(f"model '{path}': unsupported version {version}")
    body = len(b) - 8
    (stored,) = struct.unpack_from("<Q", b, body)
    if fnv1a(b[:body]) != stored:
        raise ParseError(f"model '{path}': checksum mismatch")
    off = 8

    def take(fmt):
        nonlocal off
        v = struct.unpack_from("<" + fmt, b, off)
        off += struct.calcsize("<" + fmt)
        if off > body:
            raise ParseError(f"model '{path}': truncated at offset {off}")
        return v

    (dt,) = take("B")
    dtype = "f32" if dt == 0 else "f64"
    h, w, c, loss, seed, nl = take("IIIBQI")
    layers = []
    for i in range(nl):
        (kind,) = take("B")
        if kind == 0:
            maps, kh, kw, st, act = take("IIIIB")
            layers.append(ConvSpec(maps, kh, kw, st, Activation(act)))
        elif kind == 1:
            ph, pw, st, mode, bias, act = take("IIIBBB")
            layers.append(PoolSpec(ph, pw, st, PoolMode(mode), bool(bias), Activation(act)))
        elif kind == 2:
            units, act = take("IB")
            layers.append(FullSpec(units, Activation(act)))
        else:
            raise ParseError(f"model '{path}': unknown layer kind {kind}")
    spec = NetworkSpec((h, w, c), layers, LossKind.softmax_ce if loss == 0 else LossKind.mse,
                       seed)
    (nb,) = take("I")
    parts = []
    for s in _blob_shapes(spec)[:nb] if nb == len(_blob_shapes(spec)) else []:
        bdt, nd = take("BI")
        dims = take("I" * nd)
        (nbytes,) = take("Q")
        width = 4 if bdt == 0 else 8
        if tuple(dims) != tuple(s) or nbytes != int(np.prod(dims)) * width:
            raise ParseError(f"model '{path}': blob shape {dims} does not match the spec {s}")
        parts.append(np.frombuffer(b, np.float32 if bdt == 0 else np.float64,
                                   int(np.prod(dims)), off))
        off += nbytes
    if nb != len(_blob_shapes(spec)):
        raise ParseError(f"model '{path}': {nb} parameter blobs, the spec needs "
                         f"{len(_blob_shapes(spec))}")
    if off != body:
        raise ParseError(f"model '{path}': {body - off} unexpected trailing bytes")
    flat = np.concatenate(parts) if parts else np.zeros(0, np.float32)
    return spec, flat, dtype
