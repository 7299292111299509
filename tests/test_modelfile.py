"""ModelFile v1: our writer/reader vs the reference's own
io.cpp save_model / load_model (compiled in oracle/_ref)."""
import os

import numpy as np
import pytest

import oracle_py as O
from paper_1501_07338_b200 import spec as S
from paper_1501_07338_b200.errors import ParseError
from paper_1501_07338_b200.modelfile import load_model, save_model

A = S.Activation
SPECS = {
    "cifar3": S.cifar3(),
    "mixed": S.NetworkSpec((9, 10, 2), [S.ConvSpec(3, 3, 2, 1, A.tanh),
                                        S.PoolSpec(2, 2, 1, S.PoolMode.max, True, A.sigmoid),
                                        S.FullSpec(3, A.identity)], S.LossKind.mse, 5),
}

needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")


@pytest.mark.parametrize("name", list(SPECS))
def test_roundtrip(tmp_path, name):
    spec = SPECS[name]
    p = np.random.default_rng(1).standard_normal(O.net_num_params(spec)).astype(np.float32)
    f = str(tmp_path / "m.vcnn")
    save_model(f, spec, p)
    spec2, p2, dt = load_model(f)
    assert dt == "f32" and spec2 == spec and np.array_equal(p2, p)


@needs_ref
@pytest.mark.parametrize("name", list(SPECS))
def test_ours_is_readable_by_the_reference(tmp_path, name):
    spec = SPECS[name]
    p = np.random.default_rng(2).standard_normal(O.net_num_params(spec)).astype(np.float32)
    f = str(tmp_path / "ours.vcnn")
    save_model(f, spec, p)
    assert np.array_equal(O.ref_load_model_f32(f, p.size), p)


@needs_ref
@pytest.mark.parametrize("name", list(SPECS))
def test_reference_file_is_readable_and_byte_identical(tmp_path, name):
    spec = SPECS[name]
    p = np.random.default_rng(3).standard_normal(O.net_num_params(spec)).astype(np.float32)
    f_ref, f_ours = str(tmp_path / "ref.vcnn"), str(tmp_path / "ours.vcnn")
    O.ref_save_model(spec, p.astype(np.float64), f_ref, f32=True)
    spec2, p2, _ = load_model(f_ref)
    assert spec2 == spec and np.array_equal(p2, p)
    save_model(f_ours, spec, p)
    assert open(f_ref, "rb").read() == open(f_ours, "rb").read()


def test_corruption_is_rejected(tmp_path):
    spec = SPECS["mixed"]
    p = np.zeros(O.net_num_params(spec), dtype=np.float32)
    f = str(tmp_path / "m.vcnn")
    save_model(f, spec, p)
    b = bytearray(open(f, "rb").read())
    b[20] ^= 1
    open(f, "wb").write(bytes(b))
    with pytest.raises(ParseError, match="checksum"):
        load_model(f)
    open(f, "wb").write(b"XXXX" + bytes(b[4:]))
    with pytest.raises(ParseError, match="magic"):
        load_model(f)


def _patched(raw: bytes, off: int, new: bytes) -> bytes:
    """raw with bytes at `off` replaced and the FNV-1a trailer recomputed."""
    import struct

    from paper_1501_07338_b200.modelfile import fnv1a
    b = bytearray(raw[:-8])
    b[off:off + len(new)] = new
    return bytes(b) + struct.pack("<Q", fnv1a(bytes(b)))


def test_malformed_fields_raise_parse_error(tmp_path):
    """The reference reader's validation (io.cpp:330-390) with a VALID
    checksum: every malformed field is a ParseError, never ValueError."""
    import struct
    spec = SPECS["mixed"]
    f = str(tmp_path / "m.vcnn")
    save_model(f, spec, np.zeros(O.net_num_params(spec), dtype=np.float32))
    raw = open(f, "rb").read()
    # header: magic 4 | ver 4 | dtype 1 | h w c 12 | loss 1 | seed 8 | nl 4 -> 34
    L0 = 34  # first layer: kind 1 | maps kh kw stride 16 | act 1
    cases = {
        "implausible input shape": (9, struct.pack("<I", 0)),
        "implausible layer count": (30, struct.pack("<I", 5000)),
        "invalid conv spec": (L0 + 1, struct.pack("<I", 0)),
        "unknown activation": (L0 + 17, b"\x09"),
        "unknown layer kind": (L0, b"\x07"),
    }
    for msg, (off, new) in cases.items():
        open(f, "wb").write(_patched(raw, off, new))
        with pytest.raises(ParseError, match=msg):
            load_model(f)
    # truncated payload (last blob cut, checksum recomputed)
    body = raw[:-8]
    from paper_1501_07338_b200.modelfile import fnv1a
    cut = body[:-3]
    open(f, "wb").write(cut + struct.pack("<Q", fnv1a(cut)))
    with pytest.raises(ParseError):
        load_model(f)


def test_checkpoint_roundtrip_keeps_velocity(tmp_path):
    from paper_1501_07338_b200.modelfile import load_checkpoint, save_checkpoint
    spec = SPECS["cifar3"]
    n = O.net_num_params(spec)
    rng = np.random.default_rng(4)
    p, v = rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)
    f = str(tmp_path / "ck.vcnn")
    save_checkpoint(f, spec, p, v)
    spec2, p2, v2 = load_checkpoint(f)
    assert spec2 == spec and np.array_equal(p2, p) and np.array_equal(v2, v)
    os.remove(f + ".vel")
    _, _, v3 = load_checkpoint(f)
    assert not v3.any()
