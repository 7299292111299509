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
