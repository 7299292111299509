"""C-ABI checks that need no GPU: the library loads, exports exactly what
include/vcnn_cuda.h declares, host-side validation mirrors the reference
errors, and compute entry points fail loudly (VCNN_ECUDA) without a device."""
import ctypes as C
import os
import re

import pytest

from paper_1501_07338_b200 import _lib, spec as S
from paper_1501_07338_b200.errors import ConfigError, CudaError, GeometryError, ShapeError

from .conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "vcnn_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vcnn_[a-zA-Z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(vlib):
    names = declared_functions()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(vlib, n)]
    assert not missing, missing
    # and the Python binding covers the whole ABI
    assert sorted(_lib.exported_symbols()) == names


def test_abi_version(vlib):
    assert vlib.vcnn_abi_version() == 1


def test_geometry_validation_host_only(vlib):
    g = _lib.ConvGeometryC()
    assert vlib.vcnn_conv_geometry_init(C.byref(g), 32, 32, 3, 128, 5, 5, 1) == 0
    assert (g.out_h, g.out_w) == (28, 28)
    assert vlib.vcnn_conv_geometry_init(C.byref(g), 4, 4, 1, 1, 5, 5, 1) == 2  # GeometryError
    assert b"exceeds input" in vlib.vcnn_last_error()
    assert vlib.vcnn_conv_geometry_init(C.byref(g), 4, 4, 1, 1, 2, 2, 0) == 2
    assert vlib.vcnn_conv_geometry_init(C.byref(g), 0, 4, 1, 1, 1, 1, 1) == 1  # ShapeError
    p = _lib.PoolGeometryC()
    assert vlib.vcnn_pool_geometry_init(C.byref(p), 28, 28, 32, 128, 2, 2, 2, 0) == 0
    assert (p.out_h, p.out_w) == (14, 14)
    assert vlib.vcnn_pool_geometry_init(C.byref(p), 3, 3, 1, 1, 2, 2, 1, 0) == 0
    assert (p.out_h, p.out_w) == (2, 2)  # overlap allowed
    assert vlib.vcnn_pool_geometry_init(C.byref(p), 2, 2, 1, 1, 3, 3, 1, 0) == 2


def test_spec_chain_matches_python_mirror(vlib):
    for name, f in S.PRESETS.items():
        spec = f()
        cs = spec.to_c()
        shapes = (C.c_int * (3 * len(spec.layers)))()
        assert vlib.vcnn_net_spec_chain(C.byref(cs), shapes) == 0
        got = [tuple(shapes[3 * i:3 * i + 3]) for i in range(len(spec.layers))]
        assert got == spec.chain(), name
    bad = S.NetworkSpec((4, 4, 1), [S.ConvSpec(2, 5, 5)])
    with pytest.raises(ShapeError, match="layer 0"):
        bad.chain()
    assert vlib.vcnn_net_spec_chain(C.byref(bad.to_c()), None) == 1
    assert b"layer 0" in vlib.vcnn_last_error()


def test_status_mapping():
    with pytest.raises(GeometryError):
        _lib.check(2)
    with pytest.raises(ConfigError):
        _lib.check(6)
    assert _lib.check(0) == 0


@pytest.mark.skipif(has_gpu(), reason="checks the no-device failure mode")
def test_compute_fails_loudly_without_gpu(vlib):
    g = _lib.ConvGeometryC()
    vlib.vcnn_conv_geometry_init(C.byref(g), 8, 8, 1, 1, 3, 3, 1)
    st = vlib.vcnn_im2col(C.byref(g), None, None, None)
    assert st == 4  # VCNN_ECUDA: no CPU fallback
    with pytest.raises(CudaError):
        _lib.check(st)
    h = C.c_void_p()
    assert vlib.vcnn_net_create(C.byref(S.cifar3().to_c()), 8, 0, C.byref(h)) == 4
