"""The C++ host API and the reference drop-in (tests/cpp), built in-tree."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def _run(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C tests/cpp)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout


def test_cpp_api_builds_against_headers():
    """The header-only C++ API compiles and links against libvcnn_cuda.so
    (no GPU needed)."""
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"),
                           os.path.join(BIN, "test_host_api")])
    assert os.path.exists(os.path.join(BIN, "test_host_api"))


@pytest.mark.gpu
def test_cpp_host_api():
    _run("test_host_api")


@pytest.mark.gpu
def test_reference_dropin_executor():
    """vcnn::Executor<float>(imp6) vs vcnn_b200::ref::Executor on the
    reference's own Network/Tensor/Targets objects."""
    _run("test_dropin")
