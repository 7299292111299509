"""pytest configuration: registers the `gpu` marker and makes sure the
in-tree artefacts exist (the oracle checker always; the CUDA library when a
build toolchain is present)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    # the C restatement of the oracle is cheap to build; do it up front
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), so])


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def vlib():
    """The product library; built in-tree if missing (nvcc cross-compiles)."""
    so = os.path.join(ROOT, "paper_1501_07338_b200", "libvcnn_cuda.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "-j8", "-C", ROOT, "lib"])
    from paper_1501_07338_b200 import _lib
    return _lib.lib()
